#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/exp_dist_emul.py 8 > gpurun_out/dist_emul_r02.jsonl 2> gpurun_out/dist_emul_r02.err
timeout 600 python tools/exp_dist_emul.py 2 >> gpurun_out/dist_emul_r02.jsonl 2>> gpurun_out/dist_emul_r02.err
cat gpurun_out/dist_emul_r02.jsonl; tail -3 gpurun_out/dist_emul_r02.err
