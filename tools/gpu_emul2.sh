#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_dist.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/pytest_dist_e5.log 2>&1; tail -2 gpurun_out/pytest_dist_e5.log
bash tools/gpu_emul.sh
