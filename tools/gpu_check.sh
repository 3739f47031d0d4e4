#!/bin/bash
# GPU run: probe, parity tests, bench.  Usage (via gpurun): bash tools/gpu_check.sh [pytest-args]
# Every step has its own timeout so a hang cannot eat the call's budget.
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia_smi.txt 2>&1
timeout 120 python -c "import paper_1607_01477_b200 as ms, torch; torch.cuda.init(); print('fp64 peak (dmma, dfma) TF:', ms.fp64_peak(50.0))" > gpurun_out/peak.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q --timeout 240 "$@" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 420 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.log 2>&1
echo "bench exit $?" >> gpurun_out/bench.log
