#!/bin/bash
# GPU parity tests with the parity log (R20 / Delta-e histograms) kept under gpurun_out/.
TAG=${1:-t}
mkdir -p gpurun_out
export MSTRSM_PARITY_LOG=gpurun_out/parity_$TAG.jsonl
: > $MSTRSM_PARITY_LOG
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 --durations=15 "${@:2}" > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
tail -25 gpurun_out/pytest_gpu_$TAG.log
