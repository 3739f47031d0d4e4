#!/bin/bash
# usage: bash tools/gpu_sanitize.sh <tool> <tag>   (one compute-sanitizer tool per gpurun call)
TOOL=${1:-racecheck}; TAG=${2:-r02}
mkdir -p gpurun_out
python tools/sanitize_run.py > gpurun_out/sanitize_plain_$TAG.log 2>&1 && \
timeout 1500 compute-sanitizer --tool $TOOL --print-limit 50 python tools/sanitize_run.py > gpurun_out/sanitize_${TOOL}_$TAG.log 2>&1
echo "exit $?" >> gpurun_out/sanitize_${TOOL}_$TAG.log
tail -5 gpurun_out/sanitize_${TOOL}_$TAG.log
