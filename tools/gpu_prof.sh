#!/bin/bash
# Launch list + one full ncu capture of the update GEMM (and optionally the diag kernel).
# Usage (via gpurun): bash tools/gpu_prof.sh <config> <tag> [kernel-regex ...]
CFG=${1:-c5}; TAG=${2:-r01}; shift 2
mkdir -p gpurun_out
python tools/profile_run.py --config $CFG > gpurun_out/plain_$TAG.log 2>&1 || { echo "plain run failed"; cat gpurun_out/plain_$TAG.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/launches_${CFG}_$TAG.csv python tools/profile_run.py --config $CFG > gpurun_out/ncu_list_$TAG.log 2>&1
for K in "$@"; do
  ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:$K -s 60 -c 1 \
      -o gpurun_out/prof_${K}_${CFG}_$TAG python tools/profile_run.py --config $CFG > gpurun_out/ncu_${K}_$TAG.log 2>&1
done
ls -la gpurun_out
