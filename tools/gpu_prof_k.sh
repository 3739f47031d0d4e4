#!/bin/bash
# Full ncu capture (with source) of one launch of a kernel on a config.
# Usage: bash tools/gpu_prof_k.sh <tag> <kernel-regex> <skip> [config] [m]
TAG=$1; K=$2; SKIP=${3:-60}; CFG=${4:-c5}; M=${5:-0}
mkdir -p gpurun_out
timeout 300 python tools/profile_run.py --config $CFG --m $M > gpurun_out/plain_$TAG.log 2>&1 || { cat gpurun_out/plain_$TAG.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:$K -s $SKIP -c ${COUNT:-1} \
    -o gpurun_out/prof_$TAG python tools/profile_run.py --config $CFG --m $M > gpurun_out/ncu_$TAG.log 2>&1
tail -3 gpurun_out/ncu_$TAG.log
