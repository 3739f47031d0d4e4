#!/bin/bash
# ncu launch list (gpu__time_duration per launch) of one profiled c5 solve (tools/profile_run.py).
TAG=${1:-x}; CFG=${2:-c5}
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/launches_${CFG}_$TAG.csv python tools/profile_run.py --config $CFG > gpurun_out/ncu_list_$TAG.log 2>&1
tail -2 gpurun_out/ncu_list_$TAG.log
