#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --section SourceCounters --section WarpStateStats --section LaunchStats --section SpeedOfLight --section Occupancy --warp-sampling-interval 0 --clock-control none --import-source on --profile-from-start off -k regex:diagw -s 64 -c 1 \
    -o gpurun_out/prof_diagw_c5s8_mid python tools/profile_run.py --config c5s8 > gpurun_out/ncu_c5s8.log 2>&1
tail -1 gpurun_out/ncu_c5s8.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/launches_c5s8.csv python tools/profile_run.py --config c5s8 > /dev/null 2>&1
