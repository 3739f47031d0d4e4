#!/bin/bash
mkdir -p gpurun_out
for s in 0 16; do
timeout 600 ncu --section SourceCounters --section WarpStateStats --section LaunchStats --section SpeedOfLight --warp-sampling-interval 0 --clock-control none --import-source on --profile-from-start off -k regex:diagl -s $s -c 1 \
    -o gpurun_out/prof_diagl_c2_s$s python tools/profile_run.py --config c2 > gpurun_out/ncu_diagl_c2_s$s.log 2>&1
tail -1 gpurun_out/ncu_diagl_c2_s$s.log
done
