#!/bin/bash
mkdir -p gpurun_out
MSTRSM_DIAG=tc python tools/profile_run.py --config c4 --iters 1 > /dev/null 2>&1 && \
MSTRSM_DIAG=tc timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:diagl -s 10 -c 1 \
    -o gpurun_out/prof_diagl_c4_e4 python tools/profile_run.py --config c4 --iters 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:diagw -s 10 -c 1 \
    -o gpurun_out/prof_diagw_c4_e4 python tools/profile_run.py --config c4 --iters 1 > /dev/null 2>&1
echo done
