#!/bin/bash
mkdir -p gpurun_out
MSTRSM_LOOKAHEAD=0 python tools/profile_run.py --config c2 > /dev/null 2>&1 && \
MSTRSM_LOOKAHEAD=0 timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:diagl -s 16 -c 1 \
    -o gpurun_out/prof_diagl_c2nola_e6 python tools/profile_run.py --config c2 > /dev/null 2>&1
echo done
