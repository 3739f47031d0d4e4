#!/bin/bash
TAG=${1:-p2}
mkdir -p gpurun_out
MSTRSM_DIAG_LPC=8 timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:diagf -s 10 -c 1 \
    -o gpurun_out/prof_diagf_c4_$TAG python tools/profile_run.py --config c4 --iters 1 > gpurun_out/ncu_diagf_c4_$TAG.log 2>&1
echo c4 $?
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:diagf -s 70 -c 1 \
    -o gpurun_out/prof_diagf_c5_$TAG python tools/profile_run.py --config c5 > gpurun_out/ncu_diagf_c5_$TAG.log 2>&1
echo c5 $?
MSTRSM_LOOKAHEAD=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --profile-from-start off \
      --log-file gpurun_out/launch_c2nola_$TAG.csv python tools/profile_run.py --config c2 > /dev/null 2>&1
MSTRSM_LOOKAHEAD=0 timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:diagf -s 16 -c 1 \
    -o gpurun_out/prof_diagf_c2nola_$TAG python tools/profile_run.py --config c2 > gpurun_out/ncu_diagf_c2nola_$TAG.log 2>&1
echo c2 $?
