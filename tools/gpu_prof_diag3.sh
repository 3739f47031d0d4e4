#!/bin/bash
TAG=${1:-p3}
mkdir -p gpurun_out
for cfg in c2 c4 c5s8 c5; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --profile-from-start off \
      --log-file gpurun_out/launch_${cfg}_$TAG.csv python tools/profile_run.py --config $cfg --iters 1 > /dev/null 2>&1
  echo "$cfg list $?"
done
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:diagw -s 10 -c 1 \
    -o gpurun_out/prof_diagw_c4_$TAG python tools/profile_run.py --config c4 --iters 1 > gpurun_out/ncu_diagw_c4_$TAG.log 2>&1
echo c4 $?
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:diagw -s 70 -c 1 \
    -o gpurun_out/prof_diagw_c5_$TAG python tools/profile_run.py --config c5 > gpurun_out/ncu_diagw_c5_$TAG.log 2>&1
echo c5 $?
MSTRSM_LOOKAHEAD=0 timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:diagw -s 16 -c 1 \
    -o gpurun_out/prof_diagw_c2_$TAG python tools/profile_run.py --config c2 > gpurun_out/ncu_diagw_c2_$TAG.log 2>&1
echo c2 $?
