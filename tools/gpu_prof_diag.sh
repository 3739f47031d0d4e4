#!/bin/bash
# Launch lists (new vs round-1 diagonal kernel) and full captures of the chunked diagonal kernel.
TAG=${1:-p}
mkdir -p gpurun_out
for cfg in c2 c5s8 c4; do
  for v in new old; do
    if [ $v = old ]; then export MSTRSM_DIAG_OLD=1; else unset MSTRSM_DIAG_OLD; fi
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --profile-from-start off \
      --log-file gpurun_out/launch_${cfg}_${v}_$TAG.csv python tools/profile_run.py --config $cfg --iters 1 > /dev/null 2>&1
    echo "$cfg $v exit $?"
  done
done
unset MSTRSM_DIAG_OLD
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:diagf -s 40 -c 1 \
    -o gpurun_out/prof_diagf_c5s8_$TAG python tools/profile_run.py --config c5s8 > gpurun_out/ncu_diagf_c5s8_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:diagf -s 20 -c 1 \
    -o gpurun_out/prof_diagf_c2_$TAG python tools/profile_run.py --config c2 > gpurun_out/ncu_diagf_c2_$TAG.log 2>&1
ls gpurun_out | grep $TAG
