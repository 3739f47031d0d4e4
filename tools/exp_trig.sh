#!/bin/bash
# Real small solves: diagl dependent-launch trigger x early A issue of gemm_ws_kernel (A/B on one box),
# then look-ahead on c1/c2.  Usage (via gpurun): bash tools/exp_trig.sh <tag>
TAG=${1:-t}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_$TAG.log
tail -2 gpurun_out/pytest_$TAG.log
OUT=gpurun_out/exp_trig_$TAG.txt
: > $OUT
for rep in 1 2 3; do
for cfg in "MSTRSM_DIAGL_TRIGGER=0 MSTRSM_EARLY_A=0" "MSTRSM_DIAGL_TRIGGER=0" "MSTRSM_DIAGL_TRIGGER=1" "MSTRSM_DIAGL_TRIGGER=1 MSTRSM_EARLY_A=0"; do
  env $cfg timeout 300 python tools/bench_rows.py --only c1,c2,trsm 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if 'z4096' in d['config']: continue
    print('$cfg', d['config'], round(d['ms_per_step'],4))
" >> $OUT
done
done
cat $OUT
ROWS=c1,c2 bash tools/exp_la_real.sh > /dev/null 2>&1
cp gpurun_out/exp_la_real.txt gpurun_out/exp_la_real_$TAG.txt
