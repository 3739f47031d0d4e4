#!/bin/bash
# Consumer-group stagger of the 3M update (MSTRSM_3P_PHASE) on the rows with short update launches.
TAG=${1:-p1}
mkdir -p gpurun_out
OUT=gpurun_out/exp_phase_short_$TAG.txt
: > $OUT
for rep in 1 2; do
for cfg in "MSTRSM_3P_PHASE=2" "MSTRSM_3P_PHASE=0" "MSTRSM_3P_PHASE=1"; do
  env $cfg timeout 400 python tools/bench_rows.py --only c3,c4,c5s8 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if d['config']=='c4d': continue
    print('$cfg', d['config'], round(d['ms_per_step'],3), 'gemm', round(d.get('gemm_ms_profiled_step',0),3))
" >> $OUT
done
done
sort $OUT
