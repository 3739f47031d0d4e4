#!/bin/bash
# Small real solves: persistent warp-specialised update GEMM (default) vs the one-tile-per-CTA
# kernel (MSTRSM_GEMM=classic), interleaved on one box.  Usage (via gpurun): bash tools/exp_small_gemm.sh <tag>
TAG=${1:-s}
mkdir -p gpurun_out
OUT=gpurun_out/exp_small_gemm_$TAG.txt
: > $OUT
for rep in 1 2 3; do
for cfg in "MSTRSM_GEMM=ws" "MSTRSM_GEMM=classic" "MSTRSM_EARLY_A=1"; do
  env $cfg timeout 300 python tools/bench_rows.py --only c1,c2,trsm 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if 'z4096' in d['config']: continue
    print('$cfg', d['config'], round(d['ms_per_step'],4), 'diag', round(d.get('diag_ms_profiled_step',0),4), 'gemm', round(d.get('gemm_ms_profiled_step',0),4))
" >> $OUT
done
done
cat $OUT
