#!/bin/bash
# Small real solves on the one-tile-per-CTA update: early A issue on/off, the update's start
# trigger, with and without the diagonal kernel's trigger; GPU tests first.
TAG=${1:-s3}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_$TAG.log
tail -2 gpurun_out/pytest_$TAG.log
OUT=gpurun_out/exp_small_gemm_$TAG.txt
: > $OUT
for rep in 1 2 3; do
for cfg in ${CFGS:-"MSTRSM_GEMM_TRIGGER=0" "MSTRSM_GEMM_REAL=auto" "MSTRSM_GEMM_TRIGGER=1"}; do
  env $cfg timeout 300 python tools/bench_rows.py --only c1,c2,trsm 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if 'z4096' in d['config']: continue
    print('$cfg', d['config'], round(d['ms_per_step'],4), 'diag', round(d.get('diag_ms_profiled_step',0),4), 'gemm', round(d.get('gemm_ms_profiled_step',0),4))
" >> $OUT
done
done
sort $OUT
