#!/bin/bash
# Real update GEMM kernel choice (MSTRSM_GEMM_REAL=ws|classic|auto default), interleaved on one box,
# after the full GPU test suite.  Usage (via gpurun): bash tools/exp_small_gemm2.sh <tag>
TAG=${1:-s2}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_$TAG.log
tail -2 gpurun_out/pytest_$TAG.log
OUT=gpurun_out/exp_small_gemm_$TAG.txt
: > $OUT
for rep in 1 2 3; do
for cfg in "MSTRSM_GEMM_REAL=ws" "MSTRSM_GEMM_REAL=auto" "MSTRSM_GEMM_REAL=classic"; do
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
