#!/bin/bash
# Finalize kernel with one round of frame loads (B = in-tree) vs the previous library (A =
# exp/lib_base.so), interleaved on one box; then the real diagonal kernel's start trigger.
TAG=${1:-f1}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_$TAG.log
tail -2 gpurun_out/pytest_$TAG.log
OUT=gpurun_out/exp_fin_$TAG.txt
: > $OUT
for rep in 1 2 3; do
for v in A B T; do
  unset MSTRSM_LIB MSTRSM_DIAGL_TRIGGER
  [ $v = A ] && export MSTRSM_LIB=$PWD/exp/lib_base.so
  [ $v = T ] && export MSTRSM_DIAGL_TRIGGER=1
  timeout 300 python tools/bench_rows.py --only c1,c2,c3,c5s8 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['config'], round(d['ms_per_step'],4))
" >> $OUT
done
done
sort $OUT
