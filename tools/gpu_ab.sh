#!/bin/bash
# A/B on one box: GPU tests with the new library, then rows + c5 bench for exp/lib_base.so (A) and
# the in-tree library (B).  $1 = tag, $2 = rows (default c2,c4,c5s8,c3), $3 = "notest" to skip tests
TAG=${1:-ab}; ROWS=${2:-c2,c4,c5s8,c3}
mkdir -p gpurun_out
if [ "$3" != "notest" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_$TAG.log 2>&1
  echo "pytest exit $?" >> gpurun_out/pytest_$TAG.log; tail -2 gpurun_out/pytest_$TAG.log
fi
for v in A B A B; do
  if [ $v = A ]; then export MSTRSM_LIB=$PWD/exp/lib_base.so; else unset MSTRSM_LIB; fi
  timeout 600 python tools/bench_rows.py --only $ROWS 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['config'], round(d['ms_per_step'],3), 'diag', round(d.get('diag_ms_profiled_step',0),3), 'gemm', round(d.get('gemm_ms_profiled_step',0),3))
" | tee -a gpurun_out/ab_$TAG.txt
  if [ -n "$C5" ]; then
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    r=d['roofline']; print('$v c5', round(d['ms_per_step'],3), 'diag', round(r.get('diag_ms_per_step',0),3), 'gemm', round(r.get('gemm_ms_per_step',0),3))
" | tee -a gpurun_out/ab_$TAG.txt
  fi
done
