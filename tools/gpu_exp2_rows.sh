#!/bin/bash
# parity tests + rows/c5 for the new kernel (with / without look-ahead) vs the round-1 kernel
TAG=${1:-e2}
mkdir -p gpurun_out



OUT=gpurun_out/exp_$TAG.txt
: > $OUT
run() {  # label, env...
  label=$1; shift
  env "$@" timeout 300 python tools/bench_rows.py --only ${ONLY:-c1,c2,c3,c4,c5s8} 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$label', d['config'], round(d['ms_per_step'],3), 'diag', round(d['diag_ms_profiled_step'],3), 'gemm', round(d['gemm_ms_profiled_step'],3))
" >> $OUT
  env "$@" timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('$label', 'c5', d.get('ms_per_step'))
" >> $OUT
}
for v in ${VARIANTS:-new old new_nola}; do
  case $v in
    new) run new X=1;;
    old) run old MSTRSM_DIAG_OLD=1;;
    new_nola) run new_nola MSTRSM_LOOKAHEAD=0;;
  esac
done
cat $OUT
