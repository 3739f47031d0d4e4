#!/bin/bash
# Experiment: chunked diag kernel vs round-1 kernel vs the chunked loop without the replay
# (timing only), with and without the look-ahead.
TAG=${1:-e1}
mkdir -p gpurun_out
OUT=gpurun_out/exp_$TAG.txt
: > $OUT
run() {  # label, env...
  label=$1; shift
  env "$@" timeout 300 python tools/bench_rows.py --only c2,c3,c4,c5s8 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$label', d['config'], round(d['ms_per_step'],3), 'diag', round(d['diag_ms_profiled_step'],3), 'gemm', round(d['gemm_ms_profiled_step'],3))
" >> $OUT
  env "$@" timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('$label', 'c5', d.get('ms_per_step'), 'diag', d.get('diag_ms_per_step', d.get('breakdown')))
" >> $OUT
}
run new X=1
run old MSTRSM_DIAG_OLD=1
run noreplay MSTRSM_LIB=exp/noreplay/libmstrsm.so
run new_nola MSTRSM_LOOKAHEAD=0
run old_nola MSTRSM_DIAG_OLD=1 MSTRSM_LOOKAHEAD=0
run noreplay_nola MSTRSM_LIB=exp/noreplay/libmstrsm.so MSTRSM_LOOKAHEAD=0
cat $OUT
