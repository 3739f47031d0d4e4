#!/bin/bash
# Look-ahead on the real small solves (c1, c2): off vs on with the diagl columns-per-CTA model.
mkdir -p gpurun_out
OUT=gpurun_out/exp_la_real.txt
: > $OUT
for rep in 1 2; do
for cfg in "MSTRSM_LOOKAHEAD=0" "MSTRSM_LOOKAHEAD=1 MSTRSM_LA_COLS=64" "MSTRSM_LOOKAHEAD=1 MSTRSM_LA_COLS=32" "MSTRSM_LOOKAHEAD=1 MSTRSM_LA_COLS=128"; do
  env $cfg timeout 300 python tools/bench_rows.py --only ${ROWS:-c1,c2,c3} 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$cfg', d['config'], round(d['ms_per_step'],4), 'diag', round(d.get('diag_ms_profiled_step',0),3), 'gemm', round(d.get('gemm_ms_profiled_step',0),3))
" >> $OUT
done
done
cat $OUT
