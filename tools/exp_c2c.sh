#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/exp_c2c.txt
for la in 1 0; do
  MSTRSM_LOOKAHEAD=$la timeout 300 python tools/bench_rows.py --only c1,c2,trsm 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('la$la', d['config'], round(d['ms_per_step'],3))
" >> gpurun_out/exp_c2c.txt
done
cat gpurun_out/exp_c2c.txt
