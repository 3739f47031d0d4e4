#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/exp_la.txt
for cfg in "MSTRSM_LOOKAHEAD=0" "MSTRSM_LA_COLS=48" "MSTRSM_LA_COLS=30" "MSTRSM_LA_COLS=24"; do
  env $cfg timeout 600 python tools/bench_rows.py --only c3,c5s8,f4 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$cfg', d['config'], round(d['ms_per_step'],3), 'diag', round(d.get('diag_ms_profiled_step',0),3), 'gemm', round(d.get('gemm_ms_profiled_step',0),3))
" >> gpurun_out/exp_la.txt
  env $cfg timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    r=d['roofline']; print('$cfg c5', round(d['ms_per_step'],3), 'diag', round(r.get('diag_ms_per_step',0),3), 'gemm', round(r.get('gemm_ms_per_step',0),3))
" >> gpurun_out/exp_la.txt
done
cat gpurun_out/exp_la.txt
