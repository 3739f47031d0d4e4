#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/exp_c5lpc.txt
for l in 0 16 32; do
  MSTRSM_DIAG_LPC=$l timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('lpc$l c5', round(d['ms_per_step'],3), 'diag', round(d['roofline']['diag_ms_per_step'],3))
" >> gpurun_out/exp_c5lpc.txt
  MSTRSM_DIAG_LPC=$l timeout 300 python tools/bench_rows.py --only c5s8 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('lpc$l', d['config'], round(d['ms_per_step'],3), 'diag', round(d['diag_ms_profiled_step'],3))
" >> gpurun_out/exp_c5lpc.txt
done
cat gpurun_out/exp_c5lpc.txt
