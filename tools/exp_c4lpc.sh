#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/exp_c4lpc.txt
for l in 4 8 16; do
  MSTRSM_DIAG_LPC=$l timeout 300 python tools/bench_rows.py --only c4 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('lpc$l', d['config'], round(d['ms_per_step'],3), 'diag', round(d['diag_ms_profiled_step'],3))
" >> gpurun_out/exp_c4lpc.txt
done
for l in 8 16 32; do
  MSTRSM_DIAG_LPC=$l timeout 300 python tools/bench_rows.py --only c3 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('lpc$l', d['config'], round(d['ms_per_step'],3), 'diag', round(d['diag_ms_profiled_step'],3))
" >> gpurun_out/exp_c4lpc.txt
done
cat gpurun_out/exp_c4lpc.txt
