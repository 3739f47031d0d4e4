#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/exp_diagg.txt
for impl in w g; do
  MSTRSM_DIAG=$impl timeout 300 python tools/bench_rows.py --only c3,c5s8 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$impl', d['config'], round(d['ms_per_step'],3), 'diag', round(d['diag_ms_profiled_step'],3))
" >> gpurun_out/exp_diagg.txt
  MSTRSM_DIAG=$impl timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('$impl c5', round(d['ms_per_step'],3), 'diag', round(d['roofline']['diag_ms_per_step'],3))
" >> gpurun_out/exp_diagg.txt
done
MSTRSM_DIAG=g timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fallback.py -m gpu -q -x 2>&1 | tail -2 >> gpurun_out/exp_diagg.txt
cat gpurun_out/exp_diagg.txt
