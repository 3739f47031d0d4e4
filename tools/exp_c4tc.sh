#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/exp_c4tc.txt
for impl in w tc; do
  MSTRSM_DIAG=$impl timeout 300 python tools/bench_rows.py --only c1,c2,c4 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$impl', d['config'], round(d['ms_per_step'],3), 'diag', round(d['diag_ms_profiled_step'],3))
" >> gpurun_out/exp_c4tc.txt
done
MSTRSM_DIAG=tc timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fallback.py -m gpu -q -x 2>&1 | tail -2 >> gpurun_out/exp_c4tc.txt
cat gpurun_out/exp_c4tc.txt
