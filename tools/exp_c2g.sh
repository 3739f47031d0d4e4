#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/exp_c2g.txt
for g in ws classic; do
  MSTRSM_GEMM=$g timeout 300 python tools/bench_rows.py --only c1,c2,trsm 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$g', d['config'], round(d['ms_per_step'],3), 'gemm', round(d['gemm_ms_profiled_step'],3))
" >> gpurun_out/exp_c2g.txt
done
cat gpurun_out/exp_c2g.txt
