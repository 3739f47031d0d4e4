#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/exp_c4g.txt
for g in 2 3; do
  MSTRSM_3M_GROUPS=$g timeout 300 python tools/bench_rows.py --only c4 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('groups$g', d['config'], round(d['ms_per_step'],3), 'gemm', round(d['gemm_ms_profiled_step'],3))
" >> gpurun_out/exp_c4g.txt
done
for ph in 0 1 3; do
  MSTRSM_3P_PHASE=$ph timeout 300 python tools/bench_rows.py --only c4 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('phase$ph', d['config'], round(d['ms_per_step'],3), 'gemm', round(d['gemm_ms_profiled_step'],3))
" >> gpurun_out/exp_c4g.txt
done
cat gpurun_out/exp_c4g.txt
