#!/bin/bash
# One iteration: full GPU tests, the rows, the c5 bench (device only).  $1 = tag
TAG=${1:-it}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_$TAG.log
timeout 600 python tools/bench_rows.py --only c1,c2,c3,c4,c4d,g1,f4,c5s8 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$TAG', d['config'], round(d['ms_per_step'],3), 'diag', round(d.get('diag_ms_profiled_step',0),3), 'gemm', round(d.get('gemm_ms_profiled_step',0),3))
" > gpurun_out/rows_$TAG.txt
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    r=d['roofline']; print('$TAG c5', round(d['ms_per_step'],3), 'diag', round(r.get('diag_ms_per_step',0),3), 'gemm', round(r.get('gemm_ms_per_step',0),3), 'frac', round(r['frac'],4))
" >> gpurun_out/rows_$TAG.txt
tail -2 gpurun_out/pytest_$TAG.log
cat gpurun_out/rows_$TAG.txt
