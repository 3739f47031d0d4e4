#!/bin/bash
# early-A: off / by size / always, interleaved, c4 c5s8 c5
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gemm_variants.py -m gpu -q -x > gpurun_out/pytest_early2.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_early2.log; tail -2 gpurun_out/pytest_early2.log
for rep in 1 2; do for v in 0 size 1; do
  if [ $v = size ]; then unset MSTRSM_EARLY_A; else export MSTRSM_EARLY_A=$v; fi
  timeout 600 python tools/bench_rows.py --only c4,c5s8 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['config'], round(d['ms_per_step'],3))"
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('$v c5', round(d['ms_per_step'],3))"
done; done
