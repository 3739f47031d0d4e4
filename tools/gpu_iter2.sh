#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_it2.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_it2.log; tail -2 gpurun_out/pytest_it2.log
for P in 8 2; do for k in 0 4 8 16; do
  MSTRSM_DIST_RESERVE_SMS=$k timeout 600 python tools/exp_dist_emul.py $P 2>/dev/null | grep -E 'emulated' | python -c "
import sys,json
for l in sys.stdin: print('P=$P k=$k', round(json.loads(l)['ms_min'],2))"
done; done
for v in A B; do
  if [ $v = A ]; then export MSTRSM_LIB=$PWD/exp/lib_base.so; else unset MSTRSM_LIB; fi
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('$v c5', round(d['ms_per_step'],3))"
done
