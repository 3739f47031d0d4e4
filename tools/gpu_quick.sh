#!/bin/bash
# Quick GPU check: parity tests, then per-row timings of the new diagonal kernel vs the round-1
# one (MSTRSM_DIAG_OLD=1).  Usage (via gpurun): bash tools/gpu_quick.sh <tag> [pytest-args]
TAG=${1:-q}
shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 "$@" > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
tail -3 gpurun_out/pytest_gpu_$TAG.log
ONLY=${ONLY:-c1,c2,c3,c4,c5s8,trsm}
timeout 600 python tools/bench_rows.py --only $ONLY > gpurun_out/rows_new_$TAG.jsonl 2> gpurun_out/rows_new_$TAG.err
MSTRSM_DIAG_OLD=1 timeout 600 python tools/bench_rows.py --only $ONLY > gpurun_out/rows_old_$TAG.jsonl 2> gpurun_out/rows_old_$TAG.err
python - <<'PY'
import json,sys
tag=sys.argv[1] if len(sys.argv)>1 else ""
PY
python -c "
import json
for f in ['new','old']:
    for l in open('gpurun_out/rows_%s_$TAG.jsonl'%f):
        d=json.loads(l); print(f, d['config'], round(d['ms_per_step'],3), 'diag', round(d['diag_ms_profiled_step'],3), 'gemm', round(d['gemm_ms_profiled_step'],3))
"
