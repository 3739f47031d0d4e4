#!/bin/bash
# The device-checked library (tools/build_checks.sh) on the sanitizer workload with each diagonal
# kernel, then the GPU parity tests against it.  (compute-sanitizer is closed on the GPU pool.)
TAG=${1:-r02}
mkdir -p gpurun_out
OUT=gpurun_out/device_checks_$TAG.log
: > $OUT
for impl in default w tc; do
  env MSTRSM_LIB=exp/checks/libmstrsm.so MSTRSM_DIAG=$impl timeout 600 python tools/sanitize_run.py >> $OUT 2>&1
  echo "sanitize_run MSTRSM_DIAG=$impl exit $?" >> $OUT
done
MSTRSM_LIB=exp/checks/libmstrsm.so timeout 1200 python -m pytest -m gpu -q --timeout 600 \
    tests/test_gpu_parity.py tests/test_gpu_fallback.py tests/test_gpu_threads.py tests/test_gpu_side.py \
    tests/test_gpu_spectral.py tests/test_gpu_dist.py >> $OUT 2>&1
echo "pytest (checked library) exit $?" >> $OUT
grep -c "device check failed" $OUT
tail -8 $OUT
