#!/bin/bash
# ABI changes (device row_end, synchronous status) on the GPU, then an ncu capture of c4's diagw.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_abi.py tests/test_gpu_gen.py -q -k "row_end or nonfinite or abi or sync" > gpurun_out/pytest_abi.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_abi.log
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:diagw -s 6 -c 1 \
    -o gpurun_out/prof_diagw_c4 python tools/profile_run.py --config c4 --iters 1 > gpurun_out/ncu_diagw_c4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/launches_c4.csv python tools/profile_run.py --config c4 --iters 1 > gpurun_out/ncu_list_c4.log 2>&1
tail -3 gpurun_out/pytest_abi.log
