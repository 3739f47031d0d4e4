#!/bin/bash
# Full ncu capture (with source) of one diag_kernel launch on c5 m=4096.
mkdir -p gpurun_out
python tools/profile_run.py --config c5 --m 4096 > gpurun_out/plain_diag.log 2>&1 || { cat gpurun_out/plain_diag.log; exit 1; }
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:diag_kernel -s 20 -c 1 \
    -o gpurun_out/prof_diag_v3 python tools/profile_run.py --config c5 --m 4096 > gpurun_out/ncu_diag_v3.log 2>&1
tail -3 gpurun_out/ncu_diag_v3.log
