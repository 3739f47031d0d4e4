#!/bin/bash
# One GPU call: parity tests, bench, ncu launch list of the bench command, full captures of
# the update GEMM and the diag kernel.  Usage (via gpurun): bash tools/gpu_round.sh <tag>
TAG=${1:-r01}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia_smi_$TAG.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_$TAG.log 2>&1
echo "bench exit $?" >> gpurun_out/bench_$TAG.log
if [ "${SKIP_NCU:-0}" = "0" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_bench_$TAG.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
    > gpurun_out/ncu_list_$TAG.log 2>&1
echo "ncu list exit $?" >> gpurun_out/ncu_list_$TAG.log
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:gemm_ws -s 60 -c 1 \
    -o gpurun_out/prof_gemm_c5_$TAG python tools/profile_run.py --config c5 > gpurun_out/ncu_gemm_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:diag_kernel -s 120 -c 1 \
    -o gpurun_out/prof_diag_c5_$TAG python tools/profile_run.py --config c5 > gpurun_out/ncu_diag_$TAG.log 2>&1
fi
ls -la gpurun_out
