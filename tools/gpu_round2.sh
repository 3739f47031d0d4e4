#!/bin/bash
# Round-2 evidence in one GPU call: bench (default flags), reference arm, launch list of the bench
# command, full captures of the update GEMM and the diagonal kernel (c5), rows of the other configs.
TAG=${1:-r02}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia_smi_$TAG.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.log 2>&1
echo "bench exit $?" >> gpurun_out/bench_$TAG.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$TAG.log 2>&1
echo "ref exit $?" >> gpurun_out/bench_ref_$TAG.log
timeout 600 python tools/bench_rows.py > gpurun_out/rows_$TAG.jsonl 2> gpurun_out/rows_$TAG.err
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_bench_$TAG.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
    > gpurun_out/ncu_list_$TAG.log 2>&1
echo "ncu list exit $?" >> gpurun_out/ncu_list_$TAG.log
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:gemm_ws -s 60 -c 1 \
    -o gpurun_out/prof_gemm_c5_$TAG python tools/profile_run.py --config c5 > gpurun_out/ncu_gemm_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:diagw -s 70 -c 1 \
    -o gpurun_out/prof_diag_c5_$TAG python tools/profile_run.py --config c5 > gpurun_out/ncu_diag_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:diagl -s 16 -c 1 \
    -o gpurun_out/prof_diagl_c2_$TAG python tools/profile_run.py --config c2 > gpurun_out/ncu_diagl_$TAG.log 2>&1
ls gpurun_out | grep $TAG
tail -2 gpurun_out/bench_$TAG.log | cut -c1-600
