#!/bin/bash
# Re-check of the committed HEAD (after tools/gpu_final.sh's tests/bench were run separately): every row,
# the 8-rank emulation, the ncu launch list of the bench command, ncu --set full of the three hot kernels.
# Usage: bash tools/gpu_final_head.sh <tag>
TAG=${1:-r02m}
mkdir -p gpurun_out
timeout 600 python tools/bench_rows.py > gpurun_out/rows_$TAG.jsonl 2> gpurun_out/rows_$TAG.err
timeout 600 python tools/exp_dist_emul.py 8 > gpurun_out/dist_emul_$TAG.jsonl 2> gpurun_out/dist_emul_$TAG.err
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
for r in gemm diag diagl; do
  f=$(ls gpurun_out/prof_${r}_*_$TAG.ncu-rep 2>/dev/null | head -1)
  [ -n "$f" ] || continue
  b=${f%.ncu-rep}
  ncu -i $f --page details > ${b}_details.txt 2>&1
  ncu -i $f --page raw --csv > ${b}_raw.csv 2>&1
  mv $f /tmp/
done
tail -2 gpurun_out/ncu_list_$TAG.log; wc -l gpurun_out/rows_$TAG.jsonl gpurun_out/dist_emul_$TAG.jsonl
