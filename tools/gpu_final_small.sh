#!/bin/bash
# Final state after the small-solve update changes: GPU tests, smoke, every row, ncu launch lists of
# one c2 and one c1 solve, ncu --set full of one c2 update launch.  Usage: bash tools/gpu_final_small.sh <tag>
TAG=${1:-r02l}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke_$TAG.log
timeout 600 python tools/bench_rows.py > gpurun_out/rows_$TAG.jsonl 2> gpurun_out/rows_$TAG.err
for c in c2 c1; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --profile-from-start off \
      --log-file gpurun_out/launches_${c}_$TAG.csv python tools/profile_run.py --config $c > gpurun_out/ncu_list_${c}_$TAG.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:gemm_update -s 12 -c 1 \
    -o gpurun_out/prof_gemmc_c2_$TAG python tools/profile_run.py --config c2 > gpurun_out/ncu_gemmc_$TAG.log 2>&1
f=gpurun_out/prof_gemmc_c2_$TAG.ncu-rep
if [ -f $f ]; then
  ncu -i $f --page details > gpurun_out/prof_gemmc_c2_${TAG}_details.txt 2>&1
  mv $f /tmp/
fi
tail -3 gpurun_out/pytest_gpu_$TAG.log; tail -2 gpurun_out/smoke_$TAG.log
