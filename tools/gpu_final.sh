#!/bin/bash
# Round-2 final evidence: parity tests (+ Delta-e log), smoke, bench (default flags), reference arm,
# rows, launch list of the bench command, ncu of the GEMM and both diagonal kernels, dist emulation.
TAG=${1:-r02f}
mkdir -p gpurun_out
export MSTRSM_PARITY_LOG=gpurun_out/parity_$TAG.jsonl
: > $MSTRSM_PARITY_LOG
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
unset MSTRSM_PARITY_LOG
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke_$TAG.log
nvidia-smi > gpurun_out/nvidia_smi_$TAG.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.log 2>&1
echo "bench exit $?" >> gpurun_out/bench_$TAG.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$TAG.log 2>&1
echo "ref exit $?" >> gpurun_out/bench_ref_$TAG.log
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
# summaries on the box (the reports themselves stay out of gpurun_out: size cap)
for r in gemm diag diagl; do
  f=$(ls gpurun_out/prof_${r}_*_$TAG.ncu-rep 2>/dev/null | head -1)
  [ -n "$f" ] || continue
  b=${f%.ncu-rep}
  ncu -i $f --page details > ${b}_details.txt 2>&1
  ncu -i $f --page raw --csv > ${b}_raw.csv 2>&1
  mv $f /tmp/
done
if [ -z "$SKIP_PHASE" ]; then
  bash tools/gpu_phase.sh > /dev/null 2>&1
  bash tools/gpu_phase_gemm.sh > /dev/null 2>&1
fi
tail -3 gpurun_out/pytest_gpu_$TAG.log; tail -2 gpurun_out/smoke_$TAG.log
timeout 900 bash tools/gpu_emul_prof.sh > /dev/null 2>&1; cp gpurun_out/launch_emul_r02.csv gpurun_out/launch_emul_$TAG.csv 2>/dev/null
