#!/bin/bash
# ncu --set full with source for the diagonal kernels of c4 (diagw 8,8), c2 (diagl), c5s8 (diagw 32,4)
# and a c5s8 GEMM; exports details + source pages (csv) and removes the reports (size cap).
mkdir -p gpurun_out
run() {  # name regex skip config
  timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:$2 -s $3 -c 1 \
    -o /tmp/$1 python tools/profile_run.py --config $4 $5 > gpurun_out/$1.log 2>&1; echo "$1 $?"
  ncu -i /tmp/$1.ncu-rep --page details > gpurun_out/$1_details.txt 2>&1
  ncu -i /tmp/$1.ncu-rep --page source --csv --print-source sass > gpurun_out/$1_sass.csv 2>&1
  ncu -i /tmp/$1.ncu-rep --page source --csv --print-source cuda > gpurun_out/$1_cuda.csv 2>&1
  gzip -f gpurun_out/$1_sass.csv
}
run src_diagw_c4 diagw 40 c4 "--iters 3"
run src_diagl_c2 diagl 16 c2
run src_diagw_c5s8 diagw 64 c5s8
run src_gemm_c5s8 gemm_ws3q 64 c5s8
ls -la gpurun_out
