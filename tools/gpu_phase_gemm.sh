#!/bin/bash
mkdir -p gpurun_out
for c in c5s8 c5 c4; do
  MSTRSM_LIB=$PWD/exp/phase/libmstrsm.so timeout 300 python tools/exp_phase_gemm.py $c > gpurun_out/gphase_$c.txt 2>&1; echo "$c $?"
done
