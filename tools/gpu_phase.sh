#!/bin/bash
mkdir -p gpurun_out
for c in c5s8 c2 c4 c5; do
  MSTRSM_LIB=$PWD/exp/phase/libmstrsm.so timeout 300 python tools/exp_phase.py $c > gpurun_out/phase_$c.txt 2>&1; echo "$c $?"
done
