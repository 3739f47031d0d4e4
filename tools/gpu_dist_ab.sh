#!/bin/bash
# A/B of the one-GPU dist emulation: exp/lib_r02h.so (A) vs the in-tree library (B), interleaved
mkdir -p gpurun_out
for v in A B A B; do
  if [ $v = A ]; then export MSTRSM_LIB=$PWD/exp/lib_r02h.so; else unset MSTRSM_LIB; fi
  timeout 600 python tools/exp_dist_emul.py 8 2>/dev/null | grep -v NCCL | sed "s/^/$v /" | tee -a gpurun_out/dist_ab.txt
done
