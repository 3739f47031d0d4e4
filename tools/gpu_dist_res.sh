#!/bin/bash
# dist emulation with k SMs reserved for the comm stream's work
mkdir -p gpurun_out
for k in ${KS:-16 24 32 48 16 24 32 48}; do
  MSTRSM_DIST_RESERVE_SMS=$k timeout 600 python tools/exp_dist_emul.py 8 2>/dev/null | grep emulated | sed "s/^/k=$k /" | tee -a gpurun_out/dist_res.txt
done
