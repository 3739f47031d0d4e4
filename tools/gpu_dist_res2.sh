#!/bin/bash
mkdir -p gpurun_out
for P in 2 4 8; do for k in 0 8 16; do
  MSTRSM_DIST_RESERVE_SMS=$k timeout 600 python tools/exp_dist_emul.py $P 2>/dev/null | grep -E 'emulated|alone' | sed "s/^/P=$P k=$k /"
done; done
