#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/dbg_pair.txt
for cfg in "MSTRSM_PAIR=1" "MSTRSM_PAIR=1 MSTRSM_DIAG=tc"; do
  echo "== $cfg" >> gpurun_out/dbg_pair.txt
  env $cfg timeout 300 python tools/dbg_pair.py >> gpurun_out/dbg_pair.txt 2>&1
done
cat gpurun_out/dbg_pair.txt
