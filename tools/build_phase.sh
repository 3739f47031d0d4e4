#!/bin/bash
# libmstrsm with the phase timing of the diagonal kernels (MSTRSM_PHASE_TIMES) into
# exp/phase/libmstrsm.so; run a workload against it with MSTRSM_LIB=exp/phase/libmstrsm.so.
set -e
cd "$(dirname "$0")/.."
N=$(python -c "import nvidia.nccl as n; print(list(n.__path__)[0])")
mkdir -p exp/phase
for u in mstrsm runtime gemm_launch diag_dN_plain diag_dN_safe diag_dC_plain diag_dC_safe diag_zN_plain diag_zN_safe \
         diag_zC_plain diag_zC_safe diag_dG_plain diag_dG_safe diag_zG_plain diag_zG_safe; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr \
       -DMSTRSM_PHASE_TIMES -I$N/include -c -o exp/phase/$u.o paper_1607_01477_b200/csrc/$u.cu &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o exp/phase/libmstrsm.so exp/phase/*.o -L$N/lib -l:libnccl.so.2 -Xlinker -rpath=$N/lib
echo built exp/phase/libmstrsm.so
