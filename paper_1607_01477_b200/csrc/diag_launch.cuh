// diag_launch.cuh -- launcher of the diagonal-block kernel (a.3/a.4); included by the
// diag_{d,z}{N,C}.cu units, each of which instantiates one (scalar, op) pair.
#pragma once
#include "runtime.cuh"

namespace mstrsm {
namespace rt {
template <typename T, int LPC, bool SAFE, int OP>
int launch_diag_t(const DiagArgs<T> &a) {
    auto kern = diag_kernel<T, LPC, 16, SAFE, OP>;
    int nfull = int(a.hi - a.lo);
    size_t smem = size_t(diag_smem_bytes(nfull, sizeof(T)));
    static bool attr_set = false;
    if (!attr_set) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr_set = true;
    }
    // warps per CTA chosen so that the grid covers every SM when there are enough columns
    // (one CTA per SM when the staged block is large), at most 16 warps.
    const int G = 32 / LPC;
    int occ1 = occupancy(kern, 512, smem);                 // CTAs per SM at 512 threads
    int64_t groups = cdiv(a.ncols, G);
    int64_t wpc = cdiv(groups, int64_t(g_num_sms) * std::max(occ1, 1));
    wpc = std::max<int64_t>(1, std::min<int64_t>(16, wpc));
    int threads = int(wpc * 32);
    int occ = occupancy(kern, threads, smem);
    int grid = int(std::min<int64_t>(cdiv(groups, wpc), int64_t(occ) * g_num_sms));
    if (grid < 1) grid = 1;
    double fl = double(a.ncols) * nfull * (nfull - 1) / 2.0 * (S<T>::cplx_ ? 8.0 : 2.0);
    ProfScope ps(PK_DIAG, fl);
    kern<<<grid, threads, smem, g_stream>>>(a);
    CK_LAUNCH("diag_kernel");
    return 0;
}

template <typename T, bool SAFE, int OP>
int launch_diag(const DiagArgs<T> &a, int nb) {
    if (nb <= 16) return launch_diag_t<T, 1, SAFE, OP>(a);
    if (nb <= 32) return launch_diag_t<T, 2, SAFE, OP>(a);
    if (nb <= 64) return launch_diag_t<T, 4, SAFE, OP>(a);
    return launch_diag_t<T, 8, SAFE, OP>(a);
}

}  // namespace rt
}  // namespace mstrsm
