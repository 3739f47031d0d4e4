// gemm_launch.cu -- launcher + instantiations of the DMMA update GEMM (a.5).
//   default: the persistent warp-specialised kernel (gemm_ws.cuh);
//   MSTRSM_GEMM=classic selects the one-tile-per-CTA kernel (gemm_kernel.cuh) for comparison.
#include <stdlib.h>
#include <string.h>

#include "gemm_ws.cuh"
#include "runtime.cuh"

namespace mstrsm {
namespace rt {
static bool use_classic() {
    static int v = -1;
    if (v < 0) { const char *e = getenv("MSTRSM_GEMM"); v = (e && !strcmp(e, "classic")) ? 1 : 0; }
    return v == 1;
}

template <typename T, bool OPC>
int launch_gemm(const GemmArgs<T> &g) {
    const double flops = double(g.M) * g.N * g.K * (S<T>::cplx_ ? 8.0 : 2.0);
    const int64_t tiles_m = cdiv(g.M, GemmCfg<T>::BM), tiles_n = cdiv(g.N, GemmCfg<T>::BN);
    if (use_classic()) {
        auto kern = gemm_update_kernel<T, OPC>;
        static bool attr_set = false;
        constexpr int smem = gemm_smem_bytes<T>();
        if (!attr_set) {
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            attr_set = true;
        }
        dim3 grid{unsigned(tiles_m), unsigned(tiles_n), 1u};
        ProfScope ps(PK_GEMM, flops);
        kern<<<grid, kGemmThreads, smem, g_stream>>>(g);
        CK_LAUNCH("gemm_update_kernel");
        return 0;
    }
    auto kern = gemm_ws_kernel<T, OPC>;
    static bool attr_set = false;
    constexpr int smem = gemm_ws_smem_bytes<T>();
    if (!attr_set) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        attr_set = true;
    }
    const int64_t ntiles = tiles_m * tiles_n;
    const int grid = int(std::min<int64_t>(ntiles, g_num_sms));
    ProfScope ps(PK_GEMM, flops);
    kern<<<grid, kWsThreads, smem, g_stream>>>(g, int(tiles_m), int(ntiles));
    CK_LAUNCH("gemm_ws_kernel");
    return 0;
}

template int launch_gemm<double, false>(const GemmArgs<double> &);
template int launch_gemm<double, true>(const GemmArgs<double> &);
template int launch_gemm<cplx, false>(const GemmArgs<cplx> &);
template int launch_gemm<cplx, true>(const GemmArgs<cplx> &);
}  // namespace rt
}  // namespace mstrsm
