// gemm_launch.cu -- launcher + instantiations of the DMMA update GEMM (a.5).
//   default: the persistent warp-specialised kernel -- complex operands with three real products
//   (gemm_ws3m.cuh), real operands gemm_ws.cuh;
//   MSTRSM_GEMM=4m: complex with four real products (gemm_ws.cuh);
//   MSTRSM_GEMM=classic: the one-tile-per-CTA kernel (gemm_kernel.cuh).  (Comparison only.)
#include <stdlib.h>
#include <string.h>

#include "gemm_ws3m.cuh"
#include "runtime.cuh"

namespace mstrsm {
namespace rt {
// 0 = ws (complex: 3M), 1 = classic, 2 = ws with four products for complex
int gemm_variant() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("MSTRSM_GEMM");
        v = (e && !strcmp(e, "classic")) ? 1 : (e && !strcmp(e, "4m")) ? 2 : 0;
    }
    return v;
}
static bool use_classic() { return gemm_variant() == 1; }

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
    if constexpr (S<T>::cplx_) {
        if (gemm_variant() == 0) {
            auto kern = gemm_ws3m_kernel<OPC>;
            static bool attr3 = false;
            if (!attr3) {
                CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, k3mSmemBytes));
                attr3 = true;
            }
            const int64_t tm = cdiv(g.M, k3mBM), tn = cdiv(g.N, k3mBN), nt = tm * tn;
            const int grid = int(std::min<int64_t>(nt, g_num_sms));
            ProfScope ps(PK_GEMM, flops);
            kern<<<grid, kWsThreads, k3mSmemBytes, g_stream>>>(g, int(tm), int(nt));
            CK_LAUNCH("gemm_ws3m_kernel");
            return 0;
        }
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
