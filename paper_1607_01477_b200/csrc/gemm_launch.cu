// gemm_launch.cu -- launcher + instantiations of the DMMA update GEMM (a.5).
#include "runtime.cuh"

namespace mstrsm {
namespace rt {
template <typename T, bool OPC>
int launch_gemm(const GemmArgs<T> &g) {
    auto kern = gemm_update_kernel<T, OPC>;
    static bool attr_set = false;
    constexpr int smem = gemm_smem_bytes<T>();
    if (!attr_set) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        attr_set = true;
    }
    dim3 grid(unsigned(cdiv(g.M, GemmCfg<T>::BM)), unsigned(cdiv(g.N, GemmCfg<T>::BN)));
    ProfScope ps(PK_GEMM, double(g.M) * g.N * g.K * (S<T>::cplx_ ? 8.0 : 2.0));
    kern<<<grid, kGemmThreads, smem, g_stream>>>(g);
    CK_LAUNCH("gemm_update_kernel");
    return 0;
}


template int launch_gemm<double, false>(const GemmArgs<double> &);
template int launch_gemm<double, true>(const GemmArgs<double> &);
template int launch_gemm<cplx, false>(const GemmArgs<cplx> &);
template int launch_gemm<cplx, true>(const GemmArgs<cplx> &);
}  // namespace rt
}  // namespace mstrsm
