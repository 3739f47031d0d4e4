// gemm_launch.cu -- launcher + instantiations of the DMMA update GEMM (a.5).
//   default: the persistent warp-specialised kernel -- complex operands with three real products
//   (gemm_ws3m.cuh), real operands gemm_ws.cuh;
//   MSTRSM_GEMM=4m: complex with four real products (gemm_ws.cuh);
//   MSTRSM_GEMM=classic: the one-tile-per-CTA kernel (gemm_kernel.cuh) for everything (comparison);
//   real launches of at most one wave take it by default (gemm_real_mode below).
#include <stdlib.h>
#include <string.h>

#include <cudaTypedefs.h>   // PFN_cuTensorMapEncodeTiled (driver entry point, no -lcuda)

#include "gemm_ws3q.cuh"
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
// MSTRSM_3M_PRESUM=0: keep the in-register operand sums (comparison only)
bool gemm_presum_enabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("MSTRSM_3M_PRESUM");
        v = (e && !strcmp(e, "0")) ? 0 : 1;
    }
    return v == 1;
}
// cuTensorMapEncodeTiled through the runtime's driver entry point
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}
// 2-D map over a column-major (rows x cols) f64 array with leading dimension ld (elements)
static bool encode_2d(CUtensorMap *tm, const void *base, uint64_t rows, uint64_t cols, uint64_t ld,
                      uint32_t box_rows, uint32_t box_cols, CUtensorMapSwizzle sw) {
    auto enc = tensor_map_encoder();
    if (!enc) return false;
    cuuint64_t dims[2] = {rows, cols}, strides[1] = {ld * 8};
    cuuint32_t box[2] = {box_rows, box_cols}, es[2] = {1, 1};
    return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void *>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// The 3-product kernel's second consumer group starts MSTRSM_3P_PHASE/4 of a tile late (default
// 2: half a tile), so the two groups' epilogues do not coincide (0: both start together)
static int gemm_3p_phase() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("MSTRSM_3P_PHASE");
        v = (e && e[0] >= '0' && e[0] <= '3' && !e[1]) ? e[0] - '0' : 2;
    }
    return v;
}

// Three consumer warpgroups (gemm_ws3q.cuh) or two (gemm_ws3p.cuh).  Three win at the blocked
// solve's K = n_b = 128 (the epilogues of two groups overlap the third's mainloop), two at K = 64
// (c4, the generalized solve: per-tile overheads of the smaller 32-row tiles) and at large K (the
// back-transformation: the 48-row tile re-reads X less); DESIGN.md §7.2.
// MSTRSM_3M_GROUPS=2|3 forces one.
// A short update (M <= 64 rows: the next block's rows in the paired-block solve) takes the three
// groups' 32-row tiles whatever K: 48-row tiles would pad M = 64 to 96.
static int gemm_3m_groups(int K, int64_t M) {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("MSTRSM_3M_GROUPS");
        v = (e && !strcmp(e, "2")) ? 2 : (e && !strcmp(e, "3")) ? 3 : 0;
    }
    if (v) return v;
    return ((K >= 96 && K <= 256) || M <= 64) ? 3 : 2;
}

static bool use_classic() { return gemm_variant() == 1; }
// Real operands: MSTRSM_GEMM_REAL=ws|classic forces the persistent warp-specialised kernel / the
// one-tile-per-CTA kernel; default (auto): the one-tile-per-CTA kernel when the launch is at most
// one wave of it (2 CTAs per SM) and no SM cap is in force -- the short updates of small real
// solves (c1, c2), where the persistent kernel's producer/consumer hand-off is pure latency.
static int gemm_real_mode() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("MSTRSM_GEMM_REAL");
        v = (e && !strcmp(e, "ws")) ? 1 : (e && !strcmp(e, "classic")) ? 2 : 0;
    }
    return v;
}
// MSTRSM_EARLY_A=0|1 forces the early U-operand issue of gemm_ws3q_kernel / gemm_ws_kernel off / on
// (default: by size)
static int gemm_early_a() {
    static int v = -2;
    if (v == -2) {
        const char *e = getenv("MSTRSM_EARLY_A");
        v = (e && (e[0] == '0' || e[0] == '1') && !e[1]) ? e[0] - '0' : -1;
    }
    return v;
}

// MSTRSM_GEMM_TRIGGER=0|1: the one-tile-per-CTA kernel lets the next grid (the next diagonal step,
// which stages its read-only triangle before its wait) launch at its start never / always.
// Default: for launches of at most g_num_sms / 4 tiles, which leave the next step's CTAs SMs of
// their own (c1 0.186 -> 0.175 ms, real trsm 256 0.124 -> 0.113 with it; c2, whose updates cover
// the GPU, 1.108 -> 1.154 with it everywhere: profiles/r02/exp_small_gemm_s3.txt).
static int gemm_classic_trigger(int64_t tiles) {
    static const int v = [] {
        const char *e = getenv("MSTRSM_GEMM_TRIGGER");
        return (e && (e[0] == '0' || e[0] == '1') && !e[1]) ? e[0] - '0' : -1;
    }();
    return v >= 0 ? v : (tiles <= g_num_sms / 4 ? 1 : 0);
}

template <typename T, bool OPC>
int launch_gemm(const GemmArgs<T> &g) {
    const double flops = double(g.M) * g.N * g.K * (S<T>::cplx_ ? 8.0 : 2.0);
    const int64_t tiles_m = cdiv(g.M, GemmCfg<T>::BM), tiles_n = cdiv(g.N, GemmCfg<T>::BN);
    const bool real_classic = !S<T>::cplx_ && gemm_variant() == 0 &&
                              (gemm_real_mode() == 2 ||
                               (gemm_real_mode() == 0 && g_cta_cap == 0 && tiles_m * tiles_n <= 2 * int64_t(g_num_sms)));
    if (use_classic() || real_classic) {
        auto kern = gemm_update_kernel<T, OPC>;
        static std::atomic<uint64_t> attr_set{0};
        constexpr int smem = gemm_smem_bytes<T>();
        if (first_on_device(attr_set)) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        dim3 grid{unsigned(tiles_m), unsigned(tiles_n), 1u};
        GemmArgs<T> ga = g;
        ga.early_a = gemm_early_a() == 1 ? 1 : 0;   // (measured no gain here: exp_small_gemm_s3.txt)
        ga.trig = gemm_classic_trigger(tiles_m * tiles_n);
        ProfScope ps(PK_GEMM, flops);
        CK(launch_k(kern, grid, dim3(kGemmThreads), smem, g_stream, ga));
        CK_LAUNCH("gemm_update_kernel");
        return 0;
    }
    if constexpr (S<T>::cplx_) {
        if (gemm_variant() == 0 && g.As && g.Xsum && g.a_r0 % 2 == 0 && g.ldas % 2 == 0 &&
            g.ldxs % 2 == 0) {                   // sums precomputed: copy-engine producer, LDS + DMMA
            // X: rows x_r0.. (as 2K doubles) x columns col0.., X+: K x N doubles; op C: A = rows a_r0..
            // (2K doubles) x columns a_c0.. (M) of U, A+ likewise in the plane
            CUtensorMap tmX, tmXs, tmA, tmAs;
            if (!encode_2d(&tmX, g.X + g.x_r0 + g.col0 * g.ldx, uint64_t(2 * g.K), uint64_t(g.N), uint64_t(2 * g.ldx),
                           2 * k3mBK, k3mBN, CU_TENSOR_MAP_SWIZZLE_128B) ||
                !encode_2d(&tmXs, g.Xsum + g.col0 * g.ldxs, uint64_t(g.K), uint64_t(g.N), uint64_t(g.ldxs), k3mBK,
                           k3mBN, CU_TENSOR_MAP_SWIZZLE_64B))
                return set_cuda_error(cudaErrorInvalidValue, "cuTensorMapEncodeTiled (3M update operands)");
            const bool q3 = gemm_3m_groups(g.K, g.M) == 3;
            const uint32_t bm = q3 ? k3qBM : k3mBM;
            if (OPC) {
                if (!encode_2d(&tmA, g.U + g.a_r0 + g.a_c0 * g.ldu, uint64_t(2 * g.K), uint64_t(g.M),
                               uint64_t(2 * g.ldu), 2 * k3mBK, bm, CU_TENSOR_MAP_SWIZZLE_128B) ||
                    !encode_2d(&tmAs, g.As + g.a_r0 + g.a_c0 * g.ldas, uint64_t(g.K), uint64_t(g.M), uint64_t(g.ldas),
                               k3mBK, bm, CU_TENSOR_MAP_SWIZZLE_64B))
                    return set_cuda_error(cudaErrorInvalidValue, "cuTensorMapEncodeTiled (3M op C operands)");
            } else {
                tmA = tmX;
                tmAs = tmXs;
            }
            if (q3) {
                auto kq = gemm_ws3q_kernel<OPC>;
                static std::atomic<uint64_t> attrq{0};
                if (first_on_device(attrq)) CK(cudaFuncSetAttribute(kq, cudaFuncAttributeMaxDynamicSharedMemorySize, k3qSmemBytes));
                const int64_t tm = cdiv(g.M, k3qBM), tn = cdiv(g.N, k3qBN), nt = tm * tn;
                const int grid = int(std::min<int64_t>(nt, g_cta_cap > 0 ? g_cta_cap : g_num_sms));
                ProfScope ps(PK_GEMM, flops);
#ifdef MSTRSM_PHASE_TIMES
                const_cast<GemmArgs<T> &>(g).pt = phase_next(1);
#endif
                // (pipeline fill issued before the dependent-launch wait on short launches: <= 4 tiles
                // per consumer group)
                const int early_a = gemm_early_a() >= 0 ? gemm_early_a() : (nt <= int64_t(grid) * 3 * 4 ? 1 : 0);
                CK(launch_k(kq, dim3(grid), dim3(k3qThreads), k3qSmemBytes, g_stream, g, int(tm), int(nt), tmX, tmXs, tmA,
                            tmAs, gemm_3p_phase(), early_a));
                CK_LAUNCH("gemm_ws3q_kernel");
                return 0;
            }
            auto kern = gemm_ws3p_kernel<OPC>;
            static std::atomic<uint64_t> attrp{0};
            if (first_on_device(attrp)) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, k3pSmemBytes));
            const int64_t tm = cdiv(g.M, k3mBM), tn = cdiv(g.N, k3mBN), nt = tm * tn;
            const int grid = int(std::min<int64_t>(nt, g_cta_cap > 0 ? g_cta_cap : g_num_sms));
            ProfScope ps(PK_GEMM, flops);
            CK(launch_k(kern, dim3(grid), dim3(kWsThreads), k3pSmemBytes, g_stream, g, int(tm), int(nt), tmX, tmXs,
                            tmA, tmAs, gemm_3p_phase()));
            CK_LAUNCH("gemm_ws3p_kernel");
            return 0;
        }
        if (gemm_variant() == 0) {
            auto kern = gemm_ws3m_kernel<OPC>;
            static std::atomic<uint64_t> attr3{0};
            if (first_on_device(attr3)) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, k3mSmemBytes));
            const int64_t tm = cdiv(g.M, k3mBM), tn = cdiv(g.N, k3mBN), nt = tm * tn;
            const int grid = int(std::min<int64_t>(nt, g_cta_cap > 0 ? g_cta_cap : g_num_sms));
            ProfScope ps(PK_GEMM, flops);
            kern<<<grid, kWsThreads, k3mSmemBytes, g_stream>>>(g, int(tm), int(nt));
            CK_LAUNCH("gemm_ws3m_kernel");
            return 0;
        }
    }
    auto kern = gemm_ws_kernel<T, OPC>;
    static std::atomic<uint64_t> attr_set{0};
    constexpr int smem = gemm_ws_smem_bytes<T>();
    if (first_on_device(attr_set)) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int64_t ntiles = tiles_m * tiles_n;
    const int grid = int(std::min<int64_t>(ntiles, g_cta_cap > 0 ? g_cta_cap : g_num_sms));
    ProfScope ps(PK_GEMM, flops);
    // (first tile's A k-tiles issued before the dependent-launch wait on short launches: <= 4
    // tiles per consumer group, as for gemm_ws3q_kernel)
    const int early_a = gemm_early_a() >= 0 ? gemm_early_a() : (ntiles <= int64_t(grid) * 2 * 4 ? 1 : 0);
    CK(launch_k(kern, dim3(grid), dim3(kWsThreads), smem, g_stream, g, int(tiles_m), int(ntiles), early_a));
    CK_LAUNCH("gemm_ws_kernel");
    return 0;
}

template int launch_gemm<double, false>(const GemmArgs<double> &);
template int launch_gemm<double, true>(const GemmArgs<double> &);
template int launch_gemm<cplx, false>(const GemmArgs<cplx> &);
template int launch_gemm<cplx, true>(const GemmArgs<cplx> &);
}  // namespace rt
}  // namespace mstrsm
