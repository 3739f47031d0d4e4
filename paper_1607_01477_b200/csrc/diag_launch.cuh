// diag_launch.cuh -- launcher of the diagonal-block kernel (a.3/a.4); included by the
// diag_{d,z}{N,C}_{plain,safe}.cu units, each of which instantiates one (scalar, op, variant).
#pragma once
#include <stdio.h>
#include <stdlib.h>

#include "runtime.cuh"
#include "diag_fast.cuh"
#include "diag_tc.cuh"

namespace mstrsm {
namespace rt {
// Pass costs of the RPL = 16 (which = 0) and RPL = 4 (which = 1) layouts in tenths of an RPL = 8
// pass (measured on the c5 launch list: 12 and 7); MSTRSM_DIAG_COST16 / MSTRSM_DIAG_COST4 override.
inline int diag_cost(int which) {
    static int v[2] = {-1, -1};
    if (v[which] < 0) {
        const char *e = getenv(which ? "MSTRSM_DIAG_COST4" : "MSTRSM_DIAG_COST16");
        const int d = which ? 7 : 12;
        v[which] = e ? atoi(e) : d;
        if (v[which] <= 0) v[which] = d;
    }
    return v[which];
}

inline bool diag_balance() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("MSTRSM_DIAG_BALANCE");   // 0: fill CTAs, short last pass
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}

template <typename T, int LPC, int RPL, bool SAFE, int OP, bool FB, bool GEN>
int launch_diag_k(const DiagArgs<T> &a, int64_t ncols_max) {
    auto kern = diag_kernel<T, LPC, RPL, SAFE, OP, FB, GEN>;
    constexpr int kMaxThreads = DiagThreads<T, RPL>::value;
    constexpr int G = 32 / LPC;
    const int nfull = int(a.hi - a.lo);
    static std::atomic<uint64_t> attr_set{0};
    if (first_on_device(attr_set)) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    // warps per CTA chosen so that the grid covers every SM when there are enough columns
    const size_t smem = size_t(diag_smem_bytes(nfull, sizeof(T), GEN));
    int occ1 = occupancy(kern, kMaxThreads, smem);
    int64_t groups = cdiv(ncols_max, G);
    const int64_t sms = g_cta_cap > 0 ? g_cta_cap : g_num_sms;
    int64_t wpc = cdiv(groups, sms * std::max(occ1, 1));
    wpc = std::max<int64_t>(1, std::min<int64_t>(kMaxThreads / 32, wpc));
    if (diag_balance()) {   // equal passes: as many warps per CTA as the pass count needs, no short last pass
        const int64_t npass = cdiv(groups, sms * std::max(occ1, 1) * (kMaxThreads / 32));
        wpc = std::max<int64_t>(1, std::min<int64_t>(kMaxThreads / 32, cdiv(groups, sms * std::max(occ1, 1) * npass)));
    }
    const int threads = int(wpc * 32);
    int occ = occupancy(kern, threads, smem);
    int grid = int(std::min<int64_t>(cdiv(groups, wpc), int64_t(occ) * sms));
    if (grid < 1) grid = 1;
    double fl = FB ? 0.0 : double(a.ncols) * nfull * (nfull - 1) / 2.0 * (S<T>::cplx_ ? 8.0 : 2.0);
    ProfScope ps(PK_DIAG, fl);
    CK(launch_k(kern, dim3(grid), dim3(threads), smem, g_stream, a));
    CK_LAUNCH("diag_kernel");
    return 0;
}

// Lane layout: LPC lanes per column, RPL rows per lane (LPC * RPL >= n_b).  RPL = 16 packs
// 32/LPC columns into a warp (the per-row scalar chain is shared by more columns); when the block
// has too few active columns to give every SM a full CTA of such warps, RPL = 8 spreads each
// column over twice the lanes instead (shorter substitution per lane, more warps).
// Safe variants follow the main launch with the synchronous fallback launch, which exits at once
// unless the main launch handed columns over (device-side count, no host synchronisation).
template <typename T, int LPC, int RPL, bool SAFE, int OP, bool GEN>
int launch_diag_pair(const DiagArgs<T> &a) {
    if (int rc = launch_diag_k<T, LPC, RPL, SAFE, OP, false, GEN>(a, a.ncols)) return rc;
    if (g_debug_sync) {
        cudaError_t e = cudaStreamSynchronize(g_stream);
        int cnt = -1;
        if (SAFE) cudaMemcpy(&cnt, a.fb_count, 4, cudaMemcpyDeviceToHost);
        fprintf(stderr, "[mstrsm debug] diag<%d,%d> block %lld main done (%s), ncols %lld, handed %d\n", LPC, RPL,
                (long long)a.b, cudaGetErrorString(e), (long long)a.ncols, cnt);
    }
    if (SAFE) return launch_diag_k<T, LPC, RPL, SAFE, OP, true, GEN>(a, std::min<int64_t>(a.ncols, int64_t(g_num_sms) * 32));
    return 0;
}

template <typename T, bool SAFE, int OP>
int launch_diag_old(const DiagArgs<T> &a, int nb) {
    // Whole passes of the grid over the columns: a pass of the RPL = 16 layout takes about 1.2x
    // one of the RPL = 8 layout (c5 launch list, profiles/r01), so pick the cheaper pass count.
    auto passes = [&](int lpc, int rpl) {
        const int64_t per_pass = int64_t(g_num_sms) * (rpl >= 16 ? DiagThreads<T, 16>::value : DiagThreads<T, 8>::value) / 32 * (32 / lpc);   // (RPL 4 uses RPL 8's CTA size)
        return cdiv(a.ncols, per_pass);
    };
    const int c16 = diag_cost(0), c4 = diag_cost(1);
    auto few = [&](int lpc16) { return 10 * passes(2 * lpc16, 8) < c16 * passes(lpc16, 16); };
    if (nb <= 16) return launch_diag_pair<T, 1, 16, SAFE, OP, false>(a);
    if (nb <= 32) return launch_diag_pair<T, 2, 16, SAFE, OP, false>(a);
    if (nb <= 64) return few(4) ? launch_diag_pair<T, 8, 8, SAFE, OP, false>(a) : launch_diag_pair<T, 4, 16, SAFE, OP, false>(a);
    if (g_cta_cap > 0) return launch_diag_pair<T, 8, 16, SAFE, OP, false>(a);   // look-ahead: densest layout
    // very few columns (the first blocks of TriangEig, every block of a multi-GPU shard): a whole
    // warp per column, 4 rows per lane -- the shortest per-row chain
    if (c4 * passes(32, 4) < 10 * passes(16, 8) && c4 * passes(32, 4) < c16 * passes(8, 16))
        return launch_diag_pair<T, 32, 4, SAFE, OP, false>(a);
    return few(8) ? launch_diag_pair<T, 16, 8, SAFE, OP, false>(a) : launch_diag_pair<T, 8, 16, SAFE, OP, false>(a);
}

// MSTRSM_DIAG_OLD=1: the round-1 row loop (diag_kernel) for the standard solve as well.
inline bool diag_old() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("MSTRSM_DIAG_OLD");
        v = (e && e[0] == '1') ? 1 : 0;
    }
    return v == 1;
}
// MSTRSM_DIAG_LPC=k forces the lanes per column of the chunked kernel (testing / tuning).
inline int diag_force_lpc() {
    static int v = -2;
    if (v == -2) {
        const char *e = getenv("MSTRSM_DIAG_LPC");
        v = e ? atoi(e) : 0;
    }
    return v;
}

template <typename T, int LPC, int RPL, bool SAFE, int OP>
int launch_diagf_k(const DiagArgs<T> &a0) {
    auto kern = diagw_kernel<T, LPC, RPL, SAFE, OP>;
    typedef DiagW<T, LPC, RPL, SAFE> W;
    constexpr int G = W::G;
    const int nfull = int(a0.hi - a0.lo);
    static std::atomic<uint64_t> attr_set{0};
    if (first_on_device(attr_set)) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    const int64_t groups = cdiv(a0.ncols, G);
    const int64_t sms = g_cta_cap > 0 ? g_cta_cap : g_num_sms;
    // one CTA per SM; equal passes: as many substitution warps per CTA as the pass count needs
    const int64_t npass = cdiv(groups, sms * W::kSub);
    // (at least 4 substitution warps per CTA, as diagl: the staging is shared by more warps)
    const int nsub = int(std::max<int64_t>(std::min<int64_t>(4, W::kSub),
                                           std::min<int64_t>(W::kSub, cdiv(groups, sms * npass))));
    const int threads = (nsub + diagw_nrep(nsub, LPC, SAFE)) * 32;
    const size_t smem = size_t(diagw_smem(nfull, LPC, RPL, sizeof(T), nsub * G, SAFE).total);
    int grid = int(std::min<int64_t>(cdiv(groups, nsub), sms));
    if (grid < 1) grid = 1;
    DiagArgs<T> a = a0;
    a.nsub = nsub;
#ifdef MSTRSM_PHASE_TIMES
    a.pt = phase_next();
#endif
    const double fl = double(a.ncols) * nfull * (nfull - 1) / 2.0 * (S<T>::cplx_ ? 8.0 : 2.0);
    ProfScope ps(PK_DIAG, fl);
    CK(launch_k(kern, dim3(grid), dim3(threads), smem, g_stream, a));
    CK_LAUNCH("diagw_kernel");
    return 0;
}

// The chunked kernel (it reruns the rare column whose values stop being finite with the
// synchronous guarded loop itself: no second launch).
template <typename T, int LPC, int RPL, bool SAFE, int OP>
int launch_diagf_pair(const DiagArgs<T> &a, int nb) {
    (void)nb;
    if (int rc = launch_diagf_k<T, LPC, RPL, SAFE, OP>(a)) return rc;
    if (g_debug_sync) {
        cudaError_t e = cudaStreamSynchronize(g_stream);
        fprintf(stderr, "[mstrsm debug] diagw<%d,%d> block %lld done (%s), ncols %lld\n", LPC, RPL, (long long)a.b,
                cudaGetErrorString(e), (long long)a.ncols);
    }
    return 0;
}

// MSTRSM_DIAG=tc|w forces the left-looking tensor-pipe kernel (diagl, where its shared memory
// fits) or the chunked one (diagw).  Default (measured, profiles/r02): diagl for real data (c2
// 1.57 -> 1.35 ms, c1 0.228 -> 0.220 ms), diagw for complex (c4 88.5 ms vs 92.9 ms with diagl;
// n_b = 128 complex does not fit diagl's scratch).
inline int diag_impl() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("MSTRSM_DIAG");
        v = (e && e[0] == 'w') ? 1 : ((e && e[0] == 't') ? 2 : ((e && e[0] == 'g') ? 3 : 0));
    }
    return v;
}

// The left-looking kernel keeps its per-warp scratch in shared memory: it is used when at least 8
// substitution warps fit beside the block's triangle (n_b <= 64 complex, <= 96 real: c1, c2, c4);
// larger blocks take the chunked kernel.
template <typename T, bool SAFE>
bool diagl_fits(int nfull) {
    const int npad = (nfull + kDLTile - 1) / kDLTile * kDLTile;
    return diagl_smem_bytes(npad, int(sizeof(T)), 8 * 8, SAFE) <= 227 * 1024;
}

// MSTRSM_DIAGL_TRIGGER=0|1: diagl_kernel triggers its dependent launch at its start, so the
// update GEMM after it becomes resident on the SMs the diagonal step leaves free and issues its
// first A k-tiles (read-only U) during that step (gemm_ws_kernel's early_a).  Default off: c2
// 1.252 ms without vs 1.274 with, c1 0.199 vs 0.198 (same box, profiles/r02/exp_trig_t1.txt).
inline int diagl_trigger() {
    static const int v = [] {
        const char *e = getenv("MSTRSM_DIAGL_TRIGGER");
        return (e && e[0] == '1' && !e[1]) ? 1 : 0;
    }();
    return v;
}

template <typename T, bool SAFE, int OP, bool GSCR = false>
int launch_diagl(const DiagArgs<T> &a0) {
    auto kern = diagl_kernel<T, SAFE, OP, GSCR>;
    static std::atomic<uint64_t> attr_set{0};
    if (first_on_device(attr_set)) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    const int nfull = int(a0.hi - a0.lo);
    const int NT = (nfull + kDLTile - 1) / kDLTile, npad = NT * kDLTile;
    const int64_t groups = cdiv(a0.ncols, 8);
    const int64_t sms = g_cta_cap > 0 ? g_cta_cap : g_num_sms;
    // substitution warps per CTA: as many as shared memory (the replay records grow with the CTA's
    // columns) and the 16-warp CTA allow, then as few as the pass count needs
    int kmax = 0;
    for (int ns = kDLMaxSub; ns >= 1; ns--) {
        if (ns + diagw_nrep(ns, 4, SAFE) > kDLMaxSub) continue;
        if (diagl_smem_bytes(npad, int(sizeof(T)), ns * 8, SAFE, GSCR) > 227 * 1024) continue;
        kmax = ns;
        break;
    }
    if (kmax == 0) return set_cuda_error(cudaErrorInvalidValue, "diagl_kernel: shared memory");
    (void)0;
    const int64_t npass = cdiv(groups, sms * kmax);
    // at least 4 substitution warps per CTA: with fewer columns than SMs x 4 warps the launch is
    // latency-bound anyway, and the triangle's staging is shared by more warps (a 1-warp CTA spent
    // a quarter of its instructions staging, ncu c2)
    const int nsub = int(std::max<int64_t>(std::min<int64_t>(4, kmax),
                                           std::min<int64_t>(kmax, cdiv(groups, sms * npass))));
    const int threads = (nsub + diagw_nrep(nsub, 4, SAFE)) * 32;
    const size_t smem = size_t(diagl_smem_bytes(npad, int(sizeof(T)), nsub * 8, SAFE, GSCR));
    int grid = int(std::min<int64_t>(cdiv(groups, nsub), sms));
    if (grid < 1) grid = 1;
    DiagArgs<T> a = a0;
    a.nsub = nsub;
    a.trig = diagl_trigger();
#ifdef MSTRSM_PHASE_TIMES
    a.pt = phase_next();
#endif
    const double fl = double(a.ncols) * nfull * (nfull - 1) / 2.0 * (S<T>::cplx_ ? 8.0 : 2.0);
    ProfScope ps(PK_DIAG, fl);
    CK(launch_k(kern, dim3(grid), dim3(threads), smem, g_stream, a));
    CK_LAUNCH("diagl_kernel");
    return 0;
}

// Layout of the chunked kernel: LPC lanes per column, RPL rows per lane (LPC RPL >= n_b).  Fewer
// lanes per column pack more columns into a warp (the per-row chain -- quotient, shuffle,
// replay -- is shared by more columns) but give each lane more rows (a longer update per row)
// and need more registers (fewer warps per SM).  Among the layouts that cover the active columns
// in the fewest passes of the grid, the one with the most lanes per column (the shortest row
// step) is taken.
template <typename T, bool SAFE, int OP>
int launch_diag(const DiagArgs<T> &a, int nb) {
    if (diag_old()) return launch_diag_old<T, SAFE, OP>(a, nb);
    const int impl = diag_impl();
    if ((impl == 2 || (impl == 0 && !S<T>::cplx_)) && diagl_fits<T, SAFE>(int(a.hi - a.lo)))
        return launch_diagl<T, SAFE, OP>(a);
    if (impl == 3 && a.Xscr) return launch_diagl<T, SAFE, OP, true>(a);   // MSTRSM_DIAG=g: global scratch
    auto passes = [&](int lpc, int nsub) {
        const int64_t per_pass = int64_t(g_cta_cap > 0 ? g_cta_cap : g_num_sms) * nsub * (32 / lpc);
        return cdiv(a.ncols, per_pass);
    };
    const int f = diag_force_lpc();
    if (nb <= 16) return launch_diagf_pair<T, 1, 16, SAFE, OP>(a, nb);
    if (nb <= 32) {
        if (f == 4 || (f == 0 && passes(4, DiagW<T, 4, 8, SAFE>::kSub) <= passes(2, DiagW<T, 2, 16, SAFE>::kSub)))
            return launch_diagf_pair<T, 4, 8, SAFE, OP>(a, nb);
        return launch_diagf_pair<T, 2, 16, SAFE, OP>(a, nb);
    }
    if (nb <= 64) {
        const int64_t p4 = passes(4, DiagW<T, 4, 16, SAFE>::kSub), p8 = passes(8, DiagW<T, 8, 8, SAFE>::kSub),
                      p16 = passes(16, DiagW<T, 16, 4, SAFE>::kSub);
        if (f == 16 || (f == 0 && p16 <= std::min(p8, p4))) return launch_diagf_pair<T, 16, 4, SAFE, OP>(a, nb);
        if (f == 8 || (f == 0 && p8 <= p4)) return launch_diagf_pair<T, 8, 8, SAFE, OP>(a, nb);
        return launch_diagf_pair<T, 4, 16, SAFE, OP>(a, nb);
    }
    // n_b > 64: (8, 16) packs 4 columns per warp but its 16 register slots make a large,
    // instruction-cache-hungry loop nest; two passes of (16, 8) beat one of (8, 16) (c5 diagonal
    // step 12.9 -> 12.2 ms, profiles/r02/exp_c5lpc.txt), so (8, 16) is only taken when forced
    const int64_t p16 = passes(16, DiagW<T, 16, 8, SAFE>::kSub), p32 = passes(32, DiagW<T, 32, 4, SAFE>::kSub);
    if (f == 8) return launch_diagf_pair<T, 8, 16, SAFE, OP>(a, nb);
    if (f == 32 || (f == 0 && p32 <= p16)) return launch_diagf_pair<T, 32, 4, SAFE, OP>(a, nb);
    return launch_diagf_pair<T, 16, 8, SAFE, OP>(a, nb);
}

// Generalized solve (Alg. 7/8, op N): U' = U - lambda V on the fly; n_b <= 64 (two packed
// triangles in shared memory).
template <typename T, bool SAFE>
int launch_diag_gen(const DiagArgs<T> &a, int nb) {
    const int64_t full_wave = int64_t(g_num_sms) * (DiagThreads<T, 16>::value / 32);
    if (nb <= 16) return launch_diag_pair<T, 1, 16, SAFE, 0, true>(a);
    if (nb <= 32) return launch_diag_pair<T, 2, 16, SAFE, 0, true>(a);
    return cdiv(a.ncols, 8) < full_wave ? launch_diag_pair<T, 8, 8, SAFE, 0, true>(a)
                                        : launch_diag_pair<T, 4, 16, SAFE, 0, true>(a);
}

}  // namespace rt
}  // namespace mstrsm
