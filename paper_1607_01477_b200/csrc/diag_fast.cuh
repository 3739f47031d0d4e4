// diag_fast.cuh -- a.3 diagonal-block multi-shift (safe) solve + a.4 column bound: the chunked,
// warp-specialised kernel of the standard solve (op N and op C, real and complex).
//
// Same operation and outputs as diag_kernel (diag_kernel.cuh, which stays as the generalized
// solve's kernel and as the synchronous fallback): for one block I1 and every active column j
//   plain:  Alg. 1 on U(I1,I1) - s_j I
//   safe :  Alg. 4 on U(I1,I1) - s_j I with block-local bounds (R5),
//           then steps (ii) and (iii) of Alg. 5.
// What differs is how the work is laid out:
//
//  * Chunks.  Lane r of an LPC-lane group owns the solve rows sc = r + LPC t (t < RPL).  Slot t
//    of the group is a chunk of LPC consecutive rows.  Within a chunk the row step is
//        x_l = y_l / d_l (owner's lane, shuffled to the group),  y(rows < l) -= U(rows, l) x_l
//    and the chunk's own slot is updated by every lane with no select: the diagonal block is
//    staged as a PADDED triangle whose column l is zero from row l to the end of l's chunk, so
//    lanes whose row is already solved (or is l itself) subtract x_l * 0.  The owner's quotient is
//    recomputed once at the end of the chunk from its (then final) y_l, bit-identical to the one
//    shuffled.
//  * Own frame.  The guarded loop of Alg. 4 only scales the whole vector by powers of two
//    (P:287), so its values are the unscaled substitution's values times 2^-K exactly
//    (K = exponents taken so far; barring subnormals, R27).  The registers hold the unscaled
//    values times 2^-F for a frame F of this kernel's own choosing: when the largest |x| of a
//    group passes 2^600 the group's registers are multiplied by 2^-s (s = that exponent) and
//    F += s.  The frame never depends on the paper's decisions, so the substitution never waits
//    for them.
//  * Replay warps.  Alg. 4's decisions are a sequential scalar chain per column.
//    The substitution warps record |x_l| (once per chunk, with the frame it was read in) in
//    shared memory and arrive on the chunk's mbarrier; one replay warp per 32 columns of the CTA
//    (one lane per column, instead of LPC lanes repeating the same chain) follows one chunk
//    behind and evaluates, in the paper's frame |x_l| = ax 2^(F - K):
//        |y_l| >= Omega |d_l|  <=>  |x_l| >= Omega (to rounding, R27)  ->  k1 = minpow2(|x_l|, Omega)
//        M = 2^-k1 |x_l|,  g = 2^-k1 g + M cnl(l),  g >= Omega  ->  k2 = minpow2(g, Omega)
//    and hands K back through the "done" mbarrier.  The substitution warps then take their
//    registers to the paper's frame with one exact power-of-two product, 2^(F - K).  A group
//    whose values stop being finite (growth of more than ~2^400 inside one chunk: tiny pivots)
//    is rerun in place by the synchronous guarded loop (diag_rows, Alg. 4 step by step).
#pragma once
#include "diag_kernel.cuh"

namespace mstrsm {

// (padtri_off, the padded triangle's column offsets: diag_kernel.cuh)

// CTA shape of an instantiation: up to kSub substitution warps (G columns each) and, for the
// safe variants, one replay warp per 32 of their columns.
// The CTA holds kWarps warps (a multiple of 4, so the register budget per thread is
// 65536 / (32 kWarps): 168 for the complex RPL = 16 layouts, 128 otherwise).
template <typename T, int LPC, int RPL, bool SAFE> struct DiagW {
    static constexpr int G = 32 / LPC;
    static constexpr int kWarps = (S<T>::cplx_ && RPL >= 16) ? 12 : 16;
    static constexpr int sub_fit(int s) { return (s + (SAFE ? (s * G + 31) / 32 : 0)) <= kWarps ? s : sub_fit(s - 1); }
    static constexpr int kSub = sub_fit(kWarps);
    static constexpr int kRep = SAFE ? (kSub * G + 31) / 32 : 0;
    static constexpr int kThreads = kWarps * 32;
};
__host__ __device__ inline int diagw_nrep(int nsub, int lpc, bool safe) { return safe ? (nsub * (32 / lpc) + 31) / 32 : 0; }

// Shared-memory carve-up (byte offsets, 16-aligned): padded triangle, diagonal, cnl, and for the
// safe variants the replay records |x| (row-major: [sc][column slot]), the chunk frames, the
// per-column g0 / live row count / K / G_j and e_j as read at the pass start, and RPL + 1 mbarriers.
struct DiagWSmem {
    int64_t pk, dg, cn, rec, fp, g0, lrows, kout, gj, ej, bar, total;
};
__host__ __device__ inline DiagWSmem diagw_smem(int nfull, int lpc, int rpl, int esize, int ncol_cta, bool safe) {
    auto al = [](int64_t v) { return (v + 15) & ~int64_t(15); };
    DiagWSmem s{};
    s.pk = 0;
    s.dg = al(padtri_off(nfull, lpc) * esize);
    s.cn = al(s.dg + int64_t(nfull) * esize);
    s.rec = al(s.cn + int64_t(nfull) * 8);
    if (!safe) { s.total = s.rec; return s; }
    s.fp = al(s.rec + int64_t(lpc) * rpl * ncol_cta * 8);
    s.g0 = al(s.fp + int64_t(rpl) * ncol_cta * 4);
    s.lrows = al(s.g0 + int64_t(ncol_cta) * 8);
    s.kout = al(s.lrows + int64_t(ncol_cta) * 4);
    s.gj = al(s.kout + int64_t(ncol_cta) * 4);
    s.ej = al(s.gj + int64_t(ncol_cta) * 8);
    s.bar = al(s.ej + int64_t(ncol_cta) * 4);
    s.total = s.bar + int64_t(rpl + 1) * 8;
    return s;
}

// The exponent of a non-negative double (biased; 0 for zero / subnormal, 2047 for inf / NaN).
__device__ __forceinline__ int bexp(double v) { return (__double2hiint(v) >> 20) & 0x7ff; }
// v with its biased exponent replaced by be (1 <= be <= 2046; v normal, non-negative).
__device__ __forceinline__ double with_bexp(double v, int be) {
    return __hiloint2double((__double2hiint(v) & 0x800fffff) | (be << 20), __double2loint(v));
}
// y := 2^s y for any integer s (one product when the factor is a normal double).
template <typename T, int N>
__device__ __forceinline__ void scale_pow2(T (&y)[N], int s) {
    if (s >= -1022 && s <= 1023) {
        const double p = pow2i(s);
#pragma unroll
        for (int t = 0; t < N; t++) {
            if constexpr (S<T>::cplx_) y[t] = make_double2(__dmul_rn(y[t].x, p), __dmul_rn(y[t].y, p));
            else y[t] = __dmul_rn(y[t], p);
        }
    } else {
        scale_all_any(y, s);
    }
}

// Alg. 4's decisions for one chunk of NR rows (solve rows sc0 + NR - 1 .. sc0) of one column: the
// replay warps' per-row chain in the paper's frame |x_l| = ax 2^(Fp - K) (R27), with
// ax = rec[sc * ldrec + c] recorded by the substitution warps.  Rows sc >= lrows are not live
// (M = 0, k1 = k2 = 0: g * 1 + 0).  cn is read at sc (0 for sc >= ncn).
template <int NR>
__device__ __forceinline__ void replay_chunk(const double *rec, int ldrec, int c, int sc0, int lrows, int Fp,
                                             const double *cn, int ncn, double &g, int &K) {
    // Branch-free form of the row for frame offsets dK = Fp - K in [-1022, 1023] and k1 <= 1022
    // (the exact products below are then single multiplications by normal powers of two); a chunk
    // in which any row leaves that range is replayed from its start by the general form.  Both
    // evaluate the same expressions, so g and K are identical.
    const double g_in = g;
    const int K_in = K;
    {
        bool bad = false;
        const double *rp = rec + (sc0 + NR - 1) * ldrec + c;
        const double *cp = cn + (sc0 + NR - 1);
#pragma unroll 8
        for (int rr = NR - 1; rr >= 0; rr--, rp -= ldrec, cp--) {
            const bool live = sc0 + rr < lrows;
            const double ax = live ? *rp : 0.0;
            const double cr = sc0 + rr < ncn ? *cp : cn[0];
            const int ea = bexp(ax);
            const int dK = Fp - K;
            const int ep = ea + dK;                       // biased exponent, paper frame
            const bool t1 = live && ea != 0 && ep >= 1993;    // |x_l| >= 2^970
            const int k1 = t1 ? ep - 1992 : 0;
            bad |= unsigned(dK + 1022) > 2045u || k1 > 1022;
            double M = t1 ? with_bexp(ax, 1992) : __dmul_rn(ax, pow2i(dK));   // 2^-k1 |x_l|
            M = live ? M : 0.0;
            const double gs = __dmul_rn(g, pow2i(-k1));   // P:287 applied to g
            const double gn = __dadd_rn(gs, __dmul_rn(M, cr));
            const bool t2 = live && gn >= kOmega;
            const int k2 = t2 ? bexp(gn) - 1992 : 0;
            g = __dmul_rn(gn, pow2i(-k2));
            K += k1 + k2;
        }
        if (!bad) return;
    }
    g = g_in;
    K = K_in;
#pragma unroll 1
    for (int rr = NR - 1; rr >= 0; rr--) {
        const int sc = sc0 + rr;
        const bool live = sc < lrows;
        const double ax = live ? rec[sc * ldrec + c] : 0.0;
        const int ea = bexp(ax);
        const int dK = Fp - K;
        const int ep = ea + dK;                           // biased exponent, paper frame
        const bool t1 = live && ea != 0 && ep >= 1993;    // |x_l| >= 2^970
        const int k1 = t1 ? ep - 1992 : 0;
        double M, gs;
        if (unsigned(dK + 1022) <= 2045u && k1 <= 1022) {
            M = t1 ? with_bexp(ax, 1992) : __dmul_rn(ax, pow2i(dK));   // 2^-k1 |x_l|
            gs = __dmul_rn(g, pow2i(-k1));                // P:287 applied to g
        } else {                                          // extreme frames (rare)
            M = t1 ? with_bexp(ax, 1992) : mulp2_any(ax, dK);
            gs = mulp2n(g, k1);
        }
        M = live ? M : 0.0;
        double gn = __dadd_rn(gs, __dmul_rn(M, cn[sc < ncn ? sc : 0]));
        const bool t2 = live && gn >= kOmega;
        const int k2 = t2 ? bexp(gn) - 1992 : 0;
        g = __dmul_rn(gn, pow2i(-k2));
        K += k1 + k2;
    }
}

// An upper bound of 1/v for the prechecks (v >= 0): the correctly rounded reciprocal raised by one
// ulp and by the smallest subnormal (its error is below both), rounded up; inf for v = 0, NaN for
// NaN.  Cheaper than __drcp_ru (no called slow path).
__device__ __forceinline__ double rcp_up(double v) {
    return __dadd_ru(__dmul_ru(__drcp_rn(v), 1.0 + 0x1p-52), 0x1p-1074);
}

template <int LPC>
__device__ __forceinline__ int group_imax(int v) {
#pragma unroll
    for (int o = 1; o < LPC; o <<= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o, LPC));
    return v;
}

__device__ __forceinline__ void dw_mbar_init(uint64_t *b, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void dw_mbar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
// Device-side checks of the diagonal kernels' shared-memory indexing and barrier protocol
// (compute-sanitizer is unavailable on the GPU pool): built with -DMSTRSM_DEVICE_CHECKS
// (tools/build_checks.sh), a failed check prints its site and traps.
#ifdef MSTRSM_DEVICE_CHECKS
#define DW_CHECK(cond, what)                                                                   \
    do {                                                                                       \
        if (!(cond)) {                                                                         \
            printf("mstrsm device check failed: %s (block %d thread %d)\n", what, int(blockIdx.x), \
                   int(threadIdx.x));                                                          \
            __trap();                                                                          \
        }                                                                                      \
    } while (0)
#else
#define DW_CHECK(cond, what) do { } while (0)
#endif

__device__ __forceinline__ void dw_mbar_wait(uint64_t *b, int parity) {
    uint32_t done = 0;
#ifdef MSTRSM_DEVICE_CHECKS
    long long spins = 0;
#endif
    do {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                     " selp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(done) : "r"(smem_u32(b)), "r"(parity) : "memory");
#ifdef MSTRSM_DEVICE_CHECKS
        DW_CHECK(++spins < (1ll << 26), "mbarrier wait does not complete (protocol deadlock)");
#endif
    } while (!done);
}

// Chunked row loop of one column group.  REC = false: Alg. 1 (the plain solve and the unguarded
// branch of Alg. 4), bit-identical to diag_subst.  REC = true: the guarded loop's substitution in
// the kernel's own frame, recording |x| of every row (rec[sc * ldrec]) and the frame of every
// chunk (fp[t * ldrec], lane 0) for the replay warps; returns false when the group's values
// stopped being finite.  Every chunk's mbarrier is arrived on (safe variants), solved or skipped.
template <typename T, int LPC, int RPL, bool SAFE, bool REC, bool CONJ, typename PivF>
__device__ __forceinline__ bool diagw_rows(T (&y)[RPL], PivF pivot, const T *__restrict__ pk, int rl, int nmax,
                                           bool guarded, double gub, double *rec, int *fp, int ldrec,
                                           uint64_t *bars, int &Fout) {
    typedef S<T> ST;
    int F = 0;
    bool nonfinite = false;
    auto uget = [&](const T *p) -> T {
        if constexpr (CONJ) return ST::conj(*p);   // op C: L = U^H staged unconjugated
        else return *p;
    };
    if constexpr (REC) {                                                   // initial frame
        const int e0 = bexp(gub);
        const bool need = guarded && e0 > 1623 && e0 < 2047;
        if (__any_sync(0xffffffffu, need)) {
            const int s = need ? min(e0 - 1023, 1022) : 0;
            scale_all<true>(y, s);
            F = s;
        }
    }
#pragma unroll
    for (int t = RPL - 1; t >= 0; t--) {
        if (t * LPC < nmax) {                                              // warp-uniform
            Piv<T> pvt;                                                    // own row of slot t
            pvt.make(pivot(t * LPC + rl));
            const int rr_hi = min(LPC - 1, nmax - 1 - t * LPC);           // rows >= nmax skipped
            const int kStride = LPC * (t + 1);                            // padded column length
            const T *pc = pk + (LPC * LPC * t * (t + 1) / 2 + rl) + rr_hi * kStride;
#pragma unroll 1
            for (int rr = rr_hi; rr >= 0; rr--, pc -= kStride) {
                DW_CHECK(pc >= pk && pc + LPC * t < pk + padtri_off(t * LPC + rr + 1, LPC), "diagw row pointer");
                T uc[RPL];                                                 // U(rows, l): loads first,
#pragma unroll                                                                     // under the quotient's shuffle
                for (int t2 = 0; t2 < RPL; t2++)
                    if (t2 <= t) uc[t2] = uget(pc + LPC * t2);
                const T xl = group_shfl<T, LPC>(pvt.apply(y[t]), rr);      // P:82 / P:297
                y[t] = ST::fnms(y[t], xl, uc[t]);                          // zero for rows >= l
#pragma unroll
                for (int t2 = t - 1; t2 >= 0; t2--) y[t2] = ST::fnms(y[t2], xl, uc[t2]);
            }
            const T xo = pvt.apply(y[t]);                                  // = the shuffled x_l
            y[t] = xo;
            if constexpr (REC) {
                const double ax = modv(xo);
                nonfinite |= !(ax <= 1.7976931348623157e308);
                DW_CHECK(t * LPC + rl < LPC * RPL, "diagw record row");
                rec[(t * LPC + rl) * ldrec] = ax;
                if (rl == 0) fp[t * ldrec] = F;
                const int em = group_imax<LPC>(bexp(ax));
                const bool need = guarded && em > 1623 && em < 2047;      // |x| >= 2^601: new frame
                if (__any_sync(0xffffffffu, need)) {
                    const int s = need ? min(em - 1023, 1022) : 0;
                    scale_all<true>(y, s);
                    F += s;
                }
            }
        }
        if constexpr (SAFE) dw_mbar_arrive(bars + t);
    }
    if constexpr (REC) {
#pragma unroll
        for (int o = 1; o < LPC; o <<= 1) nonfinite |= __shfl_xor_sync(0xffffffffu, nonfinite, o, LPC);
    }
    Fout = F;
    return !(guarded && nonfinite);
}

// One launch = one diagonal block for the active columns [c0, c0 + ncols).  Warps 0 .. nsub-1
// substitute (G columns each), the rest replay (safe variants).  The column loop runs in passes of
// nsub G columns per CTA; every warp of the CTA takes part in every pass.
template <typename T, int LPC, int RPL, bool SAFE, int OP>
__global__ void __launch_bounds__(DiagW<T, LPC, RPL, SAFE>::kThreads, 1) diagw_kernel(DiagArgs<T> a) {
    typedef S<T> ST;
    constexpr int G = 32 / LPC;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int nfull = int(a.hi - a.lo);
    const int64_t ncols = a.ncols;
    const int nsub = a.nsub, C = nsub * G;
    const DiagWSmem L = diagw_smem(nfull, LPC, RPL, int(sizeof(T)), C, SAFE);
    T *pk = reinterpret_cast<T *>(smem_raw + L.pk);
    T *dg = reinterpret_cast<T *>(smem_raw + L.dg);
    double *cn = reinterpret_cast<double *>(smem_raw + L.cn);
    double *s_rec = reinterpret_cast<double *>(smem_raw + L.rec);
    int *s_fp = reinterpret_cast<int *>(smem_raw + L.fp);
    double *s_g0 = reinterpret_cast<double *>(smem_raw + L.g0);
    int *s_lrows = reinterpret_cast<int *>(smem_raw + L.lrows);
    int *s_k = reinterpret_cast<int *>(smem_raw + L.kout);
    double *s_gj = reinterpret_cast<double *>(smem_raw + L.gj);
    int *s_ej = reinterpret_cast<int *>(smem_raw + L.ej);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + L.bar);   // [0, RPL): chunks, [RPL]: done
    const int tid = threadIdx.x, nth = blockDim.x;
    const int warp = tid >> 5, lane = tid & 31;

    // ---- stage U(I1,I1) as the padded triangle (solve coordinates), its diagonal and cnl.  U and
    //      cnl are never written during a solve, so a launch after the solve's first one stages
    //      them before waiting for the preceding grid (a.early) ----
    pdl_trigger();
    PT_MARK(a.pt, 0, tid == 0);
    PT_MARK(a.pt, 1, tid == 0);
    if (!a.early) pdl_wait();
    for (int cq = tid >> 5; cq < nfull; cq += nth >> 5) {                 // a warp per column of U,
        for (int r = tid & 31; r < cq; r += 32) {                           // lanes down its rows
            const T *src = a.U + (a.lo + r) + (a.lo + cq) * a.ldu;         // U(lo + r, lo + cq)
            DW_CHECK(padtri_off(cq, LPC) + r < padtri_off(nfull, LPC) &&
                         padtri_off(nfull - 1 - r, LPC) + (nfull - 1 - cq) < padtri_off(nfull, LPC), "diagw staging index");
            if (OP == 0) cp_async<sizeof(T)>(pk + padtri_off(cq, LPC) + r, src, true);
            else cp_async<sizeof(T)>(pk + padtri_off(nfull - 1 - r, LPC) + (nfull - 1 - cq), src, true);
        }
    }
    for (int idx = tid; idx < nfull * LPC; idx += nth) {                 // zeros from row l down
        const int l = idx / LPC, r = (l / LPC) * LPC + idx % LPC;
        if (r >= l) pk[padtri_off(l, LPC) + r] = ST::zero();
    }
    for (int c = tid; c < nfull; c += nth) {
        const int64_t row = OP == 0 ? a.lo + c : a.hi - 1 - c;
        const T u = a.U[row + row * a.ldu];
        dg[c] = OP == 0 ? u : ST::conj(u);
        cn[c] = SAFE ? a.cnl[row] : 0.0;
    }
    if (SAFE && tid == 0) {
        for (int t = 0; t < RPL; t++) dw_mbar_init(bars + t, nsub * 32);
        dw_mbar_init(bars + RPL, diagw_nrep(nsub, LPC, true) * 32);
    }
    cp_async_commit();
    if (a.early) pdl_wait();
    __syncthreads();                                                       // diagonal, cnl, barriers
    PT_MARK(a.pt, 2, tid == 0);
    bool staged = false;
    auto stage_wait = [&]() { cp_async_wait<0>(); __syncthreads(); staged = true; };

    const int64_t cstride = int64_t(gridDim.x) * C;
    if (warp >= nsub) {
        // =========================== replay warp: one lane per column slot ===========================
        if constexpr (SAFE) {
            stage_wait();
            PT_MARK(a.pt, 10, warp == nsub && lane == 0);
            const int c = (warp - nsub) * 32 + lane;
            int pass = 0;
            for (int64_t cb = int64_t(blockIdx.x) * C; cb < ncols; cb += cstride, pass++) {
                const int par = pass & 1;
                int K = 0, lrows = 0;
                double g = 0.0;
#pragma unroll 1
                for (int t = RPL - 1; t >= 0; t--) {
                    dw_mbar_wait(bars + t, par);
                    if (t == RPL - 1 && c < C) { g = s_g0[c]; lrows = s_lrows[c]; }
                    if (!__any_sync(0xffffffffu, lrows > t * LPC)) continue;
                    const int Fp = lrows > t * LPC ? s_fp[t * C + c] : 0;
                    replay_chunk<LPC>(s_rec, C, c, t * LPC, lrows, Fp, cn, nfull, g, K);
                }
                if (c < C) s_k[c] = K;
                PT_MARK(a.pt, 11, warp == nsub && lane == 0 && pass == 0);
                dw_mbar_arrive(bars + RPL);
            }
        }
        if (!staged) stage_wait();
        return;
    }

    // =============================== substitution warps ===============================
    const int grp = lane / LPC, rl = lane % LPC;
    const int c = warp * G + grp;                                         // column slot in the CTA
    const double delta = SAFE ? a.delta[0] : 0.0;
    const double Pb = SAFE ? diag_panel_sum(a) : 0.0;
    int pass = 0;
    for (int64_t cb = int64_t(blockIdx.x) * C; cb < ncols; cb += cstride, pass++) {
        const int64_t q = cb + c;
        const bool valid = q < ncols;
        const int64_t j = a.c0 + (valid ? q : 0);
        // the pass's column loads (shift, G_j, e_j) issue together, before the row end is known
        T *x = a.B + j * a.ldb;
        auto rowof = [&](int sc) -> int64_t { return OP == 0 ? a.lo + sc : a.hi - 1 - sc; };
        T sh = valid ? a.shifts[j * a.sstride] : ST::zero();
        const double Gj0 = (SAFE && valid) ? a.G[j] : 0.0;
        const int64_t r = valid ? ((OP == 0 && a.rowend) ? a.rowend[j] : a.m) : 0;
        const bool active = valid && r > a.lo;
        if (SAFE && valid && !active && rl == 0) a.dblk[j] = 0;           // inactive column: no rescale
        if (SAFE && rl == 0) {                                             // (kept for the finish)
            s_gj[c] = Gj0;
            s_ej[c] = valid ? a.e[j] : 0;
        }
        const int nrow = active ? (OP == 0 ? int((a.hi < r ? a.hi : r) - a.lo) : nfull) : 0;
        int nmax = nrow;
#pragma unroll
        for (int o = LPC; o < 32; o <<= 1) nmax = max(nmax, __shfl_xor_sync(0xffffffffu, nmax, o));
        if (!active) sh = ST::zero();
        if (OP == 1) sh = ST::conj(sh);
        auto pivot = [&](int sc) -> T {                                    // d_l = U(l,l) - s_j
            T dd = sc < nrow ? ST::sub(dg[sc], sh) : ST::real(1.0);
            if (SAFE && ST::is_zero(dd)) dd = ST::real(delta);
            return dd;
        };
        T y[RPL];
#pragma unroll
        for (int t = 0; t < RPL; t++) {
            const int sc = rl + LPC * t;
            y[t] = sc < nrow ? x[rowof(sc)] : ST::zero();
        }
        PT_MARK(a.pt, 3, tid == 0 && pass == 0);

        bool guarded = false;
        double g0 = 0.0, gub = 0.0;
        if (SAFE) {
            // ---- precheck, eqs. (4)-(5), with upper bounds (R36): ||y(I1)||_inf <=
            //      G_j, every suffix product <= the whole block's product of (1 + cnl/|d|), every
            //      1/|d| <= their max.  It only picks the unguarded loop when no rescale can
            //      trigger; the guarded one returns the same values whenever none does ----
            double prod = 1.0, minv = 0.0;
#pragma unroll
            for (int t = 0; t < RPL; t++) {
                const int sc = rl + LPC * t;
                if (sc < nrow) {
                    const double inv = rcp_up(maxabs(pivot(sc)));         // >= 1/|d_l|
                    prod = __dmul_ru(prod, __dadd_ru(1.0, __dmul_ru(cn[sc], inv)));
                    minv = fmax(minv, inv);
                }
            }
#pragma unroll
            for (int o = 1; o < LPC; o <<= 1) {
                prod = __dmul_ru(prod, __shfl_xor_sync(0xffffffffu, prod, o, LPC));
                minv = fmax(minv, __shfl_xor_sync(0xffffffffu, minv, o, LPC));
            }
            const double gtop = active ? __dmul_ru(Gj0, 1.0 + 0x1p-40) : 0.0;      // >= ||y(I1)||_inf
            const double carry = __dmul_ru(gtop, prod);
            const bool okM = __dmul_ru(carry, minv) < kOmega;
            // initial frame bound for the guarded loop: the registers' largest |y| (upper bound)
#pragma unroll
            for (int t = 0; t < RPL; t++)
                if (rl + LPC * t < nrow) gub = fmax(gub, maxabs(y[t]));
            gub = group_max<LPC>(gub);
            if constexpr (ST::cplx_) gub = __dmul_ru(gub, 1.4142135623730951);
            guarded = active && !(okM && carry < kOmega);
            if (__any_sync(0xffffffffu, guarded)) {                        // g := ||y(I1)||_inf
                if constexpr (ST::cplx_) {
                    g0 = modv_max(y, RPL);                                 // (rows >= nrow hold 0)
                } else {
#pragma unroll
                    for (int t = 0; t < RPL; t++)
                        if (rl + LPC * t < nrow) g0 = fmax(g0, modv(y[t]));
                }
                g0 = group_max<LPC>(g0);
            }
            if (rl == 0) {                                                 // the replay's inputs
                s_g0[c] = g0;
                s_lrows[c] = guarded ? nrow : 0;
            }
        }

        PT_MARK(a.pt, 4, tid == 0 && pass == 0);
        if (!staged) stage_wait();
        PT_MARK(a.pt, 5, tid == 0 && pass == 0);
        int F = 0;
        bool failed = false;
        if (SAFE && __any_sync(0xffffffffu, guarded)) {
            failed = !diagw_rows<T, LPC, RPL, SAFE, true, OP == 1>(y, pivot, pk, rl, nmax, guarded, gub, s_rec + c,
                                                                   s_fp + c, C, bars, F) ||
                     (a.force_fb && guarded);
        } else {
            diagw_rows<T, LPC, RPL, SAFE, false, OP == 1>(y, pivot, pk, rl, nmax, false, 0.0, s_rec + c, s_fp + c,
                                                          C, bars, F);
        }
        PT_MARK(a.pt, 6, tid == 0 && pass == 0);
        // steps (ii) and (iii) of Alg. 5 and the stores, for the groups with `keep`
        auto finish = [&](int kt, bool keep) {
            if (SAFE) {
                int ej = 0;
                double Gj = 0.0;
                if (active) { ej = s_ej[c]; Gj = s_gj[c]; }
                if (kt > 0) {                                              // P:376-386, step (ii)
                    ej -= kt;
                    Gj = mulp2n(Gj, kt);
                }
                double xm = 0.0;
                if constexpr (ST::cplx_) {
                    xm = modv_max(y, RPL);
                } else {
#pragma unroll
                    for (int t = 0; t < RPL; t++) xm = fmax(xm, modv(y[t]));
                }
                xm = group_max<LPC>(xm);
                Gj = __dadd_rn(Gj, __dmul_rn(Pb, xm));
                int k3 = 0;
                if (Gj >= kOmega) {
                    k3 = minpow2_bits(Gj, kOmega);
                    scale_all<false>(y, k3);
                    ej -= k3;
                    Gj = mulp2n(Gj, k3);
                }
                if (active && rl == 0 && keep) {
                    a.e[j] = ej;
                    a.G[j] = Gj;
                    a.dblk[j] = -(kt + k3);
                    a.Etab[a.b * a.n + j] = ej;
                }
                if (active && keep) pair_fix(a, j, -(kt + k3), ej, rl, LPC);
            }
#pragma unroll
            for (int t = 0; t < RPL; t++) {
                const int sc = rl + LPC * t;
                if (sc < nrow && keep) x[rowof(sc)] = y[t];
            }
            if constexpr (ST::cplx_) {  // operand sums for the 3M update GEMM
                if (a.Xsum && valid && keep) {
                    double *xs = a.Xsum + j * a.ldxs;
#pragma unroll
                    for (int t = 0; t < RPL; t++) {
                        const int sc = rl + LPC * t;
                        if (sc < nfull) xs[rowof(sc) - a.lo] = __dadd_rn(y[t].x, y[t].y);
                    }
                }
            }
        };
        int kt = 0;
        if (SAFE) {
            dw_mbar_wait(bars + RPL, pass & 1);                            // K from the replay warp
            kt = s_k[c];
            PT_MARK(a.pt, 7, tid == 0 && pass == 0);
            if (!failed && F != kt) scale_pow2(y, F - kt);                 // to the paper's frame
        }
        finish(kt, !failed);
        PT_MARK(a.pt, 8, tid == 0 && pass == 0);
        if (SAFE && __any_sync(0xffffffffu, failed)) {
            // a group whose values stopped being finite (tiny pivots: growth beyond the frame's
            // headroom inside one chunk) is rerun from its inputs by the synchronous guarded loop,
            // Alg. 4 step by step; the other groups of the warp idle through it
            const int nrow_f = failed ? nrow : 0;
            int nmax_f = nrow_f;
#pragma unroll
            for (int o = LPC; o < 32; o <<= 1) nmax_f = max(nmax_f, __shfl_xor_sync(0xffffffffu, nmax_f, o));
#pragma unroll
            for (int t = 0; t < RPL; t++) {
                const int sc = rl + LPC * t;
                y[t] = sc < nrow_f ? x[rowof(sc)] : ST::zero();
            }
            auto pivot_f = [&](int sc) -> T {
                T dd = sc < nrow_f ? ST::sub(dg[sc], sh) : ST::real(1.0);
                if (ST::is_zero(dd)) dd = ST::real(delta);
                return dd;
            };
            const UAcc<T, false, OP == 1> ua{pk, nullptr, cn, nullptr, ST::zero(), 0.0};
            double g = g0;
            int kt2 = 0;
            diag_rows<T, LPC, RPL, true, LPC>(y, pivot_f, ua, rl, nrow_f, nmax_f, failed, g, kt2);
            finish(kt2, failed);
        }
    }
    if (!staged) stage_wait();
    PT_MARK(a.pt, 9, tid == 0);
    PT_MARK(a.pt, 15, tid == 0);
}

}  // namespace mstrsm
