// diag_tc.cuh -- a.3 diagonal-block multi-shift (safe) solve + a.4 column bound, left-looking, with
// the in-block update on the FP64 tensor pipe (DMMA).  Standard solve, op N and op C, real and
// complex, plain and safe; same operation and outputs as diagw_kernel (diag_fast.cuh):
//   plain:  Alg. 1 on U(I1,I1) - s_j I
//   safe :  Alg. 4 on U(I1,I1) - s_j I with block-local bounds (R5),
//           then steps (ii) and (iii) of Alg. 5.
//
// Layout.  A warp owns 8 columns (lane = 4 column + r, r < 4) and walks the block's rows in tiles
// of 8 (solve coordinates, highest tile first).  Lane r of a column holds rows 8u + 2r and
// 8u + 2r + 1 of tile u: exactly the accumulator fragment of mma.sync.m8n8k4.f64 with the columns
// as M and the tile's rows as N.  Tile u is
//   1. loaded (its right-hand sides, in the column's current frame),
//   2. updated left-looking by every tile already solved: y(tile u) -= U(tile u, solved) x(solved),
//      as DMMAs over k-steps of 4 solved rows: A = -x (the column's solved values, 8 columns x 4
//      rows, from a per-column scratch), B = U(8 rows of tile u, 4 solved rows) from the block's
//      padded triangle in shared memory -- the bulk of the block's flops on the tensor pipe;
//   3. solved row by row inside the tile (x_l = y_l / d_l, shuffled to the column's 4 lanes, the
//      tile's other rows updated from the padded triangle: no selects);
//   4. its |x| recorded for the replay warps (safe), its -x written to the scratch.
// The power-of-two frame, the replay warps and the synchronous fallback are those of
// diag_fast.cuh (one chunk = one tile of 8 rows): the registers hold the unscaled substitution's
// values times 2^-F (F raised when |x| passes 2^600; the solved rows in the scratch are rescaled
// with it), the replay warps evaluate Alg. 4's decisions in the paper's frame (R27) and return K,
// and a column whose values stop being finite is rerun in place by the synchronous guarded loop
// (diag_rows, one warp per column).  The output rows are written once, at the end, in the paper's
// frame 2^(F - K - k3).  Summation order of the update: the tensor pipe's (R24, R20).
//
// Precheck (eqs. (4)-(5)).  Its only role is to pick the unguarded loop when no rescale
// can trigger; the guarded loop gives the same result whenever none does.  It is evaluated with
// upper bounds: ||y(I1)||_inf <= G_j (Alg. 5's column bound, P:354-360 / P:390-406, which bounds
// every remaining entry of the column), the whole-block product of (1 + cnl_l/|d_l|) for every
// suffix product and max 1/|d_l| for every 1/|d_l| -- a column the exact test passes may be
// guarded, never the reverse.
#pragma once
#include "diag_fast.cuh"

namespace mstrsm {

constexpr int kDLTile = 8;          // rows per tile (the DMMA n dimension)
constexpr int kDLMaxSub = 16;       // substitution warps per CTA (8 columns each)

__device__ __forceinline__ void dl_dmma(double &c0, double &c1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(c0), "+d"(c1)
        : "d"(a), "d"(b));
}

// y += U x or y += conj(U) x for one k-step (x = the A fragment, already negated: -x_solved).
template <typename T, bool CONJ>
__device__ __forceinline__ void dl_kstep(T &acc0, T &acc1, const T nx, const T u) {
    if constexpr (S<T>::cplx_) {
        if constexpr (!CONJ) {                 // re += nx.re U.re - nx.im U.im ; im += nx.im U.re + nx.re U.im
            dl_dmma(acc0.x, acc1.x, nx.x, u.x);
            dl_dmma(acc0.x, acc1.x, -nx.y, u.y);
            dl_dmma(acc0.y, acc1.y, nx.y, u.x);
            dl_dmma(acc0.y, acc1.y, nx.x, u.y);
        } else {                               // conj(U): re += nx.re U.re + nx.im U.im ; im += nx.im U.re - nx.re U.im
            dl_dmma(acc0.x, acc1.x, nx.x, u.x);
            dl_dmma(acc0.x, acc1.x, nx.y, u.y);
            dl_dmma(acc0.y, acc1.y, nx.y, u.x);
            dl_dmma(acc0.y, acc1.y, -nx.x, u.y);
        }
    } else {
        dl_dmma(acc0, acc1, nx, u);
    }
}

__device__ __forceinline__ double dl_scale1(double v, int s) {     // v 2^s, exact power of two
    return (s >= -1022 && s <= 1023) ? __dmul_rn(v, pow2i(s)) : mulp2_any(v, s);
}
__device__ __forceinline__ cplx dl_scale1(cplx v, int s) { return make_double2(dl_scale1(v.x, s), dl_scale1(v.y, s)); }

template <int W>
__device__ __forceinline__ double dl_gmax(double v) {
#pragma unroll
    for (int o = 1; o < W; o <<= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o, W));
    return v;
}
template <int W>
__device__ __forceinline__ double dl_gprod_ru(double v) {
#pragma unroll
    for (int o = 1; o < W; o <<= 1) v = __dmul_ru(v, __shfl_xor_sync(0xffffffffu, v, o, W));
    return v;
}

// Shared-memory bytes of one launch: diag_fast.cuh's carve-up (tiles as chunks of 8 rows) plus
// the solved rows' scratch (column stride diagl_scr_ld).
// Column stride of the scratch: a k-step's 32 lanes (8 columns x 4 rows) read word gq S + tq;
// for 8-byte elements S = npad + 4 (= 4 or 12 mod 16: every 8-byte bank pair serves two lanes,
// the 2-wavefront minimum; npad + 1 put up to 4 lanes on one pair), for 16-byte elements npad + 1
// (each 16-byte bank group already serves 4 lanes, the minimum).
__host__ __device__ inline int64_t diagl_scr_ld(int npad, int esize) { return npad + (esize == 8 ? 4 : 1); }
__host__ __device__ inline int64_t diagl_scr_offset(int npad, int esize, int ncol, bool safe) {
    return (diagw_smem(npad, kDLTile, npad / kDLTile, esize, ncol, safe).total + 15) & ~int64_t(15);
}
__host__ __device__ inline int64_t diagl_smem_bytes(int npad, int esize, int ncol, bool safe, bool gscr = false) {
    return diagl_scr_offset(npad, esize, ncol, safe) + (gscr ? 0 : int64_t(ncol) * diagl_scr_ld(npad, esize) * esize);
}

// GSCR: the solved rows' scratch lives in global memory (a.Xscr, L2-resident; for blocks whose
// triangle leaves no room for it in shared memory: n_b = 128 complex), read through a 4-deep
// register prefetch ring; otherwise in shared memory.
template <typename T, bool SAFE, int OP, bool GSCR = false>
__global__ void __launch_bounds__((kDLMaxSub) * 32, 1) diagl_kernel(DiagArgs<T> a) {
    typedef S<T> ST;
    constexpr int G = 8, TR = kDLTile;
    constexpr bool CONJ = OP == 1;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int nfull = int(a.hi - a.lo);
    const int NT = (nfull + TR - 1) / TR, npad = NT * TR;
    const int64_t ncols = a.ncols;
    const int nsub = a.nsub, C = nsub * G;
    const DiagWSmem L = diagw_smem(npad, TR, NT, int(sizeof(T)), C, SAFE);
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
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + L.bar);   // [0, NT): tiles, [NT]: done
    const int tid = threadIdx.x, nth = blockDim.x;
    const int warp = tid >> 5, lane = tid & 31;

    // ---- stage U(I1,I1) as the padded triangle with 8-row chunks (solve coordinates; columns
    //      nfull .. npad-1 all zero), its diagonal (1 past nfull) and cnl (0 past nfull).  U and
    //      cnl are never written during a solve: launches after the first stage before the wait ----
    if (a.trig) pdl_trigger();                                             // (launcher's choice)
    PT_MARK(a.pt, 0, tid == 0);
    PT_MARK(a.pt, 1, tid == 0);
    if (!a.early) pdl_wait();
    for (int cq = tid >> 5; cq < nfull; cq += nth >> 5) {                 // a warp per column of U,
        for (int r = tid & 31; r < cq; r += 32) {                           // lanes down its rows
            const T *src = a.U + (a.lo + r) + (a.lo + cq) * a.ldu;         // U(lo + r, lo + cq)
            DW_CHECK(padtri_off(cq, TR) + r < padtri_off(npad, TR) &&
                         padtri_off(nfull - 1 - r, TR) + (nfull - 1 - cq) < padtri_off(npad, TR), "diagl staging index");
            if (OP == 0) cp_async<sizeof(T)>(pk + padtri_off(cq, TR) + r, src, true);
            else cp_async<sizeof(T)>(pk + padtri_off(nfull - 1 - r, TR) + (nfull - 1 - cq), src, true);
        }
    }
    for (int idx = tid; idx < npad * TR; idx += nth) {                   // zeros from row l down
        const int l = idx / TR, r = (l / TR) * TR + idx % TR;
        if (r >= l || l >= nfull) pk[padtri_off(l, TR) + r] = ST::zero();
    }
    for (int idx = tid; idx < (npad - nfull) * npad; idx += nth) {       // padding columns: rows < l
        const int l = nfull + idx / npad, r = idx % npad;
        if (r < l) pk[padtri_off(l, TR) + r] = ST::zero();
    }
    for (int c = tid; c < npad; c += nth) {
        if (c < nfull) {
            const int64_t row = OP == 0 ? a.lo + c : a.hi - 1 - c;
            const T u = a.U[row + row * a.ldu];
            dg[c] = OP == 0 ? u : ST::conj(u);
            cn[c] = SAFE ? a.cnl[row] : 0.0;
        } else {
            dg[c] = ST::real(1.0);
            cn[c] = 0.0;
        }
    }
    if (SAFE && tid == 0) {
        for (int t = 0; t < NT; t++) dw_mbar_init(bars + t, nsub * 32);
        dw_mbar_init(bars + NT, diagw_nrep(nsub, 4, true) * 32);
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
                for (int t = NT - 1; t >= 0; t--) {
                    dw_mbar_wait(bars + t, par);
                    if (t == NT - 1 && c < C) { g = s_g0[c]; lrows = s_lrows[c]; }
                    if (!__any_sync(0xffffffffu, lrows > t * TR)) continue;
                    const int Fp = lrows > t * TR ? s_fp[t * C + c] : 0;
                    replay_chunk<TR>(s_rec, C, c, t * TR, lrows, Fp, cn, npad, g, K);
                }
                if (c < C) s_k[c] = K;
                PT_MARK(a.pt, 11, warp == nsub && lane == 0 && pass == 0);
                dw_mbar_arrive(bars + NT);
            }
        }
        if (!staged) stage_wait();
        return;
    }

    // =============================== substitution warps ===============================
    const int gq = lane >> 2, tq = lane & 3;
    const int c = warp * G + gq;                                          // column slot in the CTA
    const double delta = SAFE ? a.delta[0] : 0.0;
    const double Pb = SAFE ? diag_panel_sum(a) : 0.0;
    int pass = 0;
    for (int64_t cb = int64_t(blockIdx.x) * C; cb < ncols; cb += cstride, pass++) {
        const int64_t q = cb + c;
        const bool valid = q < ncols;
        const int64_t j = a.c0 + (valid ? q : 0);
        T sh = valid ? a.shifts[j * a.sstride] : ST::zero();              // (the pass's loads together)
        const double Gj0 = (SAFE && valid) ? a.G[j] : 0.0;
        const int64_t r = valid ? ((OP == 0 && a.rowend) ? a.rowend[j] : a.m) : 0;
        const bool active = valid && r > a.lo;
        if (SAFE && valid && !active && tq == 0) a.dblk[j] = 0;           // inactive column: no rescale
        if (SAFE && tq == 0) {                                             // (kept for the finish)
            s_gj[c] = Gj0;
            s_ej[c] = valid ? a.e[j] : 0;
        }
        const int nrow = active ? (OP == 0 ? int((a.hi < r ? a.hi : r) - a.lo) : nfull) : 0;
        int nmax = nrow;
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) nmax = max(nmax, __shfl_xor_sync(0xffffffffu, nmax, o));
        if (!active) sh = ST::zero();
        if (OP == 1) sh = ST::conj(sh);
        T *x = a.B + j * a.ldb;
        T *xs = GSCR ? a.Xscr + j * a.ldscr
                     : reinterpret_cast<T *>(smem_raw + diagl_scr_offset(npad, int(sizeof(T)), C, SAFE)) +
                           c * diagl_scr_ld(npad, int(sizeof(T)));         // -x of the solved rows
        auto rowof = [&](int sc) -> int64_t { return OP == 0 ? a.lo + sc : a.hi - 1 - sc; };
        auto pivot = [&](int sc) -> T {                                    // d_l = U(l,l) - s_j
            T dd = sc < nrow ? ST::sub(dg[sc], sh) : ST::real(1.0);
            if (SAFE && ST::is_zero(dd)) dd = ST::real(delta);
            return dd;
        };

        bool guarded = false;
        double g0 = 0.0;
        if (SAFE) {
            // ---- precheck with upper bounds (see the header) ----
            double prod = 1.0, minv = 0.0;
            for (int sc = tq; sc < nrow; sc += 4) {
                const double inv = rcp_up(maxabs(pivot(sc)));             // >= 1/|d_l|
                prod = __dmul_ru(prod, __dadd_ru(1.0, __dmul_ru(cn[sc], inv)));
                minv = fmax(minv, inv);
            }
            prod = dl_gprod_ru<4>(prod);
            minv = dl_gmax<4>(minv);
            const double gtop = active ? __dmul_ru(Gj0, 1.0 + 0x1p-40) : 0.0;      // >= ||y(I1)||_inf
            const double gfin = __dmul_ru(gtop, prod);
            guarded = active && !(gfin < kOmega && __dmul_ru(gfin, minv) < kOmega);
            if (__any_sync(0xffffffffu, guarded)) {                        // g := ||y(I1)||_inf
                for (int sc = tq; sc < nrow; sc += 4) g0 = fmax(g0, modv(x[rowof(sc)]));
                g0 = dl_gmax<4>(g0);
            }
            if (tq == 0) {                                                 // the replay's inputs
                s_g0[c] = g0;
                s_lrows[c] = guarded ? nrow : 0;
            }
        }
        PT_MARK(a.pt, 4, tid == 0 && pass == 0);
        if (!staged) stage_wait();
        PT_MARK(a.pt, 5, tid == 0 && pass == 0);

        const bool rec = SAFE && __any_sync(0xffffffffu, guarded);        // warp-uniform
        int F = 0;                                                         // this column's frame
        double axm = 0.0;                                                  // max |x|, frame F
        bool nonfinite = false;
        T py0 = ST::zero(), py1 = ST::zero();                              // next tile's right-hand sides
        {
            const int r0 = (NT - 1) * TR + 2 * tq;
            py0 = r0 < nrow ? x[rowof(r0)] : ST::zero();
            py1 = r0 + 1 < nrow ? x[rowof(r0 + 1)] : ST::zero();
        }
#pragma unroll 1
        for (int u = NT - 1; u >= 0; u--) {
            const int r0 = u * TR + 2 * tq;                                // this lane's rows r0, r0 + 1
            T y0 = py0, y1 = py1;                                          // (loaded one tile ahead)
            if (u > 0) {                                                   // prefetch the next tile's rows
                py0 = r0 - TR < nrow ? x[rowof(r0 - TR)] : ST::zero();
                py1 = r0 - TR + 1 < nrow ? x[rowof(r0 - TR + 1)] : ST::zero();
            }
            if (u * TR < nmax) {                                           // warp-uniform
                if (F != 0) {                                              // into the column's frame
                    y0 = dl_scale1(y0, -F);
                    y1 = dl_scale1(y1, -F);
                }
                // ---- left-looking update by the solved tiles (DMMA): y += U(tile u, k) (-x_k) ----
                {
                    // k-step pair of solved tile w: rows 8w + tq (set a) and 8w + 4 + tq (set b) of -x;
                    // U(8u + gq, 8w + r) sits at padtri_off(8w + r, 8) = 32 w (w + 1) + 8 r (w + 1) + row,
                    // which grows by 64 (w + 1) + 8 r from one w to the next
                    T b0 = ST::zero(), b1 = ST::zero();                    // second accumulator set
                    const T *ua_p = pk + u * TR + gq + padtri_off((u + 1) * TR + tq, TR);
                    const T *ub_p = pk + u * TR + gq + padtri_off((u + 1) * TR + 4 + tq, TR);
                    const T *xa_p = xs + (u + 1) * TR + tq;
                    int stp_a = 64 * (u + 2) + 8 * tq, stp_b = stp_a + 32;
                    if constexpr (GSCR) {
                        // scratch in L2: loads run 4 k-step pairs ahead of their DMMAs
                        constexpr int PD = 4;
                        const int nw = NT - 1 - u;
                        T ra[PD], rb[PD];
#pragma unroll
                        for (int i = 0; i < PD; i++) {
                            ra[i] = i < nw ? xa_p[TR * i] : ST::zero();
                            rb[i] = i < nw ? xa_p[TR * i + 4] : ST::zero();
                        }
#pragma unroll 1
                        for (int w0 = 0; w0 < nw; w0 += PD) {
#pragma unroll
                            for (int i = 0; i < PD; i++) {
                                if (w0 + i < nw) {
                                    const T nxa = ra[i], nxb = rb[i];
                                    if (w0 + i + PD < nw) {
                                        ra[i] = xa_p[TR * (w0 + i + PD)];
                                        rb[i] = xa_p[TR * (w0 + i + PD) + 4];
                                    }
                                    const T ua = *ua_p, ub = *ub_p;
                                    dl_kstep<T, CONJ>(y0, y1, nxa, ua);
                                    dl_kstep<T, CONJ>(b0, b1, nxb, ub);
                                    ua_p += stp_a;
                                    ub_p += stp_b;
                                    stp_a += 64;
                                    stp_b += 64;
                                }
                            }
                        }
                    } else
#pragma unroll 2
                    for (int w = u + 1; w < NT; w++) {
                        DW_CHECK(ua_p == pk + u * TR + gq + padtri_off(w * TR + tq, TR) &&
                                 ub_p == pk + u * TR + gq + padtri_off(w * TR + 4 + tq, TR) &&
                                 xa_p == xs + w * TR + tq && w * TR + 4 + tq < npad, "diagl k-step operands");
                        const T nxa = xa_p[0], nxb = xa_p[4];
                        const T ua = *ua_p, ub = *ub_p;
                        dl_kstep<T, CONJ>(y0, y1, nxa, ua);
                        dl_kstep<T, CONJ>(b0, b1, nxb, ub);
                        xa_p += TR;
                        ua_p += stp_a;
                        ub_p += stp_b;
                        stp_a += 64;
                        stp_b += 64;
                    }
                    y0 = ST::fnms(y0, ST::real(-1.0), b0);                 // y + b (exact: -(-1) b)
                    y1 = ST::fnms(y1, ST::real(-1.0), b1);
                }
                // ---- the tile's own rows, one by one (P:82 / P:297, P:84 / P:315) ----
                Piv<T> p0, p1;
                p0.make(pivot(r0));
                p1.make(pivot(r0 + 1));
                const T *tb = pk + padtri_off(u * TR, TR) + r0;           // column 8u, rows r0, r0 + 1
                const int tstride = TR * (u + 1);                          // padded column length
#pragma unroll
                for (int n = TR - 1; n >= 0; n--) {
                    const T *cu = tb + n * tstride;                        // U(r0 + {0,1}, 8u + n), zero for row >= 8u + n
                    const T u0 = CONJ ? ST::conj(cu[0]) : cu[0], u1 = CONJ ? ST::conj(cu[1]) : cu[1];   // (loads first)
                    const T qv = (n & 1) ? p1.apply(y1) : p0.apply(y0);
                    const T xl = group_shfl<T, 4>(qv, n >> 1);
                    y0 = ST::fnms(y0, xl, u0);
                    y1 = ST::fnms(y1, xl, u1);
                }
                T x0 = p0.apply(y0), x1 = p1.apply(y1);                    // = the shuffled values
                const double ax0 = modv(x0), ax1 = modv(x1);
                if (rec) {
                    DW_CHECK(r0 + 1 < npad && c < C, "diagl record row");
                    nonfinite |= !(ax0 <= 1.7976931348623157e308) || !(ax1 <= 1.7976931348623157e308);
                    s_rec[r0 * C + c] = ax0;
                    s_rec[(r0 + 1) * C + c] = ax1;
                    if (tq == 0) s_fp[u * C + c] = F;
                    int em = max(bexp(ax0), bexp(ax1));
                    em = max(em, __shfl_xor_sync(0xffffffffu, em, 1, 4));
                    em = max(em, __shfl_xor_sync(0xffffffffu, em, 2, 4));
                    const bool need = guarded && em > 1623 && em < 2047;  // |x| >= 2^601: new frame
                    if (__any_sync(0xffffffffu, need)) {
                        const int s = need ? min(em - 1023, 1022) : 0;
                        if (s) {
                            const double p = pow2i(-s);
                            x0 = ST::fnms(ST::zero(), ST::real(-p), x0);   // x 2^-s (exact)
                            x1 = ST::fnms(ST::zero(), ST::real(-p), x1);
                            axm = __dmul_rn(axm, p);
                            for (int rr = (u + 1) * TR + tq; rr < npad; rr += 4)   // solved rows, same frame
                                xs[rr] = dl_scale1(xs[rr], -s);
                            F += s;
                        }
                    }
                }
                axm = fmax(axm, fmax(modv(x0), modv(x1)));
                if (valid) {
                    xs[r0] = ST::neg(x0);
                    xs[r0 + 1] = ST::neg(x1);
                }
            } else if (valid) {                                            // beyond every row: zeros
                xs[r0] = ST::zero();
                xs[r0 + 1] = ST::zero();
            }
            __syncwarp();                                                  // scratch rows seen by the column's lanes
            if constexpr (SAFE) dw_mbar_arrive(bars + u);
        }
        PT_MARK(a.pt, 6, tid == 0 && pass == 0);
        nonfinite |= __shfl_xor_sync(0xffffffffu, nonfinite, 1, 4);
        nonfinite |= __shfl_xor_sync(0xffffffffu, nonfinite, 2, 4);
        const bool failed = SAFE && guarded && (nonfinite || a.force_fb);

        int kt = 0;
        if (SAFE) {
            dw_mbar_wait(bars + NT, pass & 1);                             // K from the replay warp
            kt = s_k[c];
        }
        PT_MARK(a.pt, 7, tid == 0 && pass == 0);
        // ---- steps (ii), (iii) and the output rows in the paper's frame 2^(F - K - k3) ----
        {
            int k3 = 0;
            if (SAFE) {
                int ej = 0;
                double Gj = 0.0;
                if (active) { ej = s_ej[c]; Gj = s_gj[c]; }
                if (kt > 0) {                                              // P:376-386, step (ii)
                    ej -= kt;
                    Gj = mulp2n(Gj, kt);
                }
                const double xm = mulp2_any(dl_gmax<4>(axm), F - kt);     // max |x(I1)|, paper frame
                Gj = __dadd_rn(Gj, __dmul_rn(Pb, xm));
                if (Gj >= kOmega) {
                    k3 = minpow2_bits(Gj, kOmega);
                    ej -= k3;
                    Gj = mulp2n(Gj, k3);
                }
                if (active && tq == 0 && !failed) {
                    a.e[j] = ej;
                    a.G[j] = Gj;
                    a.dblk[j] = -(kt + k3);
                    a.Etab[a.b * a.n + j] = ej;
                }
                if (active && !failed) pair_fix(a, j, -(kt + k3), ej, tq, 4);
            }
            const int sfin = F - kt - k3;
            if (valid && !failed) {
                double *xsum = nullptr;
                if constexpr (ST::cplx_) xsum = a.Xsum ? a.Xsum + j * a.ldxs : nullptr;
                for (int sc = tq; sc < nfull; sc += 4) {
                    T v = sc < nrow ? ST::neg(xs[sc]) : ST::zero();
                    if (sfin != 0) {
                        if (sfin >= -1022 && sfin <= 1023) v = ST::fnms(ST::zero(), ST::real(-pow2i(sfin)), v);
                        else v = dl_scale1(v, sfin);
                    }
                    if (sc < nrow) x[rowof(sc)] = v;
                    if constexpr (ST::cplx_) {
                        if (xsum) xsum[rowof(sc) - a.lo] = __dadd_rn(v.x, v.y);   // 3M operand sums (§7.2)
                    }
                }
            }
        }
        PT_MARK(a.pt, 8, tid == 0 && pass == 0);
        // ---- a column whose values stopped being finite (tiny pivots: growth beyond the frame's
        //      headroom inside one tile) is rerun from its inputs by the synchronous guarded loop,
        //      Alg. 4 step by step, one warp per column ----
        if (SAFE) {
            unsigned fm = __ballot_sync(0xffffffffu, failed && tq == 0);
            while (fm) {
                const int fl = __ffs(fm) - 1;
                fm &= fm - 1;
                const int64_t jf = __shfl_sync(0xffffffffu, j, fl);
                const int nrf = __shfl_sync(0xffffffffu, nrow, fl);
                const double g0f = __shfl_sync(0xffffffffu, g0, fl);
                T shf;
                if constexpr (ST::cplx_)
                    shf = make_double2(__shfl_sync(0xffffffffu, sh.x, fl), __shfl_sync(0xffffffffu, sh.y, fl));
                else
                    shf = __shfl_sync(0xffffffffu, sh, fl);
                T *xf = a.B + jf * a.ldb;
                constexpr int RF = 128 / 32;
                T yf[RF];
#pragma unroll
                for (int t = 0; t < RF; t++) {
                    const int sc = lane + 32 * t;
                    yf[t] = sc < nrf ? xf[rowof(sc)] : ST::zero();
                }
                auto pivot_f = [&](int sc) -> T {
                    T dd = sc < nrf ? ST::sub(dg[sc], shf) : ST::real(1.0);
                    if (ST::is_zero(dd)) dd = ST::real(delta);
                    return dd;
                };
                const UAcc<T, false, CONJ> ua{pk, nullptr, cn, nullptr, ST::zero(), 0.0};
                double g = g0f;
                int ktf = 0;
                diag_rows<T, 32, RF, true, TR>(yf, pivot_f, ua, lane, nrf, nrf, true, g, ktf);
                int ej = a.e[jf];
                double Gj = a.G[jf];
                if (ktf > 0) {
                    ej -= ktf;
                    Gj = mulp2n(Gj, ktf);
                }
                double xm = 0.0;
#pragma unroll
                for (int t = 0; t < RF; t++) xm = fmax(xm, modv(yf[t]));
                xm = dl_gmax<32>(xm);
                Gj = __dadd_rn(Gj, __dmul_rn(Pb, xm));
                int k3 = 0;
                if (Gj >= kOmega) {
                    k3 = minpow2_bits(Gj, kOmega);
                    scale_all<false>(yf, k3);
                    ej -= k3;
                    Gj = mulp2n(Gj, k3);
                }
                if (lane == 0) {
                    a.e[jf] = ej;
                    a.G[jf] = Gj;
                    a.dblk[jf] = -(ktf + k3);
                    a.Etab[a.b * a.n + jf] = ej;
                }
                pair_fix(a, jf, -(ktf + k3), ej, lane, 32);
                double *xsum = nullptr;
                if constexpr (ST::cplx_) xsum = a.Xsum ? a.Xsum + jf * a.ldxs : nullptr;
#pragma unroll
                for (int t = 0; t < RF; t++) {
                    const int sc = lane + 32 * t;
                    if (sc < nrf) xf[rowof(sc)] = yf[t];
                    if constexpr (ST::cplx_) {
                        if (xsum && sc < nfull) xsum[rowof(sc) - a.lo] = __dadd_rn(yf[t].x, yf[t].y);
                    }
                }
            }
        }
    }
    if (!staged) stage_wait();
    PT_MARK(a.pt, 9, tid == 0);
    PT_MARK(a.pt, 15, tid == 0);
}

}  // namespace mstrsm
