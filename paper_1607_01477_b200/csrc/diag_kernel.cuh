// diag_kernel.cuh -- a.3 diagonal-block multi-shift (safe) solve + a.4 column bound.
//
// For one block I1 and every active column j (P:170-175 / P:371-388):
//   plain:  Alg. 1 on U(I1,I1) - s_j I
//   safe :  Alg. 4 on U(I1,I1) - s_j I with block-local bounds (R5):
//           precheck (eqs. 4-5) -> Trsv, else the guarded loop with
//           power-of-two rescales (R2); then step (ii) e_j -= kt, step (iii)
//           G_j += P_b max|x(I1)| and rescale if >= Omega.
// The rescale of rows outside I1 is LAZY: d_j = total exponent change of this block is handed to
// the GEMM epilogue (rows I0, still pending) and E[b][j] = e_j records the frame of the rows
// finalised here (rows I2 are fixed up once at the end by finalize_kernel).
//
// Layout.  A warp holds G = 32/LPC columns; LPC lanes share one column and lane r of a group
// owns the solve rows sc = r + LPC*t, t < RPL (LPC*RPL >= n_b).  The per-row scalar chain of
// Alg. 4 (|y_l|, the division, |x_l|, the bound checks) is therefore executed once per group and
// serves G columns per warp instruction, while the substitution within the block is spread over
// the LPC lanes.  The diagonal block is staged once per CTA in shared memory as a packed
// strictly-upper triangle in "solve coordinates" sc (op N: sc = row - lo; op C: sc = hi-1-row,
// the flip of R9), so one loop serves back substitution (op N) and forward substitution with
// L = U^H (op C).  Persistent CTAs loop over column groups.
#pragma once
#include "common.cuh"

namespace mstrsm {

template <typename T>
struct DiagArgs {
    const T *U; int64_t ldu, m;
    const T *shifts; int64_t sstride;
    T *B; int64_t ldb;
    int64_t c0, ncols, n;          // columns [c0, c0 + ncols) of an n-column solve
    const int64_t *rowend;         // device, nullable (op N only)
    int64_t lo, hi, b;             // block b = rows [lo, hi)
    const double *cnl;             // block-local column norms, indexed by global row
    const double *P;               // panel sums, P[b]
    const double *delta;           // device scalar (R4)
    double *G; int *e; int *dblk; int *Etab;
};

__host__ __device__ inline int64_t diag_smem_bytes(int nfull, int esize) {
    int64_t pk = int64_t(nfull) * (nfull - 1) / 2 + 128;
    return pk * esize + int64_t(nfull) * esize + int64_t(nfull) * 8;
}

// 1/d for the division x = y/d, computed once per row and group (Smith's scaling, R7).
template <typename T> struct Recip;
template <> struct Recip<double> {
    double v;
    __device__ __forceinline__ void make(double d) { v = d; }
    __device__ __forceinline__ double apply(double y) const { return __ddiv_rn(y, v); }   // exact IEEE division
};
template <> struct Recip<cplx> {
    double r, inv; bool sw;
    __device__ __forceinline__ void make(cplx d) {
        sw = fabs(d.y) > fabs(d.x);
        if (!sw) { r = __ddiv_rn(d.y, d.x); inv = __drcp_rn(__dadd_rn(d.x, __dmul_rn(d.y, r))); }
        else { r = __ddiv_rn(d.x, d.y); inv = __drcp_rn(__dadd_rn(d.y, __dmul_rn(d.x, r))); }
    }
    // Smith's numerators times the rounded reciprocal of the denominator (<= 1.5 ulp from the
    // oracle's Smith quotient; R24 covers the difference).
    __device__ __forceinline__ cplx apply(cplx a) const {
        if (!sw) return make_double2(__dmul_rn(__dadd_rn(a.x, __dmul_rn(a.y, r)), inv),
                                     __dmul_rn(__dsub_rn(a.y, __dmul_rn(a.x, r)), inv));
        return make_double2(__dmul_rn(__dadd_rn(__dmul_rn(a.x, r), a.y), inv),
                            __dmul_rn(__dsub_rn(__dmul_rn(a.y, r), a.x), inv));
    }
};

// 2^k as a double for -1022 <= k <= 1023 (exact, built from the exponent bits).
__device__ __forceinline__ double pow2i(int k) { return __longlong_as_double((long long)(1023 + k) << 52); }
__device__ __forceinline__ double maxabs(double v) { return fabs(v); }
__device__ __forceinline__ double maxabs(cplx v) { return fmax(fabs(v.x), fabs(v.y)); }
__device__ __forceinline__ double scale_pw(double v, double p) { return __dmul_rn(v, p); }
__device__ __forceinline__ cplx scale_pw(cplx v, double p) { return make_double2(__dmul_rn(v.x, p), __dmul_rn(v.y, p)); }

template <int LPC>
__device__ __forceinline__ double group_max(double v) {
#pragma unroll
    for (int o = 1; o < LPC; o <<= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o, LPC));
    return v;
}

template <typename T, int LPC>
__device__ __forceinline__ T group_shfl(T v, int src) {
    if constexpr (S<T>::cplx_)
        return make_double2(__shfl_sync(0xffffffffu, v.x, src, LPC), __shfl_sync(0xffffffffu, v.y, src, LPC));
    else
        return __shfl_sync(0xffffffffu, v, src, LPC);
}

template <typename T, int LPC, int RPL, bool SAFE, int OP>
__global__ void __launch_bounds__(512) diag_kernel(DiagArgs<T> a) {
    typedef S<T> ST;
    constexpr int G = 32 / LPC;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int nfull = int(a.hi - a.lo);
    const int64_t npk = int64_t(nfull) * (nfull - 1) / 2 + 128;
    T *pk = reinterpret_cast<T *>(smem_raw);
    T *dg = pk + npk;
    double *cn = reinterpret_cast<double *>(dg + nfull);

    // ---- stage U(I1,I1) (packed, solve coordinates), its diagonal and cnl ----
    const int tid = threadIdx.x, nth = blockDim.x;
    {
        for (int idx = tid; idx < nfull * 128; idx += nth) {       // any blockDim
            const int cq = idx >> 7, rl = idx & 127;
            if (rl < cq) {
                if (OP == 0) {      // U~(i,c) = U(lo+i, lo+c)
                    pk[int64_t(cq) * (cq - 1) / 2 + rl] = a.U[(a.lo + rl) + (a.lo + cq) * a.ldu];
                } else {            // U~(i,c) = conj(U(hi-1-c, hi-1-i)); U column lo+cq, row lo+rl
                    int ci = nfull - 1 - cq, cc = nfull - 1 - rl;
                    pk[int64_t(cc) * (cc - 1) / 2 + ci] = ST::conj(a.U[(a.lo + rl) + (a.lo + cq) * a.ldu]);
                }
            }
        }
        for (int c = tid; c < nfull; c += nth) {
            int64_t row = OP == 0 ? a.lo + c : a.hi - 1 - c;
            T u = a.U[row + row * a.ldu];
            dg[c] = OP == 0 ? u : ST::conj(u);
            cn[c] = SAFE ? a.cnl[row] : 0.0;
        }
    }
    __syncthreads();

    const int lane = tid & 31, grp = lane / LPC, rl = lane % LPC;
    const int64_t wid = (int64_t(blockIdx.x) * nth + tid) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * nth) >> 5;
    const double delta = SAFE ? *a.delta : 0.0;
    const double Pb = SAFE ? a.P[a.b] : 0.0;

    for (int64_t base = wid * G; base < a.ncols; base += nw * G) {
        const int64_t q = base + grp;
        const bool valid = q < a.ncols;
        const int64_t j = a.c0 + (valid ? q : 0);
        const int64_t r = valid ? ((OP == 0 && a.rowend) ? a.rowend[j] : a.m) : 0;
        const bool active = valid && r > a.lo;
        if (SAFE && valid && !active && rl == 0) a.dblk[j] = 0;     // inactive column: no rescale
        const int nrow = active ? (OP == 0 ? int((a.hi < r ? a.hi : r) - a.lo) : nfull) : 0;
        int nmax = nrow;
#pragma unroll
        for (int o = LPC; o < 32; o <<= 1) nmax = max(nmax, __shfl_xor_sync(0xffffffffu, nmax, o));
        if (nmax == 0) continue;                                      // warp-uniform
        T sh = active ? a.shifts[j * a.sstride] : ST::zero();
        if (OP == 1) sh = ST::conj(sh);
        T *x = a.B + j * a.ldb;
        auto rowof = [&](int sc) -> int64_t { return OP == 0 ? a.lo + sc : a.hi - 1 - sc; };
        auto dof = [&](int sc) -> T {
            T dd = ST::sub(dg[sc], sh);
            if (SAFE && ST::is_zero(dd)) dd = ST::real(delta);
            return dd;
        };

        bool guarded = false;
        double g = 0.0;
        if (SAFE) {
            // ---- precheck, eqs. (4)-(5), in the oracle's order:
            //      M = max_l g_l/|d_l|,  g_{l-1} = g_l * (1 + cnl_l/|d_l|),  g_top = ||y(I1)||_inf ----
            double g0 = 0.0;
#pragma unroll
            for (int t = 0; t < RPL; t++) {
                int sc = rl + LPC * t;
                if (sc < nrow) g0 = fmax(g0, ST::mod(x[rowof(sc)]));
            }
            g0 = group_max<LPC>(g0);
            double ad[RPL], tf[RPL], gb[RPL];
#pragma unroll
            for (int t = 0; t < RPL; t++) {
                int sc = rl + LPC * t;
                ad[t] = 1.0; tf[t] = 1.0; gb[t] = 0.0;
                if (sc < nrow) {
                    ad[t] = ST::mod(dof(sc));
                    tf[t] = __dadd_rn(1.0, __ddiv_rn(cn[sc], ad[t]));
                }
            }
            double gg = g0;
            for (int sc = nmax - 1; sc >= 0; sc--) {
                const int t = sc / LPC, rr = sc % LPC;
                double own = 1.0;
#pragma unroll
                for (int t2 = 0; t2 < RPL; t2++)
                    if (t2 == t) own = tf[t2];
                double tfv = __shfl_sync(0xffffffffu, own, rr, LPC);
                if (sc < nrow) {
#pragma unroll
                    for (int t2 = 0; t2 < RPL; t2++)
                        if (t2 == t && rl == rr) gb[t2] = gg;
                    gg = __dmul_rn(gg, tfv);
                }
            }
            double M = 0.0;
#pragma unroll
            for (int t = 0; t < RPL; t++)
                if (rl + LPC * t < nrow) M = fmax(M, __ddiv_rn(gb[t], ad[t]));
            M = group_max<LPC>(M);
            guarded = active && !(M < kOmega && gg < kOmega);
            g = g0;
        }

        T y[RPL];
#pragma unroll
        for (int t = 0; t < RPL; t++) {
            int sc = rl + LPC * t;
            y[t] = sc < nrow ? x[rowof(sc)] : ST::zero();
        }

        // ---- Trsv / guarded loop over solve rows sc = nmax-1 .. 0 ----
        // Rescales "y := t y" of the guarded loop are applied LAZILY to the rows
        // held in registers: y[] lives in a frame 2^pend above the true (oracle) frame; the
        // chain values are brought to the true frame exactly (power-of-two scaling commutes
        // with rounding), and the registers are flushed once pend reaches 12 bits, which keeps
        // |y|, |x u| below DBL_MAX for max|U| <= 2^40 (R8).
        // The step loop is a runtime loop (compact code: the I-cache, not the ALUs, bounded an
        // unrolled version); the lane-local row slot t = sc / LPC is selected with predicates.
        int kt = 0, pend = 0;
        for (int sc = nmax - 1; sc >= 0; sc--) {
            const int t = sc / LPC, rr = sc % LPC;
            T own = ST::zero();
#pragma unroll
            for (int t2 = 0; t2 < RPL; t2++)
                if (t2 == t) own = y[t2];
            T yl = group_shfl<T, LPC>(own, rr);
            if (sc < nrow) {
                T dl = dof(sc);
                Recip<T> rd;
                rd.make(dl);
                T xl;
                if (SAFE && guarded) {
                    if (pend) yl = scale_pw(yl, pow2i(-pend));         // true frame (exact)
                    xl = rd.apply(yl);                                 // P:297 diagonal step
                    // P:282-295 (R8): |y_l| >= Omega |d_l|.  Cheap conservative pre-test:
                    // |y| <= 1.4143 max|y_c|, |d| >= max|d_c|.
                    if (!(1.5 * maxabs(yl) < kOmega * maxabs(dl))) {
                        double ay = ST::mod(yl), lim = __dmul_rn(kOmega, ST::mod(dl));
                        if (ay >= lim) {
                            int k = minpow2(ay, lim);
                            pend += k;
                            yl = ST::ldx(yl, -k);
                            xl = rd.apply(yl);
                            kt += k;
                            g = ldexp(g, -k);
                        }
                    }
                    double M = ST::mod(xl);
                    g = __dadd_rn(g, __dmul_rn(M, cn[sc]));
                    if (g >= kOmega) {
                        int k = minpow2(g, kOmega);
                        pend += k;
                        xl = ST::ldx(xl, -k);
                        kt += k;
                        g = ldexp(g, -k);
                    }
                    if (pend >= 12) {                                  // flush registers -> true frame
                        if (pend < 1000) {
                            double p = pow2i(-pend);
#pragma unroll
                            for (int t2 = 0; t2 < RPL; t2++) y[t2] = scale_pw(y[t2], p);
                        } else {
#pragma unroll
                            for (int t2 = 0; t2 < RPL; t2++) y[t2] = ST::ldx(y[t2], -pend);
                        }
                        pend = 0;
                    } else if (pend) {
                        xl = scale_pw(xl, pow2i(pend));                // register frame for the update
                    }
                } else {
                    xl = rd.apply(yl);                                 // P:297 / P:82
                }
                // owner stores x_l; substitution within the block (P:315 / P:84): rows sc' < sc
                const T *col = pk + int64_t(sc) * (sc - 1) / 2;
#pragma unroll
                for (int t2 = 0; t2 < RPL; t2++) {
                    int i = rl + LPC * t2;
                    if (i < sc) y[t2] = ST::fnms(y[t2], xl, col[i]);
                    else if (i == sc) y[t2] = xl;
                }
            }
        }
        if (SAFE && pend) {
#pragma unroll
            for (int t2 = 0; t2 < RPL; t2++) y[t2] = ST::ldx(y[t2], -pend);
        }

        if (SAFE) {
            int ej = 0;
            double Gj = 0.0;
            if (active) { ej = a.e[j]; Gj = a.G[j]; }
            if (kt > 0) {                                              // P:376-386, step (ii)
                ej -= kt;
                Gj = ldexp(Gj, -kt);
            }
            double xm = 0.0;
#pragma unroll
            for (int t = 0; t < RPL; t++) xm = fmax(xm, ST::mod(y[t]));
            xm = group_max<LPC>(xm);
            Gj = __dadd_rn(Gj, __dmul_rn(Pb, xm));
            int k3 = 0;
            if (Gj >= kOmega) {
                k3 = minpow2(Gj, kOmega);
#pragma unroll
                for (int t = 0; t < RPL; t++) y[t] = ST::ldx(y[t], -k3);
                ej -= k3;
                Gj = ldexp(Gj, -k3);
            }
            if (active && rl == 0) {
                a.e[j] = ej;
                a.G[j] = Gj;
                a.dblk[j] = -(kt + k3);
                a.Etab[a.b * a.n + j] = ej;
            }
        }
#pragma unroll
        for (int t = 0; t < RPL; t++) {
            int sc = rl + LPC * t;
            if (sc < nrow) x[rowof(sc)] = y[t];
        }
    }
}

}  // namespace mstrsm
