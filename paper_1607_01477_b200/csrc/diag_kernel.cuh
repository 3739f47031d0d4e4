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
// Layout.  A warp holds G = 32/LPC columns; LPC lanes share one column and lane r of a group owns
// the solve rows sc = r + LPC*t, t < RPL (LPC*RPL >= n_b), in registers.  The row loop is
// "for t = RPL-1..0 (unrolled) for r = LPC-1..0 (runtime)", so every register slot index is a
// compile-time constant and row sc's update touches only the slots t2 <= t that still hold
// unsolved rows.  The diagonal block is staged once per CTA in shared memory as a packed strictly
// upper triangle in "solve coordinates" sc (op N: sc = row - lo; op C: sc = hi-1-row, the flip of
// R9), so one loop serves back substitution (op N) and forward substitution with L = U^H (op C).
// Persistent CTAs loop over column groups.
//
// Per-row pivot data (1/d_l, Omega*|d_l|) depend only on the shift, not on the running solution,
// so every lane precomputes them for its own rows before the loop and the sequential chain only
// shuffles them.  In the guarded loop the solution lives in a register frame 2^pend above the
// true (paper) frame: a rescale "y := 2^-k y" only adds k to pend, which leaves
// the register values -- and therefore the substitution -- untouched; the registers are brought
// back to the true frame once pend reaches 12 bits.  The bound chain (|y_l|, |x_l|, g, the
// rescale exponents) is branch-free and runs beside the substitution instead of in front of it.
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
    int *fb_list; int *fb_count;   // columns handed to the synchronous fallback (safe variants)
    int force_fb;                  // testing: hand every guarded column to the fallback
    int early;                     // U / cnl may be staged before waiting for the preceding grid
    int nsub;                      // diagw_kernel: substitution warps per CTA (set by the launcher)
    T *Xscr; int64_t ldscr;        // diagl_kernel: per-column scratch of the solved rows (n_b rounded to 8 x n)
    const double *Ppart;           // nullable: P_b = sum of Ppart[k], k in [lo, hi) ascending (else P[b])
    // generalized solve (Alg. 7/8, op N): V with its norms, and the output C = -lambda_j X(I1,j)
    // (n_b x n, column j at Cbuf + j * ldc) that the V product of the update reads
    const T *V; int64_t ldv;
    const double *cnlV, *PV, *deltaV;
    T *Cbuf; int64_t ldc;
    // complex 3M update (nullable): Re + Im of the finished rows I1, Xsum[(row - lo) + j * ldxs]
    double *Xsum; int64_t ldxs;
    // paired blocks (the merged update; nullable): this block is the second of a pair
    // whose first block p = rows [plo, phi), columns from c0prev, solved just before it, wrote its
    // exponent deltas to dprev; xsprev = p's X+ rows (ld ldxs, complex 3M only)
    const int *dprev; int64_t c0prev, plo, phi, bprev;
    double *xsprev;
    long long *pt;                 // phase times (MSTRSM_PHASE_TIMES builds only; nullable)
    int trig;                      // diagl_kernel: let the next grid launch at this one's start
};

template <typename T> struct DiagArgs;
// P_b of the block (R6): the precomputed panel sum, or -- when the multi-GPU path fed the
// panels one by one -- the ascending sum of the panel's per-column maxima (as panel_sum_kernel)
template <typename T>
__device__ __forceinline__ double diag_panel_sum(const DiagArgs<T> &a) {
    if (!a.Ppart) return a.P[a.b];
    double s = 0.0;
    for (int64_t k = a.lo; k < a.hi; k++) s = __dadd_rn(s, a.Ppart[k]);
    return s;
}

// Offset of column l of the padded triangle with chunks of lpc rows (column l holds
// lpc (floor(l/lpc) + 1) elements: rows 0 .. l-1 of U and zeros to the end of l's chunk).
__host__ __device__ __forceinline__ int64_t padtri_off(int l, int lpc) {
    const int64_t t = l / lpc, r = l % lpc;
    return int64_t(lpc) * lpc * t * (t + 1) / 2 + r * lpc * (t + 1);
}

// Shared memory: the packed strictly upper triangle, the diagonal and cnl (generalized: the same
// three for V as well).
__host__ __device__ inline int64_t diag_smem_bytes(int nfull, int esize, bool gen = false) {
    int64_t pk = int64_t(nfull) * (nfull - 1) / 2 + 128;
    return (gen ? 2 : 1) * (pk * esize + int64_t(nfull) * esize + int64_t(nfull) * 8);
}

// Threads per CTA of an instantiation (its __launch_bounds__): 12 warps when each lane holds 16
// rows (up to 168 registers), 14 warps when it holds 8 (up to 146).
template <typename T, int RPL> struct DiagThreads {
#ifndef MSTRSM_DIAG_T16
#define MSTRSM_DIAG_T16 384
#endif
    static constexpr int value = RPL >= 16 ? MSTRSM_DIAG_T16 : 448;
};

// 2^k as a double for -1022 <= k <= 1023 (exact, built from the exponent bits).
__device__ __forceinline__ double pow2i(int k) { return __longlong_as_double((long long)(1023 + k) << 52); }
// v * 2^-k for k >= 0 as a product with an exact power of two: rounded exactly like ldexp(v, -k)
// for k <= 1022; beyond that (only after extreme rescales) two products, which can differ from
// ldexp by the double rounding of a subnormal result.
__device__ __forceinline__ double mulp2n(double v, int k) {
    if (k <= 1022) return __dmul_rn(v, pow2i(-k));
    return __dmul_rn(__dmul_rn(v, pow2i(-1022)), pow2i(-min(k - 1022, 1022)));
}
__device__ __forceinline__ cplx mulp2n(cplx v, int k) { return make_double2(mulp2n(v.x, k), mulp2n(v.y, k)); }

// Paired blocks (merged update).  The update of the rows beyond a pair (p, b) of
// consecutive blocks is one GEMM with K = K_p + K_b, run after b's diagonal step:
//   C := 2^(d_p + d_b) C - U(., I_p) (2^d_b X_p) - U(., I_b) X_b,
// the same sum Alg. 5 forms with two GEMMs, 2^d_b (2^d_p C - U(., I_p) X_p) - U(., I_b) X_b, to
// rounding.  So when column j rescales in b's step (d_b = d < 0), X_p's rows (and its X+ rows)
// are scaled by 2^d in place -- exact powers of two -- and Etab(p, j) moves to b's frame e_j (the
// a.6 fix-up then scales them by 2^(e - E_bj) like b's rows), and dblk[j] (the merged update's
// factor) becomes d_p + d.  Called by the nl lanes of column j's group (lane < nl) after the
// step's e_j / dblk writes, for an active column.
template <typename T>
__device__ __forceinline__ void pair_fix(const DiagArgs<T> &a, int64_t j, int d, int ej, int lane, int nl) {
    if (!a.dprev) return;
    const bool inp = j >= a.c0prev;                  // (columns before p's range: X_p = 0, d_p = 0)
    if (lane == 0) a.dblk[j] = d + (inp ? a.dprev[j] : 0);
    if (d == 0 || !inp) return;
    T *x = a.B + j * a.ldb;
    for (int64_t r = a.plo + lane; r < a.phi; r += nl) x[r] = mulp2n(x[r], -d);
    if (a.xsprev) {
        double *xs = a.xsprev + j * a.ldxs;
        for (int64_t r = lane; r < a.phi - a.plo; r += nl) xs[r] = mulp2n(xs[r], -d);
    }
    if (lane == 0) a.Etab[a.bprev * a.n + j] = ej;
}
// y := 2^-k y for a whole register array (one scale factor for all elements); k <= 1022 when
// SMALL, any k >= 0 otherwise.
template <bool SMALL, typename T, int N>
__device__ __forceinline__ void scale_all(T (&y)[N], int k) {
    const double p1 = SMALL || k <= 1022 ? pow2i(-k) : pow2i(-1022);
#pragma unroll
    for (int t = 0; t < N; t++) {
        if constexpr (S<T>::cplx_) y[t] = make_double2(__dmul_rn(y[t].x, p1), __dmul_rn(y[t].y, p1));
        else y[t] = __dmul_rn(y[t], p1);
    }
    if (!SMALL && k > 1022) {
        const double p2 = pow2i(-min(k - 1022, 1022));
#pragma unroll
        for (int t = 0; t < N; t++) {
            if constexpr (S<T>::cplx_) y[t] = make_double2(__dmul_rn(y[t].x, p2), __dmul_rn(y[t].y, p2));
            else y[t] = __dmul_rn(y[t], p2);
        }
    }
}
// v * 2^s for |s| <= 1074 as two exact power-of-two products.
__device__ __forceinline__ double mulp2s(double v, int s) {
    const int h = s / 2;
    return __dmul_rn(__dmul_rn(v, pow2i(h)), pow2i(s - h));
}
// v * 2^s for any integer s as (at most) three exact power-of-two products.
__device__ __forceinline__ double mulp2_any(double v, int s) {
    const int s1 = max(-1022, min(1023, s));
    const int s2 = max(-1022, min(1023, s - s1));
    const int s3 = max(-1022, min(1023, s - s1 - s2));
    return __dmul_rn(__dmul_rn(__dmul_rn(v, pow2i(s1)), pow2i(s2)), pow2i(s3));
}
template <typename T, int N>
__device__ __forceinline__ void scale_all_any(T (&y)[N], int s) {
    const int s1 = max(-1022, min(1023, s));
    const int s2 = max(-1022, min(1023, s - s1));
    const int s3 = max(-1022, min(1023, s - s1 - s2));
    const double p1 = pow2i(s1), p2 = pow2i(s2), p3 = pow2i(s3);
#pragma unroll
    for (int t = 0; t < N; t++) {
        if constexpr (S<T>::cplx_)
            y[t] = make_double2(__dmul_rn(__dmul_rn(__dmul_rn(y[t].x, p1), p2), p3),
                                __dmul_rn(__dmul_rn(__dmul_rn(y[t].y, p1), p2), p3));
        else y[t] = __dmul_rn(__dmul_rn(__dmul_rn(y[t], p1), p2), p3);
    }
}
__device__ __forceinline__ double maxabs(double v) { return fabs(v); }
__device__ __forceinline__ double maxabs(cplx v) { return fmax(fabs(v.x), fabs(v.y)); }

// |z| of R7 (prescaled sqrt(re^2 + im^2), no FMA) without branches; equal to S<cplx>::mod for
// finite z.
__device__ __forceinline__ double modv(double a) { return fabs(a); }
__device__ __forceinline__ double modv(cplx a) {
    double x = fabs(a.x), y = fabs(a.y), big = fmax(x, y);
    double s = big > 0x1p+500 ? 0x1p-600 : (big < 0x1p-500 ? 0x1p+600 : 1.0);
    double si = big > 0x1p+500 ? 0x1p+600 : (big < 0x1p-500 ? 0x1p-600 : 1.0);
    x = __dmul_rn(x, s);
    y = __dmul_rn(y, s);
    return __dmul_rn(__dsqrt_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y))), si);
}
// max_t modv(y[t]) (t < n, the others ignored), bit for bit, with one square root: for components
// in [2^-500, 2^500) modv is sqrt_rn(x^2 + y^2) (no prescale), a monotone function of the rounded
// sum, so the largest sum gives the largest modulus (non-negative doubles order like their bits);
// zeros add nothing; any other element takes modv itself.
template <int N>
__device__ __forceinline__ double modv_max(const cplx (&y)[N], int n_live) {
    long long qb = -1;
    double other = 0.0;
#pragma unroll
    for (int t = 0; t < N; t++) {
        if (t < n_live) {
            const unsigned hx = unsigned(__double2hiint(y[t].x)) & 0x7fffffffu;
            const unsigned hy = unsigned(__double2hiint(y[t].y)) & 0x7fffffffu;
            const unsigned hb = max(hx, hy);
            if ((hb >> 20) - 523u <= 999u) {
                const double q = __dadd_rn(__dmul_rn(y[t].x, y[t].x), __dmul_rn(y[t].y, y[t].y));
                qb = max(qb, __double_as_longlong(q));
            } else if ((hb | unsigned(__double2loint(y[t].x)) | unsigned(__double2loint(y[t].y))) != 0u) {
                other = fmax(other, modv(y[t]));
            }
        }
    }
    return qb >= 0 ? fmax(__dsqrt_rn(__longlong_as_double(qb)), other) : other;
}

// R2's minpow2(a, L) (smallest k >= 1 with 2^-k a < L) for positive a >= L from the exponent and
// mantissa bits: 2^-k a < L  <=>  k > e_a - e_L, or k = e_a - e_L with mant(a) < mant(L).
__device__ __forceinline__ void exp_mant(double x, int &e, long long &mnt) {
    long long b = __double_as_longlong(x);
    e = int(b >> 52);
    if (e == 0) { b = __double_as_longlong(__dmul_rn(x, 0x1p+64)); e = int(b >> 52) - 64; }   // subnormal
    mnt = b & 0xFFFFFFFFFFFFFll;
}
__device__ __forceinline__ int minpow2_bits(double a, double L) {
    if (!(a <= 1.7976931348623157e308)) return 1100;
    int ea, el;
    long long ma, ml;
    exp_mant(a, ea, ma);
    exp_mant(L, el, ml);
    int k = ea - el + (ma >= ml ? 1 : 0);
    return k < 1 ? 1 : k;
}

// Pivot data of one row: x = y / d.
//   real:    d and its correctly rounded reciprocal; the quotient is q0 = y r, rem = y - q0 d
//            (exact by FMA), q = q0 + rem r, which is the correctly rounded y / d (Markstein) when
//            nothing under/overflows -- otherwise the IEEE division itself (bit-exact with the
//            oracle's y / d).
//   complex: 1/d from an exactly prescaled conj(d)/|d|^2; x = y * (1/d) differs from the
//            oracle's Smith quotient by a few ulps (R24).
template <typename T> struct Piv;
// Real pivots: y / d correctly rounded, as q0 = y r, one residual correction (exact when q and d
// are well inside the normal range), else the IEEE division.  The range tests are integer tests of
// the biased exponents (FP64 compares issue on the FP64 pipe the row loop needs): |d| in
// [2^-999, 2^999) once per pivot, |q| in [2^-959, 2^999) per quotient -- inside the ranges the
// correction is exact on, so both branches give the same correctly rounded quotient.
template <> struct Piv<double> {
    double d, r;
    bool dok;
    __device__ __forceinline__ void make(double dd) {
        d = dd;
        r = __drcp_rn(dd);
        dok = unsigned(((__double2hiint(dd) >> 20) & 0x7ff) - 24) <= 1997u;
    }
    __device__ __forceinline__ double apply(double y) const {
        double q0 = __dmul_rn(y, r);
        double rem = fma(-q0, d, y);
        double q = fma(rem, r, q0);
        const bool qok = unsigned(((__double2hiint(q) >> 20) & 0x7ff) - 64) <= 1957u;
        const bool yzero = ((unsigned(__double2hiint(y)) << 1) | unsigned(__double2loint(y))) == 0u;
        return (dok && qok) || yzero ? q : __ddiv_rn(y, d);
    }
    __device__ __forceinline__ double absd() const { return fabs(d); }
    template <int W> __device__ __forceinline__ Piv shfl(int src) const {
        Piv o;
        o.d = __shfl_sync(0xffffffffu, d, src, W);
        o.r = __shfl_sync(0xffffffffu, r, src, W);
        o.dok = __shfl_sync(0xffffffffu, int(dok), src, W) != 0;
        return o;
    }
};
template <> struct Piv<cplx> {
    cplx r;
    __device__ __forceinline__ void make(cplx dd) {
        // (range tests on the exponent bits: FP64 compares would issue on the FP64 pipe)
        const unsigned hx = unsigned(__double2hiint(dd.x)) & 0x7fffffffu, hy = unsigned(__double2hiint(dd.y)) & 0x7fffffffu;
        const bool zx = (hx | unsigned(__double2loint(dd.x))) == 0u, zy = (hy | unsigned(__double2loint(dd.y))) == 0u;
        if ((zx && zy) || max(hx, hy) >= 0x7ff00000u) {               // 0 or non-finite pivot
            r = make_double2(__longlong_as_double(0x7ff8000000000000ll), __longlong_as_double(0x7ff8000000000000ll));
            return;
        }
        // Fast path: components 0 or in [2^-250, 2^250) keep every intermediate below normal --
        // scaling by a power of two commutes with each rounded step, so this is bit for bit the
        // prescaled computation below
        if ((zx || (hx >> 20) - 773u <= 499u) && (zy || (hy >> 20) - 773u <= 499u)) {
            const double inv = __drcp_rn(fma(dd.x, dd.x, __dmul_rn(dd.y, dd.y)));
            r = make_double2(__dmul_rn(dd.x, inv), -__dmul_rn(dd.y, inv));
            return;
        }
        const double big = fmax(fabs(dd.x), fabs(dd.y));
        int e;
        long long mnt;
        exp_mant(big, e, mnt);
        e -= 1023;                                                        // big in [2^e, 2^(e+1))
        double dx = mulp2s(dd.x, -e), dy = mulp2s(dd.y, -e);              // max component in [1, 2)
        double inv = __drcp_rn(fma(dx, dx, __dmul_rn(dy, dy)));          // 1 / |d 2^-e|^2
        r = make_double2(mulp2s(__dmul_rn(dx, inv), -e), mulp2s(-__dmul_rn(dy, inv), -e));
    }
    __device__ __forceinline__ cplx apply(cplx y) const {
        return make_double2(fma(y.x, r.x, -__dmul_rn(y.y, r.y)), fma(y.x, r.y, __dmul_rn(y.y, r.x)));
    }
    template <int W> __device__ __forceinline__ Piv shfl(int src) const {
        Piv o;
        o.r = make_double2(__shfl_sync(0xffffffffu, r.x, src, W), __shfl_sync(0xffffffffu, r.y, src, W));
        return o;
    }
};

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

// Element and bound accessor of the matrix a row loop solves with.  Standard solve: U'(i,l) =
// U(i,l) from the packed triangle, cnl(l) of U.  Generalized solve (Alg. 7/8): U'(i,l) =
// U(i,l) - lambda_j V(i,l) formed on the fly (P:873 / P:924, one fused complex multiply-subtract),
// bound cnlU(l) + |lambda_j| cnlV(l) (R30).
template <typename T, bool GEN, bool CONJ = false>
struct UAcc {
    const T *pk, *pkV;
    const double *cn, *cnV;
    T lam;
    double alam;
    __device__ __forceinline__ T operator()(int idx) const {
        if constexpr (GEN) return S<T>::fnms(pk[idx], lam, pkV[idx]);
        else if constexpr (CONJ) return S<T>::conj(pk[idx]);      // op C: L = U^H staged unconjugated
        else return pk[idx];
    }
    __device__ __forceinline__ double cnl(int sc) const {
        if constexpr (GEN) return fma(alam, cnV[sc], cn[sc]);
        else return cn[sc];
    }
};

#ifndef MSTRSM_DIAG_RR_UNROLL
#define MSTRSM_DIAG_RR_UNROLL 1
#endif
constexpr int kDiagRrUnroll = MSTRSM_DIAG_RR_UNROLL;     // unroll of the runtime row loop

// The substitution of one column group (Alg. 1; the unguarded branch of Alg. 4):
// x_l = y_l / d_l, y(rows < l) -= x_l U(rows < l, l).  Every lane forms the quotient of its own
// row of slot t and the owner's quotient is shuffled to the group, so the step-to-step chain is
// one multiply, one shuffle and one fused update.
template <typename T, int LPC, int RPL, typename PivF, typename Acc>
__device__ __forceinline__ void diag_subst(T (&y)[RPL], PivF pivot, const Acc &ua,
                                           int rl, int nrow, int nmax) {
    typedef S<T> ST;
#pragma unroll
    for (int t = RPL - 1; t >= 0; t--) {
        if (t * LPC >= nmax) continue;                                     // warp-uniform
        Piv<T> pvt;                                                        // own row of slot t
        pvt.make(pivot(t * LPC + rl));
        const int rr_hi = min(LPC - 1, nmax - 1 - t * LPC);               // rows >= nmax skipped
#pragma unroll kDiagRrUnroll
        for (int rr = rr_hi; rr >= 0; rr--) {
            const int sc = t * LPC + rr;
            // rows sc >= nrow (past this column's row end) need no masking: their y starts at 0,
            // nothing updates them before their turn (they are solved first) and their pivot is 1,
            // so x_l = 0 there and every update below is exact
            const T xl = group_shfl<T, LPC>(pvt.apply(y[t]), rr);          // P:82 / P:297
            const int col = (sc * (sc - 1)) / 2;
            const T upd = ST::fnms(y[t], xl, ua(col + rl + LPC * t));
            y[t] = rl < rr ? upd : (rl == rr ? xl : y[t]);
#pragma unroll
            for (int t2 = t - 1; t2 >= 0; t2--) y[t2] = ST::fnms(y[t2], xl, ua(col + rl + LPC * t2));
        }
    }
}

// Alg. 4's guarded loop with its decisions replayed LAG rows behind the substitution.
//
// The guarded loop only ever scales the whole vector by powers of two, so its
// values are the unscaled substitution's values times 2^-K (K = exponents taken so far) exactly,
// barring subnormals.  The registers therefore run the plain substitution, in a frame 2^pend
// above the paper's (pend = exponents decided but not yet applied), and the decisions for row l
// are taken LAG steps later from |x_l| (kept in shared memory), in the paper's order:
//   |y_l| >= Omega |d_l|  <=>  |x_l| >= Omega (to rounding)  ->  k1 = minpow2(|x_l|, Omega)
//   M = 2^-k1 |x_l|,  g = 2^-k1 g + M cnl(l),  g >= Omega  ->  k2 = minpow2(g, Omega)
// with minpow2 against Omega = 2^970 read off the exponent bits.  The registers are brought to the
// paper's frame one step after pend passes 12 bits; with the lag they stay within
// ~2^(12 + growth of LAG+2 rows) of it (LAG = 2, flush at 12 bits: no c5 column overflows; LAG = 4
// or a 20-bit flush sent 248 / 307906 c5 columns to the fallback, measured).  A group whose registers stop being finite (growth beyond
// 2^54 within that window, e.g. tiny pivots) returns false and is rerun by the synchronous loop.
template <typename T, int LPC, int RPL, typename PivF, typename Acc>
__device__ __forceinline__ bool diag_lagged(T (&y)[RPL], PivF pivot, const Acc &ua, int rl, int nrow, int nmax,
                                            bool guarded, double g, int &kt) {
    typedef S<T> ST;
#ifndef MSTRSM_DIAG_LAG
#define MSTRSM_DIAG_LAG 2
#endif
#ifndef MSTRSM_DIAG_FLUSH
#define MSTRSM_DIAG_FLUSH 12
#endif
    constexpr int LAG = LPC < MSTRSM_DIAG_LAG ? LPC : MSTRSM_DIAG_LAG;
    // K: exponents decided so far; Fl: exponents applied to the registers so far
    // (registers = unscaled * 2^-Fl, paper = unscaled * 2^-K).  Every LAG steps each lane of the
    // chunk just solved records |x| of its own row of the slot (ax_cur) and the register frame it
    // was read in (fl_cur); the previous slot's records move to ax_prev / fl_prev.
    int K = 0, Fl = 0, pend_prev = 0;
    double ax_cur = 0.0, ax_prev = 0.0;
    int fl_cur = 0, fl_prev = 0;
    bool nonfinite = false;
    auto replay = [&](int sc2, double axr, int fls, bool rep) {
        const bool live = rep && guarded && sc2 < nrow;
        const double axt = __dmul_rn(axr, pow2i(fls - K));                 // paper frame
        const bool t1 = live && axt >= kOmega;
        const int k1 = t1 ? int(__double_as_longlong(axt) >> 52) - 1992 : 0;
        const double M = t1 ? __dmul_rn(axt, pow2i(-k1)) : axt;
        double gn = __dadd_rn(t1 ? __dmul_rn(g, pow2i(-k1)) : g, __dmul_rn(M, ua.cnl(sc2 < nmax ? sc2 : 0)));
        const bool t2 = live && gn >= kOmega;
        const int k2 = t2 ? int(__double_as_longlong(gn) >> 52) - 1992 : 0;
        if (t2) gn = __dmul_rn(gn, pow2i(-k2));
        g = live ? gn : g;
        K += k1 + k2;
    };
#pragma unroll
    for (int t = RPL - 1; t >= 0; t--) {
        if (t * LPC >= nmax) continue;                                     // warp-uniform
        ax_prev = ax_cur;
        fl_prev = fl_cur;
        Piv<T> pvt;                                                        // own row of slot t
        pvt.make(pivot(t * LPC + rl));
        const int rr_hi = min(LPC - 1, nmax - 1 - t * LPC);               // rows >= nmax skipped
#pragma unroll kDiagRrUnroll
        for (int rr = rr_hi; rr >= 0; rr--) {
            const int sc = t * LPC + rr;
            const T xl = group_shfl<T, LPC>(pvt.apply(y[t]), rr);          // P:297 (x_l = 0 past row end)
            const int col = (sc * (sc - 1)) / 2;
            const T upd = ST::fnms(y[t], xl, ua(col + rl + LPC * t));      // (index in the padded triangle)
            y[t] = rl < rr ? upd : (rl == rr ? xl : y[t]);
#pragma unroll
            for (int t2 = t - 1; t2 >= 0; t2--) y[t2] = ST::fnms(y[t2], xl, ua(col + rl + LPC * t2));
            {                                                              // replay row sc + LAG
                const bool prev = rr + LAG >= LPC;
                const int src = (rr + LAG) & (LPC - 1);
                const double axr = __shfl_sync(0xffffffffu, prev ? ax_prev : ax_cur, src, LPC);
                const int fls = __shfl_sync(0xffffffffu, prev ? fl_prev : fl_cur, src, LPC);
                replay(sc + LAG, axr, fls, sc + LAG < nmax);
            }
            if (pend_prev >= MSTRSM_DIAG_FLUSH) {                          // lagged flush (rare)
                scale_all<true>(y, pend_prev);
                Fl += pend_prev;
            }
            pend_prev = K - Fl;
            if ((rr & (LAG - 1)) == 0) {                                   // warp-uniform: record the chunk
                const bool rec = rl >= rr && rl < rr + LAG;
                const double axn = modv(y[t]);
                ax_cur = rec ? axn : ax_cur;
                fl_cur = rec ? Fl : fl_cur;
                nonfinite |= rec && !(axn <= 1.7976931348623157e308);     // every solved row passes here
            }
        }
    }
#pragma unroll
    for (int sc2 = LAG - 1; sc2 >= 0; sc2--) {
        if (sc2 < nmax) {
            const double axr = __shfl_sync(0xffffffffu, ax_cur, sc2, LPC);
            const int fls = __shfl_sync(0xffffffffu, fl_cur, sc2, LPC);
            replay(sc2, axr, fls, true);
        }
    }
    if (K != Fl) scale_all<false>(y, K - Fl);
    kt = K;
#pragma unroll
    for (int o = 1; o < LPC; o <<= 1) nonfinite |= __shfl_xor_sync(0xffffffffu, nonfinite, o, LPC);
    return !(guarded && nonfinite);
}

// The synchronous guarded loop (fallback when phase 1 overflows): Alg. 4 step by step
// with the rescales applied lazily through pend.
// PADLPC > 0: the triangle is the padded layout of diag_fast.cuh / diag_tc.cuh with chunks of
// PADLPC rows (column l at padtri_off(l, PADLPC)) instead of the packed one (column l at l(l-1)/2).
template <typename T, int LPC, int RPL, bool GUARD, int PADLPC = 0, typename PivF, typename Acc>
__device__ __forceinline__ void diag_rows(T (&y)[RPL], PivF pivot, const Acc &ua,
                                          int rl, int nrow, int nmax, bool guarded, double &g, int &kt) {
    typedef S<T> ST;
    int pend = 0;
#pragma unroll
    for (int t = RPL - 1; t >= 0; t--) {
        if (t * LPC >= nmax) continue;                                     // warp-uniform
        Piv<T> pvt;                                                        // own row of slot t
        const T dt = pivot(t * LPC + rl);
        pvt.make(dt);
        const double oadt = __dmul_rn(kOmega, modv(dt));
#pragma unroll 1
        for (int rr = LPC - 1; rr >= 0; rr--) {
            const int sc = t * LPC + rr;
            if (sc >= nmax) continue;                                      // warp-uniform
            const bool in = sc < nrow;
            const T yl = group_shfl<T, LPC>(y[t], rr);                     // register frame
            const Piv<T> p = pvt.template shfl<LPC>(rr);
            T xv = p.apply(yl);                                            // P:297 / P:82
            if constexpr (GUARD) {
                const double oadv = __shfl_sync(0xffffffffu, oadt, rr, LPC);   // Omega |d_l|
                const double cnv = ua.cnl(sc);
                const bool live = in && guarded;
                // P:279-295 (R8): |y_l| >= Omega |d_l| in the true frame (pend <= 11 here: exact)
                const double ay = __dmul_rn(modv(yl), pow2i(-pend));
                const bool t1 = live && ay >= oadv;
                const int k1 = t1 ? minpow2_bits(ay, oadv) : 0;
                const int pend1 = pend + k1;
                // the register-frame quotient would overflow (tiny pivot): take x_l in the true
                // frame and bring the registers there before the substitution (rare)
                const bool xtrue = t1 && !(maxabs(xv) < 0x1p+1020);
                if (xtrue) xv = p.apply(mulp2n(yl, pend1));
                // M = |x_l|, g += M cnl(l), rescale when g >= Omega
                const double M = xtrue ? modv(xv) : mulp2n(modv(xv), pend1);
                double gn = __dadd_rn(t1 ? mulp2n(g, k1) : g, __dmul_rn(M, cnv));
                const bool t2 = live && gn >= kOmega;
                const int k2 = t2 ? minpow2_bits(gn, kOmega) : 0;
                if (t2) gn = mulp2n(gn, k2);
                g = live ? gn : g;
                kt += k1 + k2;
                pend = pend1 + k2;
                if (xtrue || pend >= 48) {
                    // keep the substitution below overflow (R8): true frame first
                    scale_all<false>(y, pend);
                    xv = mulp2n(xv, xtrue ? k2 : pend);
                    pend = 0;
                }
            }
            const T xr = in ? xv : ST::zero();
            // owner stores x_l; substitution within the block (P:315 / P:84): rows sc' < sc
            const int col = PADLPC ? int(padtri_off(sc, PADLPC)) : (sc * (sc - 1)) / 2;
            {
                const int i = rl + LPC * t;
                if (rl < rr) y[t] = ST::fnms(y[t], xr, ua(col + i));
                else if (rl == rr && in) y[t] = xv;
            }
#pragma unroll
            for (int t2 = t - 1; t2 >= 0; t2--) y[t2] = ST::fnms(y[t2], xr, ua(col + rl + LPC * t2));
            if constexpr (GUARD) {
                if (pend >= 12) {                                          // back to the true frame
                    scale_all<true>(y, pend);
                    pend = 0;
                }
            }
        }
    }
    if constexpr (GUARD) {
        if (pend) scale_all<true>(y, pend);
    }
}

// One launch = one diagonal block for all (FB = false: columns [c0, c0 + ncols); FB = true: the
// columns the main launch handed to the synchronous fallback) active columns.
template <typename T, int LPC, int RPL, bool SAFE, int OP, bool FB, bool GEN = false>
__global__ void __launch_bounds__(DiagThreads<T, RPL>::value, 1) diag_kernel(DiagArgs<T> a) {
    typedef S<T> ST;
    constexpr int G = 32 / LPC;
    static_assert(!GEN || OP == 0, "the generalized solve is op N only");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int nfull = int(a.hi - a.lo);
    pdl_wait();                    // before any global access, fb_count included (it is written
                                   // by the main launch that precedes this one in the stream)
    const int64_t ncols = FB ? int64_t(*a.fb_count) : a.ncols;
    if (ncols == 0) return;
    const int64_t npk = int64_t(nfull) * (nfull - 1) / 2 + 128;
    T *pk = reinterpret_cast<T *>(smem_raw);
    T *pkV = pk + (GEN ? npk : 0);
    T *dg = pkV + npk;
    T *dgV = dg + (GEN ? nfull : 0);
    double *cn = reinterpret_cast<double *>(dgV + nfull);
    double *cnV = cn + (GEN ? nfull : 0);

    // ---- stage U(I1,I1) (packed, solve coordinates), its diagonal and cnl ----
    const int tid = threadIdx.x, nth = blockDim.x;
    {
        for (int idx = tid; idx < nfull * 128; idx += nth) {       // any blockDim
            const int cq = idx >> 7, rl = idx & 127;
            if (rl < cq) {
                if (OP == 0) {      // U~(i,c) = U(lo+i, lo+c), asynchronous (waited for below)
                    cp_async<sizeof(T)>(pk + int64_t(cq) * (cq - 1) / 2 + rl,
                                        a.U + (a.lo + rl) + (a.lo + cq) * a.ldu, true);
                } else {            // U~(i,c) = conj(U(hi-1-c, hi-1-i)) (conjugated at use, UAcc)
                    int ci = nfull - 1 - cq, cc = nfull - 1 - rl;
                    cp_async<sizeof(T)>(pk + int64_t(cc) * (cc - 1) / 2 + ci,
                                        a.U + (a.lo + rl) + (a.lo + cq) * a.ldu, true);
                }
            }
        }
        for (int c = tid; c < nfull; c += nth) {
            int64_t row = OP == 0 ? a.lo + c : a.hi - 1 - c;
            T u = a.U[row + row * a.ldu];
            dg[c] = OP == 0 ? u : ST::conj(u);
            cn[c] = SAFE ? a.cnl[row] : 0.0;
        }
        if constexpr (GEN) {                                        // V(I1,I1), its diagonal, cnlV
            for (int idx = tid; idx < nfull * 128; idx += nth) {
                const int cq = idx >> 7, rl = idx & 127;
                if (rl < cq)
                    cp_async<sizeof(T)>(pkV + int64_t(cq) * (cq - 1) / 2 + rl,
                                        a.V + (a.lo + rl) + (a.lo + cq) * a.ldv, true);
            }
            for (int c = tid; c < nfull; c += nth) {
                const int64_t row = a.lo + c;
                dgV[c] = a.V[row + row * a.ldv];
                cnV[c] = SAFE ? a.cnlV[row] : 0.0;
            }
        }
        cp_async_commit();
    }
    __syncthreads();                                               // diagonal and cnl visible
    // the first column group's loads and precheck overlap the staging of the triangle; every warp
    // passes this second barrier exactly once (in its first iteration, or after the loop)
    bool staged = false;
    auto stage_wait = [&]() { cp_async_wait<0>(); __syncthreads(); staged = true; };

    const int lane = tid & 31, grp = lane / LPC, rl = lane % LPC;
    const int64_t wid = (int64_t(blockIdx.x) * nth + tid) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * nth) >> 5;
    const double delta = SAFE ? a.delta[0] : 0.0;
    const double Pb = SAFE ? diag_panel_sum(a) : 0.0;
    const double PbV = SAFE && GEN ? a.PV[a.b] : 0.0;
    const double rawU = SAFE && GEN ? a.delta[1] : 0.0, rawV = SAFE && GEN ? a.deltaV[1] : 0.0;

    for (int64_t base = wid * G; base < ncols; base += nw * G) {
        const int64_t q = base + grp;
        const bool valid = q < ncols;
        const int64_t j = FB ? (valid ? int64_t(a.fb_list[q]) : a.c0) : a.c0 + (valid ? q : 0);
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
        const double alam = GEN ? modv(sh) : 0.0;
        double delta_j = delta;
        if (GEN) {                                                    // R31
            delta_j = fma(alam, rawV, rawU);
            if (!(delta_j > 0.0)) delta_j = 2.2250738585072014e-308;
        }
        auto pivot = [&](int sc) -> T {                               // d_l = U(l,l) - s_j (V(l,l))
            T dd = sc < nrow ? (GEN ? ST::fnms(dg[sc], sh, dgV[sc]) : ST::sub(dg[sc], sh)) : ST::real(1.0);
            if (SAFE && ST::is_zero(dd)) dd = ST::real(delta_j);
            return dd;
        };
        const UAcc<T, GEN, OP == 1> ua{pk, pkV, cn, cnV, sh, alam};
        // ---- load the rows ----
        T y[RPL];
#pragma unroll
        for (int t = 0; t < RPL; t++) {
            const int sc = rl + LPC * t;
            y[t] = sc < nrow ? x[rowof(sc)] : ST::zero();
        }

        bool guarded = false;
        double g0 = 0.0;
        if (SAFE) {
            // ---- precheck, eqs. (4)-(5): g_top = ||y(I1)||_inf, g_{l-1} = g_l (1 +
            //      cnl_l/|d_l|), M = max_l g_l/|d_l| (tested as g_l < Omega |d_l|).  The products
            //      g_l = g_top prod_{l' > l} tf_l' are formed slot by slot with a suffix scan over
            //      the LPC lanes (rounding order differs from the sequential product at the ulp
            //      level, R24) ----
            //      The test only chooses between the unguarded loop and the guarded one, which
            //      produces the same result whenever no rescale triggers, so it uses upper bounds of
            //      |y| (sqrt 2 max(|re|,|im|)) and lower bounds of |d| (max(|re|,|im|)): a column
            //      the exact test would pass may take the guarded loop, never the reverse ----
            double gub = 0.0;
#pragma unroll
            for (int t = 0; t < RPL; t++)
                if (rl + LPC * t < nrow) gub = fmax(gub, maxabs(y[t]));
            gub = group_max<LPC>(gub);
            if constexpr (ST::cplx_) gub = __dmul_ru(gub, 1.4142135623730951);
            double carry = gub;                                        // g at the top of the slot
            bool okM = true;
#pragma unroll 1
            for (int t = RPL - 1; t >= 0; t--) {
                if (t * LPC >= nmax) continue;
                const int sc = t * LPC + rl;
                const bool in = sc < nrow;
                const double ad = maxabs(pivot(sc));                   // <= |d_l|
                const double tf = in ? __dadd_ru(1.0, __ddiv_ru(ua.cnl(sc < nfull ? sc : 0), ad)) : 1.0;
                double suf = tf;                                       // inclusive suffix product
#pragma unroll
                for (int o = 1; o < LPC; o <<= 1) {
                    const double v = __shfl_down_sync(0xffffffffu, suf, o, LPC);
                    if (rl + o < LPC) suf = __dmul_ru(suf, v);
                }
                double exc = __shfl_down_sync(0xffffffffu, suf, 1, LPC);   // rows above, this slot
                if (rl == LPC - 1) exc = 1.0;
                const double gl = __dmul_ru(carry, exc);
                okM = okM && (!in || gl < __dmul_rn(kOmega, ad));
                carry = __dmul_ru(carry, __shfl_sync(0xffffffffu, suf, 0, LPC));
            }
#pragma unroll
            for (int o = 1; o < LPC; o <<= 1) {                       // group AND (every lane shuffles)
                const bool other = __shfl_xor_sync(0xffffffffu, okM, o, LPC);
                okM = okM && other;
            }
            guarded = active && !(okM && carry < kOmega);
            if (__any_sync(0xffffffffu, guarded)) {                    // g := ||y(I1)||_inf
#pragma unroll
                for (int t = 0; t < RPL; t++)
                    if (rl + LPC * t < nrow) g0 = fmax(g0, modv(y[t]));
                g0 = group_max<LPC>(g0);
            }
        }

        // ---- the row loop ----
        if (!staged) stage_wait();
        int kt = 0;
        bool handed = false;
        if constexpr (FB) {
            double g = g0;
            diag_rows<T, LPC, RPL, true>(y, pivot, ua, rl, nrow, nmax, guarded, g, kt);
        } else {
            if (SAFE && __any_sync(0xffffffffu, guarded)) {
                const bool ok = diag_lagged<T, LPC, RPL>(y, pivot, ua, rl, nrow, nmax, guarded, g0, kt) &&
                                !(a.force_fb && guarded);
                if (!ok) {                                             // hand the column over
                    handed = true;
                    if (rl == 0) a.fb_list[atomicAdd(a.fb_count, 1)] = int(j);
                }
            } else {
                diag_subst<T, LPC, RPL>(y, pivot, ua, rl, nrow, nmax);
            }
        }

        if (SAFE) {
            int ej = 0;
            double Gj = 0.0;
            if (active) { ej = a.e[j]; Gj = a.G[j]; }
            if (kt > 0) {                                              // P:376-386, step (ii)
                ej -= kt;
                Gj = mulp2n(Gj, kt);
            }
            double xm = 0.0;
#pragma unroll
            for (int t = 0; t < RPL; t++) xm = fmax(xm, modv(y[t]));
            xm = group_max<LPC>(xm);
            Gj = __dadd_rn(Gj, __dmul_rn(GEN ? fma(alam, PbV, Pb) : Pb, xm));   // P:392 / P:952 (R30)
            int k3 = 0;
            if (Gj >= kOmega) {
                k3 = minpow2_bits(Gj, kOmega);
                scale_all<false>(y, k3);
                ej -= k3;
                Gj = mulp2n(Gj, k3);
            }
            if (active && rl == 0 && !handed) {
                a.e[j] = ej;
                a.G[j] = Gj;
                a.dblk[j] = -(kt + k3);
                a.Etab[a.b * a.n + j] = ej;
            }
        }
#pragma unroll
        for (int t = 0; t < RPL; t++) {
            int sc = rl + LPC * t;
            if (sc < nrow && !handed) x[rowof(sc)] = y[t];
        }
        if constexpr (ST::cplx_) {  // operand sums for the 3M update GEMM
            if (a.Xsum && valid && !handed) {
                double *xs = a.Xsum + j * a.ldxs;
#pragma unroll
                for (int t = 0; t < RPL; t++) {
                    const int sc = rl + LPC * t;
                    if (sc < nfull) xs[rowof(sc) - a.lo] = __dadd_rn(y[t].x, y[t].y);
                }
            }
        }
        if constexpr (GEN) {       // C(:,j) = -lambda_j X(I1,j), after the rescales (R32)
            if (valid && !handed) {
                const T nl = ST::neg(sh);
                T *cj = a.Cbuf + j * a.ldc;
#pragma unroll
                for (int t = 0; t < RPL; t++) {
                    const int sc = rl + LPC * t;
                    if (sc < nfull) cj[sc] = ST::fnms(ST::zero(), nl, ST::neg(y[t]));   // = -lambda y
                }
            }
        }
    }
    if (!staged) stage_wait();
}

}  // namespace mstrsm
