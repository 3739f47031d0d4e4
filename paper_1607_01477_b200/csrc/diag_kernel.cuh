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
// Layout: one warp per column (persistent CTAs loop over columns).  The diagonal block is
// staged once per CTA in shared memory as a packed strictly-upper triangle in "solve
// coordinates" sc (op N: sc = row - lo; op C: sc = hi-1-row, the flip of DESIGN §4 / R9), so
// the same loop serves back substitution (op N) and forward substitution with L = U^H (op C).
// Lane `lane` owns solve rows sc = rr*32 + lane, rr < RPL.
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

template <typename T, int RPL, bool SAFE, int OP>
__global__ void __launch_bounds__(512) diag_kernel(DiagArgs<T> a) {
    typedef S<T> ST;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int nfull = int(a.hi - a.lo);
    const int64_t npk = int64_t(nfull) * (nfull - 1) / 2 + 128;
    T *pk = reinterpret_cast<T *>(smem_raw);
    T *dg = pk + npk;
    double *cn = reinterpret_cast<double *>(dg + nfull);

    // ---- stage U(I1,I1) (packed, solve coordinates), its diagonal and cnl ----
    const int tid = threadIdx.x, nth = blockDim.x;
    {
        const int rl = tid & 127, cstep = nth >> 7;
        for (int cq = tid >> 7; cq < nfull; cq += cstep) {
            if (rl < cq) {
                if (OP == 0) {      // U~(i,c) = U(lo+i, lo+c)
                    pk[int64_t(cq) * (cq - 1) / 2 + rl] = a.U[(a.lo + rl) + (a.lo + cq) * a.ldu];
                } else {            // U~(i,c) = conj(U(hi-1-c, hi-1-i)); read U column q = lo+cq, row r = lo+rl
                    int ci = nfull - 1 - cq;          // solve index of the U column
                    int cc = nfull - 1 - rl;          // solve index of the U row
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

    const int lane = tid & 31;
    const int64_t wid = (int64_t(blockIdx.x) * nth + tid) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * nth) >> 5;
    const double delta = SAFE ? *a.delta : 0.0;
    const double Pb = SAFE ? a.P[a.b] : 0.0;

    for (int64_t q = wid; q < a.ncols; q += nw) {
        const int64_t j = a.c0 + q;
        const int64_t r = (OP == 0 && a.rowend) ? a.rowend[j] : a.m;
        if (r <= a.lo) {                      // column not active in this block
            if (SAFE && lane == 0) a.dblk[j] = 0;
            continue;
        }
        const int nrow = OP == 0 ? int((a.hi < r ? a.hi : r) - a.lo) : nfull;
        T sh = a.shifts[j * a.sstride];
        if (OP == 1) sh = ST::conj(sh);
        T *x = a.B + j * a.ldb;

        T y[RPL], d[RPL];
#pragma unroll
        for (int rr = 0; rr < RPL; rr++) {
            int sc = rr * 32 + lane;
            if (sc < nrow) {
                int64_t row = OP == 0 ? a.lo + sc : a.hi - 1 - sc;
                y[rr] = x[row];
                T dd = ST::sub(dg[sc], sh);
                if (SAFE && ST::is_zero(dd)) dd = ST::real(delta);
                d[rr] = dd;
            } else {
                y[rr] = ST::zero();
                d[rr] = ST::real(1.0);
            }
        }

        bool guarded = false;
        double g = 0.0;
        int kt = 0;
        if (SAFE) {
            // ---- precheck, eqs. (4)-(5): M = max(g/|d_l|, M); g = g (1 + cnl/|d_l|),
            // evaluated in the oracle's order: the product chain is sequential, the quotients
            // use the value of g before each step. ----
            double ad[RPL], tf[RPL], gb[RPL];
            double g0 = 0.0;
#pragma unroll
            for (int rr = 0; rr < RPL; rr++) {
                int sc = rr * 32 + lane;
                g0 = fmax(g0, ST::mod(y[rr]));
                ad[rr] = ST::mod(d[rr]);
                tf[rr] = __dadd_rn(1.0, __ddiv_rn(sc < nrow ? cn[sc] : 0.0, ad[rr]));
                gb[rr] = 0.0;
            }
            g0 = warp_max(g0);
            double gg = g0;
#pragma unroll
            for (int rr = RPL - 1; rr >= 0; rr--) {
                for (int t = 31; t >= 0; t--) {
                    if (rr * 32 + t >= nrow) continue;
                    if (lane == t) gb[rr] = gg;
                    gg = __dmul_rn(gg, __shfl_sync(0xffffffffu, tf[rr], t));
                }
            }
            double M = 0.0;
#pragma unroll
            for (int rr = 0; rr < RPL; rr++)
                if (rr * 32 + lane < nrow) M = fmax(M, __ddiv_rn(gb[rr], ad[rr]));
            M = warp_max(M);
            guarded = !(M < kOmega && gg < kOmega);
            g = g0;
        }

        // ---- Trsv / guarded loop, solve coordinate sc = nrow-1 .. 0 ----
#pragma unroll
        for (int rr = RPL - 1; rr >= 0; rr--) {
            for (int t = 31; t >= 0; t--) {
                const int sc = rr * 32 + t;
                if (sc >= nrow) continue;
                T yl = ST::shfl(y[rr], t);
                T dl = ST::shfl(d[rr], t);
                if (SAFE && guarded) {
                    double ay = ST::mod(yl), adl = ST::mod(dl);
                    double lim = __dmul_rn(kOmega, adl);
                    if (ay >= lim) {                                   // P:282-295 (R8)
                        int k = minpow2(ay, lim);
#pragma unroll
                        for (int q2 = 0; q2 < RPL; q2++) y[q2] = ST::ldx(y[q2], -k);
                        yl = ST::ldx(yl, -k);
                        kt += k;
                        g = ldexp(g, -k);
                    }
                }
                T xl = ST::div(yl, dl);                                // P:297 diagonal step
                if (SAFE && guarded) {
                    double M = ST::mod(xl);
                    g = __dadd_rn(g, __dmul_rn(M, cn[sc]));
                    if (g >= kOmega) {
                        int k = minpow2(g, kOmega);
#pragma unroll
                        for (int q2 = 0; q2 < RPL; q2++) y[q2] = ST::ldx(y[q2], -k);
                        xl = ST::ldx(xl, -k);
                        kt += k;
                        g = ldexp(g, -k);
                    }
                }
                if (lane == t) y[rr] = xl;
                // substitution within the block (P:315 / P:84): rows sc' < sc
                const T *col = pk + int64_t(sc) * (sc - 1) / 2;
#pragma unroll
                for (int q2 = 0; q2 <= rr; q2++) {
                    int i = q2 * 32 + lane;
                    if (i < sc) y[q2] = ST::fnms(y[q2], xl, col[i]);
                }
            }
        }

        if (SAFE) {
            int ej = a.e[j];
            double Gj = a.G[j];
            if (kt > 0) {                                              // P:376-386, step (ii)
                ej -= kt;
                Gj = ldexp(Gj, -kt);
            }
            double xm = 0.0;
#pragma unroll
            for (int rr = 0; rr < RPL; rr++) xm = fmax(xm, ST::mod(y[rr]));
            xm = warp_max(xm);
            Gj = __dadd_rn(Gj, __dmul_rn(Pb, xm));
            int k3 = 0;
            if (Gj >= kOmega) {
                k3 = minpow2(Gj, kOmega);
#pragma unroll
                for (int rr = 0; rr < RPL; rr++) y[rr] = ST::ldx(y[rr], -k3);
                ej -= k3;
                Gj = ldexp(Gj, -k3);
            }
            if (lane == 0) {
                a.e[j] = ej;
                a.G[j] = Gj;
                a.dblk[j] = -(kt + k3);
                a.Etab[a.b * a.n + j] = ej;
            }
        }
#pragma unroll
        for (int rr = 0; rr < RPL; rr++) {
            int sc = rr * 32 + lane;
            if (sc < nrow) x[OP == 0 ? a.lo + sc : a.hi - 1 - sc] = y[rr];
        }
    }
}

}  // namespace mstrsm
