// aux_kernels.cuh -- the memory-bound steps of the path (HBM-roofline kernels):
//   a.1 RHS / state init  (eigen: P:519-525)
//   a.2 norm pass          (delta: P:231-234)
//   a.6 finalize           (lazy form of the xSCAL rescales P:378-380; diag Z P:530)
#pragma once
#include "common.cuh"

namespace mstrsm {

// ------------------------------------------------------------------------------------------
// a.2 norm pass, op N.  One warp per column k (grid-stride):
//   cnl[k]  = max_{lo(k) <= l < k} |U(l,k)|   (block-local off-diagonal column norm, R5)
//   pcol[k] = max_{l < lo(k)} |U(l,k)|          (panel part of P_b, R6)
// and flags a non-finite entry in U(0:k, k) (diagonal included).  max is order-free, so the
// results are bit-identical to a sequential evaluation.
template <typename T>
__global__ void norm_cols_n_kernel(const T *__restrict__ U, int64_t ldu, int64_t m, int nb,
                                   double *__restrict__ cnl, double *__restrict__ pcol,
                                   int *__restrict__ nonfinite) {
    int lane = threadIdx.x & 31;
    int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t k = w; k < m; k += nw) {
        int64_t b = (m - 1 - k) / nb;
        Blk bl = block_rows(0, m, nb, b);
        const T *col = U + k * ldu;
        double c = 0.0, p = 0.0;
        bool bad = false;
        for (int64_t l = lane; l <= k; l += 32) {
            T v = col[l];
            double a = S<T>::mod(v);
            bad |= !(a <= 1.7976931348623157e308);
            if (l < bl.lo) p = fmax(p, a);
            else if (l < k) c = fmax(c, a);
        }
        c = warp_max(c);
        p = warp_max(p);
        bad = __any_sync(0xffffffffu, bad);
        if (lane == 0) {
            cnl[k] = c;
            pcol[k] = p;
            if (bad) atomicExch(nonfinite, 1);
        }
    }
}

// Panel sums P_b, one thread per block, in the fixed order of R6 (op N: k ascending; op C:
// l descending), sequential -> bit-identical to the oracle given bit-identical inputs.
__global__ void panel_sum_kernel(int op, int64_t m, int nb, int64_t nblk,
                                 const double *__restrict__ part, double *__restrict__ P, int64_t b0 = 0) {
    int64_t b = b0 + int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (b >= nblk) return;
    Blk bl = block_rows(op, m, nb, b);
    double s = 0.0;
    if (op == 0) for (int64_t k = bl.lo; k < bl.hi; k++) s = __dadd_rn(s, part[k]);
    else for (int64_t l = bl.hi - 1; l >= bl.lo; l--) s = __dadd_rn(s, part[l]);
    P[b] = s;
}

// ||U||_inf for delta (R4).  op N: row sums sum_{k >= i} |U(i,k)|, ascending k, one thread per
// row, warp walks columns in lockstep (coalesced).  op C: column sums sum_{l = i..0} |U(l,i)|
// (= rows of U^H), descending l, one thread per column.
constexpr int kRowsumChunk = 64;    // columns per partial sum (more chunks: more loads in flight)

template <typename T>
__global__ void rowsum_n_kernel(const T *__restrict__ U, int64_t ldu, int64_t m,
                                double *__restrict__ part) {
    // grid (row blocks of 128, column chunks); partial sum of row i over the chunk's columns
    // k >= i, ascending k.  A second pass adds the chunks in ascending order (fixed order,
    // deterministic; differs from a single sequential sum only in rounding, which moves delta
    // by ulps).
    int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    int64_t k0 = int64_t(blockIdx.y) * kRowsumChunk, k1 = k0 + kRowsumChunk < m ? k0 + kRowsumChunk : m;
    double s = 0.0;
    if (i < m && k1 > i) {
        const int64_t kb = k0 > i ? k0 : i;
#pragma unroll 8
        for (int64_t k = kb; k < k1; k++) s = __dadd_rn(s, S<T>::mod(U[i + k * ldu]));   // ascending k
    }
    if (i < m) part[int64_t(blockIdx.y) * m + i] = s;
}

__global__ void rowsum_reduce_kernel(int64_t m, int64_t nchunks, const double *__restrict__ part,
                                     double *__restrict__ rs) {
    int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= m) return;
    double s = 0.0;
    for (int64_t c = 0; c < nchunks; c++) s = __dadd_rn(s, part[c * m + i]);
    rs[i] = s;
}


// delta[0] = 2^-52 max(rs) (or DBL_MIN when U == 0); delta[1] = 2^-52 max(rs) (the raw value the
// generalized solve combines per shift, R31).  One block.
__global__ void delta_kernel(int64_t m, const double *__restrict__ rs, double *__restrict__ delta) {
    __shared__ double red[32];
    double v = 0.0;
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) v = fmax(v, rs[i]);
    v = warp_max(v);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
        v = warp_max(v);
        if (threadIdx.x == 0) {
            delta[0] = v > 0.0 ? ldexp(v, -52) : 2.2250738585072014e-308;
            delta[1] = ldexp(v, -52);
        }
    }
}

// ------------------------------------------------------------------------------------------
// a.1 init (general RHS).  One warp per column j: G_j = max_{l < r_j} |B(l,j)|,
// e_j = 0, rows [r_j, m) zeroed (R26); flags non-finite shifts.
template <typename T>
__global__ void init_rhs_kernel(T *__restrict__ B, int64_t ldb, int64_t m, int64_t n,
                                const int64_t *__restrict__ rowend, const T *__restrict__ shifts,
                                int64_t sstride, double *__restrict__ G, int *__restrict__ e,
                                int *__restrict__ nonfinite) {
    int lane = threadIdx.x & 31;
    int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t j = w; j < n; j += nw) {
        int64_t r = rowend ? rowend[j] : m;
        r = r < 0 ? 0 : (r > m ? m : r);
        T *x = B + j * ldb;
        double g = 0.0;
        for (int64_t l = lane; l < m; l += 32) {
            if (l < r) g = fmax(g, S<T>::mod(x[l]));
            else x[l] = S<T>::zero();
        }
        g = warp_max(g);
        if (lane == 0) {
            if (G) G[j] = g;
            if (e) e[j] = 0;
            if (shifts && nonfinite && !(S<T>::mod(shifts[j * sstride]) <= 1.7976931348623157e308))
                atomicExch(nonfinite, 1);
        }
    }
}

// a.1 init for TriangEig (Alg. 6).  Column q holds eigenvector k = cols[q]:
//   Z(l,q) = -T(l,k) for l < k, 0 for l >= k;  G_q = max_{l<k} |T(l,k)|;  shift_q = T(k,k);
//   row_end_q = k (the P:503-508 shortcut).
template <typename T>
__global__ void init_trevc_kernel(const T *__restrict__ Tm, int64_t ldt, int64_t m,
                                  const int64_t *__restrict__ cols, int64_t ncols,
                                  T *__restrict__ Z, int64_t ldz, T *__restrict__ shifts,
                                  int64_t *__restrict__ rowend, double *__restrict__ G,
                                  int *__restrict__ e, int *__restrict__ nonfinite) {
    int lane = threadIdx.x & 31;
    int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t q = w; q < ncols; q += nw) {
        int64_t k = cols ? cols[q] : q;
        const T *tc = Tm + k * ldt;
        T *z = Z + q * ldz;
        double g = 0.0;
        for (int64_t l = lane; l < m; l += 32) {
            if (l < k) {
                T v = tc[l];
                g = fmax(g, S<T>::mod(v));
                z[l] = S<T>::neg(v);
            } else {
                z[l] = S<T>::zero();
            }
        }
        g = warp_max(g);
        if (lane == 0) {
            T d = tc[k];
            shifts[q] = d;
            rowend[q] = k;
            G[q] = g;
            e[q] = 0;
            if (!(S<T>::mod(d) <= 1.7976931348623157e308)) atomicExch(nonfinite, 1);
        }
    }
}

// a.1 + a.2 (column part) + the 3M sum plane fused for TriangEig over all m columns (column q =
// eigenvector q): one read of T(0:k, k) per column gives cnl / pcol (norm_cols_n_kernel), Z and
// G / rowend / shifts / e (init_trevc_kernel; G = max(cnl, pcol) = max_{l<k} |T(l,k)|) and, when
// P is non-null, the plane P(l,k) = Re + Im (presum_kernel) -- |T(l,k)| evaluated once.
// qof (nullable): column subset -- eigenvector k goes to column qof[k] of Z (-1: not in the subset);
// the norms and the plane always cover every column of T.
// Running max of |v| over a column without a square root per element (prepass, a.1/a.2): for a
// complex v with both components in [2^-500, 2^500) |v| = sqrt_rn(x^2 + y^2) with no prescale
// (S<cplx>::mod), a monotone function of the rounded sum, so the maximum is sqrt_rn of the largest
// sum (non-negative doubles order like their bits); zeros add nothing; any other element takes
// S<T>::mod itself, which also flags non-finite entries.  Bit-identical to max_l S<T>::mod(v_l).
struct ModMax {
    long long qb = -1;
    double other = 0.0;
    bool bad = false;
    __device__ __forceinline__ void add(double v) {
        const double a = fabs(v);
        bad |= !(a <= 1.7976931348623157e308);
        other = fmax(other, a);
    }
    __device__ __forceinline__ void add(cplx v) {
        const unsigned hx = unsigned(__double2hiint(v.x)) & 0x7fffffffu;
        const unsigned hy = unsigned(__double2hiint(v.y)) & 0x7fffffffu;
        const unsigned hb = max(hx, hy);
        if ((hb >> 20) - 523u <= 999u) {
            const double q = __dadd_rn(__dmul_rn(v.x, v.x), __dmul_rn(v.y, v.y));
            qb = max(qb, __double_as_longlong(q));
        } else if ((hb | unsigned(__double2loint(v.x)) | unsigned(__double2loint(v.y))) != 0u) {
            const double a = S<cplx>::mod(v);
            bad |= !(a <= 1.7976931348623157e308);
            other = fmax(other, a);
        }
    }
    __device__ __forceinline__ double get() const {
        return qb >= 0 ? fmax(__dsqrt_rn(__longlong_as_double(qb)), other) : other;
    }
};

template <typename T>
__global__ void trevc_prepass_kernel(const T *__restrict__ Tm, int64_t ldt, int64_t m, int nb,
                                     double *__restrict__ cnl, double *__restrict__ pcol,
                                     T *__restrict__ Z, int64_t ldz, T *__restrict__ shifts,
                                     int64_t *__restrict__ rowend, double *__restrict__ G, int *__restrict__ e,
                                     double *__restrict__ P, int64_t ldp, int *__restrict__ nonfinite,
                                     const int *__restrict__ qof = nullptr, int64_t k0 = 0, int64_t k1 = -1) {
    // columns [k0, k1) of T (k1 < 0: all); the multi-GPU path runs it panel by panel as T arrives
    const int lane = threadIdx.x & 31;
    const int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    const int64_t kend = k1 < 0 ? m : k1;
    for (int64_t k = k0 + w; k < kend; k += nw) {
        const int64_t b = (m - 1 - k) / nb;
        const Blk bl = block_rows(0, m, nb, b);
        const T *tc = Tm + k * ldt;
        const int64_t q = qof ? int64_t(qof[k]) : k;
        T *z = q >= 0 ? Z + q * ldz : nullptr;
        ModMax mc, mp;
        for (int64_t l = lane; l < m; l += 32) {
            if (l < k) {
                const T v = tc[l];
                if (l < bl.lo) mp.add(v);
                else mc.add(v);
                if (z) z[l] = S<T>::neg(v);
                if constexpr (S<T>::cplx_) {
                    if (P) P[l + k * ldp] = __dadd_rn(v.x, v.y);
                }
            } else if (z) {
                z[l] = S<T>::zero();
            }
        }
        const double c = warp_max(mc.get());
        const double p = warp_max(mp.get());
        const bool bad = __any_sync(0xffffffffu, mc.bad || mp.bad);
        if (lane == 0) {
            const T d = tc[k];
            cnl[k] = c;
            pcol[k] = p;
            if (q >= 0) {
                shifts[q] = d;
                rowend[q] = k;
                G[q] = fmax(c, p);
                e[q] = 0;
            }
            if (bad || !(S<T>::mod(d) <= 1.7976931348623157e308)) atomicExch(nonfinite, 1);
        }
    }
}

// trevc_prepass_kernel for the columns [k0, k1) of one panel of T (the multi-GPU path runs it as
// each panel arrives): the same values, with every column split over gridDim.y row chunks so that
// one panel fills the GPU.  The maxima are combined with atomicMax on the bit patterns
// (non-negative doubles order like their bits; max is exact, so the result does not depend on
// the order): cnl, pcol and G must be zero beforehand.  Chunk 0 writes the per-column scalars.
__device__ __forceinline__ void atomic_max_nonneg(double *a, double v) {
    atomicMax(reinterpret_cast<unsigned long long *>(a), static_cast<unsigned long long>(__double_as_longlong(v)));
}
// a.2 norm pass, op C (L = U^H):
//   cnl[l]  = max_{l < i < hi(l)} |U(l,i)|     (block-local column norm of L)
//   prow[l] = max_{i >= hi(l)} |U(l,i)|
// One thread per row l of U (a warp reads consecutive rows of one column: coalesced), the columns
// split in chunks of kRowsumChunk over a 2-D grid and combined with atomic_max_nonneg.  max is
// exact, so the result does not depend on the split; cnl and prow must be zero beforehand.  (The
// first version walked whole rows on m / 128 CTAs: 0.65 ms at m = 1024.)
template <typename T>
__global__ void norm_rows_c_chunk_kernel(const T *__restrict__ U, int64_t ldu, int64_t m, int nb,
                                         double *__restrict__ cnl, double *__restrict__ prow,
                                         int *__restrict__ nonfinite) {
    const int64_t l = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t i0 = int64_t(blockIdx.y) * kRowsumChunk;
    const int64_t i1 = i0 + kRowsumChunk < m ? i0 + kRowsumChunk : m;
    if (l >= m || i1 <= l) return;
    const int64_t hi = block_rows(1, m, nb, l / nb).hi;
    double c = 0.0, p = 0.0;
    bool bad = false;
#pragma unroll 4
    for (int64_t i = i0 > l ? i0 : l; i < i1; i++) {
        const double a = S<T>::mod(U[l + i * ldu]);
        bad |= !(a <= 1.7976931348623157e308);
        if (i > l) {
            if (i < hi) c = fmax(c, a); else p = fmax(p, a);
        }
    }
    if (c > 0.0) atomic_max_nonneg(cnl + l, c);
    if (p > 0.0) atomic_max_nonneg(prow + l, p);
    if (bad) atomicExch(nonfinite, 1);
}

// ||U||_inf for delta (R4), op C: rs[i] = sum_{l = i..0} |U(l,i)|, descending l (R6's fixed order),
// one sequential sum per column.  A CTA owns 32 columns: its 8 warps stage
// 32 x 32 tiles of |U| in shared memory (a warp per column, lanes down the rows: coalesced), then
// lane c of warp 0 adds column c's tile rows in descending order.  (The first version, one thread
// per column, read 32 columns per warp access on m / 128 CTAs: 0.38 ms at m = 1024.)
template <typename T>
__global__ void __launch_bounds__(256) colsum_c_tiled_kernel(const T *__restrict__ U, int64_t ldu, int64_t m,
                                                             double *__restrict__ rs) {
    __shared__ double tile[2][32][33];                                     // [buffer][column][row]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t i0 = int64_t(blockIdx.x) * 32;
    const int64_t i = i0 + lane;
    const int64_t imax = i0 + 31 < m - 1 ? i0 + 31 : m - 1;
    double s = 0.0;
    for (int64_t tt = imax / 32; tt >= 0; tt--) {
        const int64_t l0 = tt * 32;
        const int buf = int(tt & 1);
        for (int cc = warp; cc < 32; cc += 8) {
            const int64_t ic = i0 + cc, l = l0 + lane;
            tile[buf][cc][lane] = (ic < m && l <= ic) ? S<T>::mod(U[l + ic * ldu]) : 0.0;
        }
        __syncthreads();          // (also orders warp 0's reads of this buffer two tiles ago)
        if (warp == 0 && i < m) {
#pragma unroll 8
            for (int r = 31; r >= 0; r--)
                if (l0 + r <= i) s = __dadd_rn(s, tile[buf][lane][r]);
        }
    }
    if (warp == 0 && i < m) rs[i] = s;
}

template <typename T>
__global__ void trevc_prepass_panel_kernel(const T *__restrict__ Tm, int64_t ldt, int64_t m, int nb,
                                           double *__restrict__ cnl, double *__restrict__ pcol,
                                           T *__restrict__ Z, int64_t ldz, T *__restrict__ shifts,
                                           int64_t *__restrict__ rowend, double *__restrict__ G, int *__restrict__ e,
                                           double *__restrict__ P, int64_t ldp, int *__restrict__ nonfinite,
                                           const int *__restrict__ qof, int64_t k0, int64_t k1, int64_t rchunk) {
    const int lane = threadIdx.x & 31;
    const int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    const int64_t r0 = int64_t(blockIdx.y) * rchunk, r1 = r0 + rchunk < m ? r0 + rchunk : m;
    for (int64_t k = k0 + w; k < k1; k += nw) {
        const int64_t b = (m - 1 - k) / nb;
        const Blk bl = block_rows(0, m, nb, b);
        const T *tc = Tm + k * ldt;
        const int64_t q = qof ? int64_t(qof[k]) : k;
        T *z = q >= 0 ? Z + q * ldz : nullptr;
        ModMax mc, mp;
        for (int64_t l = r0 + lane; l < r1; l += 32) {
            if (l < k) {
                const T v = tc[l];
                if (l < bl.lo) mp.add(v);
                else mc.add(v);
                if (z) z[l] = S<T>::neg(v);
                if constexpr (S<T>::cplx_) {
                    if (P) P[l + k * ldp] = __dadd_rn(v.x, v.y);
                }
            } else if (z) {
                z[l] = S<T>::zero();
            }
        }
        const double c = warp_max(mc.get());
        const double p = warp_max(mp.get());
        const bool bad = __any_sync(0xffffffffu, mc.bad || mp.bad);
        if (lane == 0) {
            if (c > 0.0) atomic_max_nonneg(cnl + k, c);
            if (p > 0.0) atomic_max_nonneg(pcol + k, p);
            if (q >= 0 && fmax(c, p) > 0.0) atomic_max_nonneg(G + q, fmax(c, p));
            if (blockIdx.y == 0) {
                const T d = tc[k];
                if (q >= 0) {
                    shifts[q] = d;
                    rowend[q] = k;
                    e[q] = 0;
                }
                if (!(S<T>::mod(d) <= 1.7976931348623157e308)) atomicExch(nonfinite, 1);
            }
            if (bad) atomicExch(nonfinite, 1);
        }
    }
}

// a.1 init for GeneralizedTriangEig (Alg. 9).  Column q holds eigenvector k = q:
//   lambda_q = T(k,k) / S(k,k);  Z(l,q) = S(l,k) lambda_q - T(l,k) for l < k, 0 for l >= k;
//   G_q = max_{l<k} |Z(l,q)|;  row_end_q = k.
template <typename T>
__global__ void init_tgevc_kernel(const T *__restrict__ Tm, int64_t ldt, const T *__restrict__ Sm,
                                  int64_t lds, int64_t m, T *__restrict__ Z, int64_t ldz,
                                  T *__restrict__ lam, int64_t *__restrict__ rowend,
                                  double *__restrict__ G, int *__restrict__ e,
                                  int *__restrict__ nonfinite) {
    int lane = threadIdx.x & 31;
    int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t k = w; k < m; k += nw) {
        const T *tc = Tm + k * ldt, *sc = Sm + k * lds;
        const T l = S<T>::div(tc[k], sc[k]);
        T *z = Z + k * ldz;
        double g = 0.0;
        for (int64_t i = lane; i < m; i += 32) {
            if (i < k) {
                const T v = S<T>::sub(S<T>::mul(sc[i], l), tc[i]);   // P:987 Z := -T + S diag(lambda)
                g = fmax(g, S<T>::mod(v));
                z[i] = v;
            } else {
                z[i] = S<T>::zero();
            }
        }
        g = warp_max(g);
        if (lane == 0) {
            lam[k] = l;
            rowend[k] = k;
            G[k] = g;
            e[k] = 0;
            if (!(S<T>::mod(l) <= 1.7976931348623157e308)) atomicExch(nonfinite, 1);
        }
    }
}

// ------------------------------------------------------------------------------------------
// Side / triangle variants (SURVEY §8f f4, P:58-62 footnote): operand transforms in 32 x 32
// shared-memory tiles (coalesced both ways).
//   tri_upper_kernel: U(i,k), i <= k, from A:  mode 0: conj(A(k,i)) (lower -> A^H),
//                     mode 1: A(k,i) (lower -> A^T),  mode 2: conj(A(i,k)) (upper -> conj A).
//   The other triangle of A is never read.
template <typename T>
__global__ void tri_upper_kernel(const T *__restrict__ A, int64_t lda, int64_t m, T *__restrict__ U,
                                 int64_t ldu, int mode) {
    __shared__ T tile[32][33];
    const int64_t ti = int64_t(blockIdx.y) * 32, tk = int64_t(blockIdx.x) * 32;   // U tile rows ti.., cols tk..
    if (ti > tk) return;                                                          // below the diagonal
    const int tx = threadIdx.x, ty = threadIdx.y;                                 // 32 x 8 threads
    for (int r = ty; r < 32; r += 8) {
        if (mode == 2) {                      // no transpose: U(ti + tx, tk + r) = conj A(ti + tx, tk + r)
            const int64_t i = ti + tx, k = tk + r;
            if (i < m && k < m && i <= k) U[i + k * ldu] = S<T>::conj(A[i + k * lda]);
        } else {                              // load A(tk + tx, ti + r) (lower: row >= col)
            const int64_t ar = tk + tx, ac = ti + r;
            if (ar < m && ac < m && ar >= ac) tile[r][tx] = A[ar + ac * lda];
        }
    }
    if (mode == 2) return;
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {        // U(ti + tx, tk + r) = f(A(tk + r, ti + tx)) = f(tile[tx][r])
        const int64_t i = ti + tx, k = tk + r;
        if (i < m && k < m && i <= k) {
            const T v = tile[tx][r];
            U[i + k * ldu] = mode == 0 ? S<T>::conj(v) : v;
        }
    }
}

// dst(c, r) = src(r, c) for r < rows, c < cols (column-major, 32 x 32 tiles)
template <typename T>
__global__ void transpose_kernel(const T *__restrict__ src, int64_t lds, int64_t rows, int64_t cols,
                                 T *__restrict__ dst, int64_t ldd) {
    __shared__ T tile[32][33];
    const int64_t r0 = int64_t(blockIdx.x) * 32, c0 = int64_t(blockIdx.y) * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;
    for (int c = ty; c < 32; c += 8)
        if (r0 + tx < rows && c0 + c < cols) tile[c][tx] = src[(r0 + tx) + (c0 + c) * lds];
    __syncthreads();
    for (int r = ty; r < 32; r += 8)
        if (c0 + tx < cols && r0 + r < rows) dst[(c0 + tx) + (r0 + r) * ldd] = tile[tx][r];
}

template <typename T>
__global__ void conj_strided_kernel(const T *__restrict__ s, int64_t stride, int64_t n, T *__restrict__ d) {
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j < n) d[j] = S<T>::conj(s[j * stride]);
}

// X := -X on an m x n column-major array (the back-transformation's sign, mstrsm.cu)
template <typename T>
__global__ void negate_kernel(T *__restrict__ X, int64_t ldx, int64_t m, int64_t n) {
    const int64_t total = m * n, stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += stride) {
        const int64_t c = i / m, r = i - c * m;
        X[r + c * ldx] = S<T>::neg(X[r + c * ldx]);
    }
}

// Operand sums for the complex 3M update GEMM: P(i,k) = Re U(i,k) + sign Im U(i,k)
// on the strictly upper triangle (op N: sign = +1; op C, whose A operand is conj(U)^T: sign = -1).
// rows = 0: strictly upper part of an m x m triangle; rows > 0: all `rows` rows of ncols columns.
__global__ void presum_kernel(const cplx *__restrict__ U, int64_t ldu, int64_t m, double *__restrict__ P,
                              int64_t ldp, double sign, int64_t rows = 0) {
    int lane = threadIdx.x & 31;
    int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t k = w; k < m; k += nw) {
        const cplx *uc = U + k * ldu;
        double *pc = P + k * ldp;
        const int64_t r = rows > 0 ? rows : k;
        for (int64_t i = lane; i < r; i += 32) pc[i] = fma(sign, uc[i].y, uc[i].x);
    }
}

// ------------------------------------------------------------------------------------------
// a.6 finalize.  Block b finalised rows I1(b) of column j in the frame E[b][j]; the final frame
// is e_j, so X(I1(b), j) *= 2^{e_j - E[b][j]} (exact powers of two; the lazy form of the
// eager xSCAL of rows I2 in P:378-380 / P:398).  Then c_j = 2^{e_j} -> scales, e_j -> exp,
// and for TriangEig Z(k,q) = c_q.
template <typename T>
__global__ void finalize_kernel(int op, T *__restrict__ B, int64_t ldb, int64_t m, int64_t n,
                                int nb, int64_t nblk, const int64_t *__restrict__ rowend,
                                const int *__restrict__ e, const int *__restrict__ Etab,
                                double *__restrict__ scales, int *__restrict__ scale_exp,
                                const int64_t *__restrict__ diag_row) {
    pdl_wait();
    int lane = threadIdx.x & 31;
    int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t j = w; j < n; j += nw) {
        int ej = e ? e[j] : 0;
        int64_t r = rowend ? rowend[j] : m;
        T *x = B + j * ldb;
        if (Etab) {
            // the frames of 32 blocks at a time, one per lane (one round of loads instead of a
            // chain of nblk), then the blocks whose frame differs, in turn, by the whole warp
            for (int64_t b0 = 0; b0 < nblk; b0 += 32) {
                const int64_t bq = b0 + lane;
                int d = 0;
                if (bq < nblk && block_rows(op, m, nb, bq).lo < r) d = ej - Etab[bq * n + j];
                unsigned todo = __ballot_sync(0xffffffffu, d != 0);
                while (todo) {
                    const int s = __ffs(todo) - 1;
                    todo &= todo - 1;
                    const int ds = __shfl_sync(0xffffffffu, d, s);
                    const Blk bl = block_rows(op, m, nb, b0 + s);
                    const int64_t hh = bl.hi < r ? bl.hi : r;
                    for (int64_t l = bl.lo + lane; l < hh; l += 32) x[l] = S<T>::ldx(x[l], ds);
                }
            }
        }
        if (lane == 0) {
            double c = ldexp(1.0, ej);
            if (scales) scales[j] = c;
            if (scale_exp) scale_exp[j] = ej;
            if (diag_row) x[diag_row[j]] = S<T>::real(c);
        }
    }
}

}  // namespace mstrsm
