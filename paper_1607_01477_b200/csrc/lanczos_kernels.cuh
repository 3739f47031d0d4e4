// lanczos_kernels.cuh -- a.7 inverse-Lanczos step of the Van Loan / Lui pseudospectra driver
// (R14, R25).  One warp per grid point; all points advance in lockstep, each operator
// application being one op-N and one op-C multi-shift solve over all points.
#pragma once
#include "common.cuh"

namespace mstrsm {

// Vectors are stored by batch slot (columns 0..n_act-1 of V, Vp, W, Y); the per-point scalars by
// point id p = pid[slot].  SpectralCloud deflation (R33) compacts the slots between steps.
struct LanczosState {
    cplx *V, *Vp, *W, *Y;        // m x npts each (column per slot)
    double *alpha, *beta;        // iters x npts, by point
    int *kdone, *active, *flags;
    double *amax, *beta_prev, *sigma, *theta_prev;
    const int *e1, *e2;          // exponents of the two solves of this step, by slot
    const int *pid;              // slot -> point
    int64_t npts;                // points in the problem (stride of alpha / beta)
    double tol;                  // deflation tolerance (0: fixed iteration count)
};

// copy src -> dst for active points (m x npts, column-major), one warp per point
// dst(:, p) = src(:, p) and the safe solve's right-hand-side set-up in the same pass (what
// init_rhs_kernel does with every row active): G_p = max_l |dst(l, p)|, e_p = 0, and the
// non-finite shift flag -- one read of the Lanczos vector instead of two.
__global__ void copy_init_rhs_kernel(const cplx *__restrict__ src, cplx *__restrict__ dst, int64_t m,
                                     int64_t npts, const cplx *__restrict__ shifts, double *__restrict__ G,
                                     int *__restrict__ e, int *__restrict__ nonfinite) {
    pdl_wait();
    int lane = threadIdx.x & 31;
    int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t p = w; p < npts; p += nw) {
        const cplx *s = src + p * m;
        cplx *d = dst + p * m;
        double g = 0.0;
        for (int64_t i = lane; i < m; i += 32) {
            const cplx v = s[i];
            d[i] = v;
            g = fmax(g, S<cplx>::mod(v));
        }
        g = warp_max(g);
        if (lane == 0) {
            G[p] = g;
            e[p] = 0;
            if (shifts && nonfinite && !(S<cplx>::mod(shifts[p]) <= 1.7976931348623157e308)) atomicExch(nonfinite, 1);
        }
    }
}

__global__ void lanczos_init_kernel(const cplx *__restrict__ v0, LanczosState st, int64_t m,
                                    int64_t npts) {
    int lane = threadIdx.x & 31;
    int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t p = w; p < npts; p += nw) {
        for (int64_t i = lane; i < m; i += 32) {
            st.V[p * m + i] = v0[i];
            st.Vp[p * m + i] = make_double2(0.0, 0.0);
        }
        if (lane == 0) {
            st.kdone[p] = 0; st.active[p] = 1; st.flags[p] = 0;
            st.amax[p] = 0.0; st.beta_prev[p] = 0.0; st.sigma[p] = 0.0; st.theta_prev[p] = 0.0;
        }
    }
}

// One Lanczos step for every active point, after y = (U - zI)^{-1} v (in Y, exponent e1) and
// w = (U - zI)^{-H} y (in W, exponent e2).
__global__ void lanczos_step_kernel(LanczosState st, int64_t m, int64_t nslots, int it, int iters) {
    pdl_wait();
    int lane = threadIdx.x & 31;
    int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    const int64_t npts = st.npts;
    for (int64_t sl = w; sl < nslots; sl += nw) {
        const int64_t p = st.pid[sl];
        if (!st.active[p]) continue;
        const cplx *V = st.V + sl * m, *Vp = st.Vp + sl * m;
        cplx *W = st.W + sl * m;
        const cplx *Y = st.Y + sl * m;
        int e1 = st.e1[sl], e2 = st.e2[sl];
        if (e1 < 0 || e2 < 0) {
            // near-singular point (R25): sigma <= c1 / ||y||_2, scaled 2-norm
            double s = 0.0;
            for (int64_t i = lane; i < m; i += 32) s = fmax(s, fmax(fabs(Y[i].x), fabs(Y[i].y)));
            s = warp_max(s);
            double acc = 0.0;
            if (s > 0.0)
                for (int64_t i = lane; i < m; i += 32) {
                    double a = Y[i].x / s, b = Y[i].y / s;
                    acc += a * a + b * b;
                }
            acc = warp_sum(acc);
            if (lane == 0) {
                double ny = s * sqrt(acc);
                st.sigma[p] = ldexp(1.0 / ny, e1);
                st.flags[p] = 1;
                st.active[p] = 0;
            }
            continue;
        }
        double a = 0.0;                                                   // alpha = Re(v^H w)
        for (int64_t i = lane; i < m; i += 32) a += V[i].x * W[i].x + V[i].y * W[i].y;
        a = warp_sum(a);
        double bp = st.beta_prev[p], bsq = 0.0;
        for (int64_t i = lane; i < m; i += 32) {                          // w -= alpha v + beta v_prev
            cplx wi = W[i], vi = V[i], pi = Vp[i];
            wi.x = (wi.x - a * vi.x) - bp * pi.x;
            wi.y = (wi.y - a * vi.y) - bp * pi.y;
            W[i] = wi;
            bsq += wi.x * wi.x + wi.y * wi.y;
        }
        bsq = warp_sum(bsq);
        double b = sqrt(bsq);
        int k = st.kdone[p];
        double amax = fmax(st.amax[p], a);
        bool brk = b <= double(m) * 0x1p-52 * amax;                       // Krylov space exhausted
        if (!brk && it + 1 < iters) {   // v_next = w / beta in W's buffer; the host then rotates
            double binv = 1.0 / b;      // (V, V_prev, W) <- (W, V, V_prev) instead of copying
            for (int64_t i = lane; i < m; i += 32) {
                cplx wi = W[i];
                W[i] = make_double2(wi.x * binv, wi.y * binv);
            }
        }
        if (lane == 0) {
            st.alpha[int64_t(k) * npts + p] = a;
            st.beta[int64_t(k) * npts + p] = b;
            st.kdone[p] = k + 1;
            st.amax[p] = amax;
            st.beta_prev[p] = b;
            if (brk) st.active[p] = 0;
        }
    }
}

// The same step with one CTA per slot and the point's vectors in registers (m <= kLsThreads *
// kLsR): one read of V, V_prev and W and one write of W, where the warp-per-point kernel above
// passes over W three times (alpha, the update, the scaling) -- the step is HBM-bound.  Same
// operations per element; alpha and ||w||^2 are summed in another order (a block reduction).
constexpr int kLsThreads = 128, kLsR = 8;
__device__ __forceinline__ double ls_block_sum(double v, double *red) {
    v = warp_sum(v);
    __syncthreads();                              // (red reused by the previous reduction)
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    return __dadd_rn(__dadd_rn(red[0], red[1]), __dadd_rn(red[2], red[3]));
}
__device__ __forceinline__ double ls_block_max(double v, double *red) {
    v = warp_max(v);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    return fmax(fmax(red[0], red[1]), fmax(red[2], red[3]));
}
__global__ void __launch_bounds__(kLsThreads) lanczos_step_reg_kernel(LanczosState st, int64_t m, int64_t nslots,
                                                                      int it, int iters) {
    pdl_wait();
    __shared__ double red[kLsThreads / 32];
    const int tid = threadIdx.x;
    for (int64_t sl = blockIdx.x; sl < nslots; sl += gridDim.x) {
        const int64_t p = st.pid[sl];
        if (!st.active[p]) continue;                                      // (uniform in the CTA)
        const cplx *V = st.V + sl * m, *Vp = st.Vp + sl * m;
        cplx *W = st.W + sl * m;
        const cplx *Y = st.Y + sl * m;
        const int e1 = st.e1[sl], e2 = st.e2[sl];
        if (e1 < 0 || e2 < 0) {
            // near-singular point (R25): sigma <= c1 / ||y||_2, scaled 2-norm
            double s = 0.0;
            for (int64_t i = tid; i < m; i += kLsThreads) s = fmax(s, fmax(fabs(Y[i].x), fabs(Y[i].y)));
            s = ls_block_max(s, red);
            double acc = 0.0;
            if (s > 0.0)
                for (int64_t i = tid; i < m; i += kLsThreads) {
                    double a = Y[i].x / s, b = Y[i].y / s;
                    acc += a * a + b * b;
                }
            acc = ls_block_sum(acc, red);
            if (tid == 0) {
                double ny = s * sqrt(acc);
                st.sigma[p] = ldexp(1.0 / ny, e1);
                st.flags[p] = 1;
                st.active[p] = 0;
            }
            continue;
        }
        cplx vr[kLsR], wr[kLsR];
#pragma unroll
        for (int r = 0; r < kLsR; r++) {
            const int64_t i = tid + int64_t(r) * kLsThreads;
            vr[r] = i < m ? V[i] : make_double2(0.0, 0.0);
            wr[r] = i < m ? W[i] : make_double2(0.0, 0.0);
        }
        double a = 0.0;                                                   // alpha = Re(v^H w)
#pragma unroll
        for (int r = 0; r < kLsR; r++) a += vr[r].x * wr[r].x + vr[r].y * wr[r].y;
        a = ls_block_sum(a, red);
        const double bp = st.beta_prev[p];
        double bsq = 0.0;
#pragma unroll
        for (int r = 0; r < kLsR; r++) {                                  // w -= alpha v + beta v_prev
            const int64_t i = tid + int64_t(r) * kLsThreads;
            const cplx pi = i < m ? Vp[i] : make_double2(0.0, 0.0);
            wr[r].x = (wr[r].x - a * vr[r].x) - bp * pi.x;
            wr[r].y = (wr[r].y - a * vr[r].y) - bp * pi.y;
            bsq += wr[r].x * wr[r].x + wr[r].y * wr[r].y;
        }
        bsq = ls_block_sum(bsq, red);
        const double b = sqrt(bsq);
        const int k = st.kdone[p];
        const double amax = fmax(st.amax[p], a);
        const bool brk = b <= double(m) * 0x1p-52 * amax;                 // Krylov space exhausted
        const double binv = (!brk && it + 1 < iters) ? 1.0 / b : 1.0;     // v_next = w / beta in W
#pragma unroll
        for (int r = 0; r < kLsR; r++) {
            const int64_t i = tid + int64_t(r) * kLsThreads;
            if (i < m) W[i] = (!brk && it + 1 < iters) ? make_double2(wr[r].x * binv, wr[r].y * binv) : wr[r];
        }
        if (tid == 0) {
            st.alpha[int64_t(k) * st.npts + p] = a;
            st.beta[int64_t(k) * st.npts + p] = b;
            st.kdone[p] = k + 1;
            st.amax[p] = amax;
            st.beta_prev[p] = b;
            if (brk) st.active[p] = 0;
        }
    }
}

// lambda_max of the k x k tridiagonal (alpha, beta) by Sturm bisection (R14); sigma = 1/sqrt.
__device__ inline int sturm_below_dev(const double *al, const double *be, int64_t stride, int k,
                                      double x, double pivmin) {
    int cnt = 0;
    double q = al[0] - x;
    if (fabs(q) < pivmin) q = -pivmin;
    if (q < 0) cnt++;
    for (int i = 1; i < k; i++) {
        double b = be[int64_t(i - 1) * stride];
        q = (al[int64_t(i) * stride] - x) - (b * b) / q;
        if (fabs(q) < pivmin) q = -pivmin;
        if (q < 0) cnt++;
    }
    return cnt;
}

// lambda_max of the k x k tridiagonal (al[i * stride], be[i * stride]) by Sturm bisection (R14).
__device__ inline double tridiag_lmax_dev(const double *al, const double *be, int64_t stride, int k) {
    if (k == 1) return al[0];
    double lo = 1.7976931348623157e308, hi = -1.7976931348623157e308, b2 = 0.0;
    for (int i = 0; i < k; i++) {
        double r = (i > 0 ? fabs(be[int64_t(i - 1) * stride]) : 0.0) + (i < k - 1 ? fabs(be[int64_t(i) * stride]) : 0.0);
        double ai = al[int64_t(i) * stride];
        lo = fmin(lo, ai - r);
        hi = fmax(hi, ai + r);
        if (i < k - 1) { double b = be[int64_t(i) * stride]; b2 = fmax(b2, b * b); }
    }
    double pivmin = 2.2250738585072014e-308 * fmax(b2, 1.0);
    for (int itb = 0; itb < 400; itb++) {
        double wd = fmax(fabs(lo), fabs(hi));
        if (hi - lo <= 4.0 * 0x1p-52 * wd) break;
        double mid = 0.5 * (lo + hi);
        if (mid <= lo || mid >= hi) break;
        if (sturm_below_dev(al, be, stride, k, mid, pivmin) == k) hi = mid; else lo = mid;
    }
    return 0.5 * (lo + hi);
}

__global__ void bisect_sigma_kernel(LanczosState st, int64_t npts) {
    int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= npts || (st.flags[p] & 1)) return;
    int k = st.kdone[p];
    if (k <= 0) { st.sigma[p] = __longlong_as_double(0x7ff0000000000000ll); return; }
    const double lmax = tridiag_lmax_dev(st.alpha + p, st.beta + p, npts, k);
    st.sigma[p] = lmax > 0.0 ? 1.0 / sqrt(lmax) : __longlong_as_double(0x7ff0000000000000ll);
}

// SpectralCloud deflation (R33), one thread per slot: after step k (>= 2) a point whose Ritz value
// moved by at most tol theta_k leaves the batch.
__global__ void converge_kernel(LanczosState st, int64_t nslots) {
    int64_t sl = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (sl >= nslots) return;
    const int64_t p = st.pid[sl];
    if (!st.active[p]) return;
    const int k = st.kdone[p];
    const double th = tridiag_lmax_dev(st.alpha + p, st.beta + p, st.npts, k);
    if (k >= 2 && fabs(th - st.theta_prev[p]) <= st.tol * th) st.active[p] = 0;
    else st.theta_prev[p] = th;
}

// Stable compaction of the active slots (one block): newpid[j] = pid[src[j]] for the j-th slot
// still active, *count = number kept.
__global__ void compact_slots_kernel(const int *__restrict__ pid, const int *__restrict__ active, int64_t nslots,
                                     int *__restrict__ newpid, int *__restrict__ src, int *__restrict__ count) {
    __shared__ int warp_tot[32];
    __shared__ int base;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nwarp = blockDim.x >> 5;
    if (tid == 0) base = 0;
    __syncthreads();
    for (int64_t c0 = 0; c0 < nslots; c0 += blockDim.x) {
        const int64_t sl = c0 + tid;
        const int keep = sl < nslots && active[pid[sl]] ? 1 : 0;
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        const int inwarp = __popc(bal & ((1u << lane) - 1u));
        if (lane == 0) warp_tot[wid] = __popc(bal);
        __syncthreads();
        int off = base;
        for (int w = 0; w < wid; w++) off += warp_tot[w];
        if (keep) {
            newpid[off + inwarp] = pid[sl];
            src[off + inwarp] = int(sl);
        }
        __syncthreads();
        if (tid == 0) {
            int t = 0;
            for (int w = 0; w < nwarp; w++) t += warp_tot[w];
            base += t;
        }
        __syncthreads();
    }
    if (tid == 0) *count = base;
}

// dst(:, j) = src(:, idx[j]) for j < n (m x n complex columns), one warp per column
__global__ void gather_cols_kernel(const cplx *__restrict__ srcv, cplx *__restrict__ dst, const int *__restrict__ idx,
                                   int64_t m, int64_t n) {
    int lane = threadIdx.x & 31;
    int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t j = w; j < n; j += nw) {
        const cplx *s = srcv + int64_t(idx[j]) * m;
        cplx *d = dst + j * m;
        for (int64_t i = lane; i < m; i += 32) d[i] = s[i];
    }
}

__global__ void gather_z_kernel(const cplx *__restrict__ z, const int *__restrict__ pid, cplx *__restrict__ zc, int64_t n) {
    int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j < n) zc[j] = z[pid[j]];
}

__global__ void iota_kernel(int *__restrict__ v, int64_t n) {
    int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j < n) v[j] = int(j);
}

// flags bit1 (R33): deflation on and the point neither settled nor stopped; its = steps taken
__global__ void cloud_finish_kernel(LanczosState st, int64_t npts, int32_t *__restrict__ its) {
    int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= npts) return;
    if (st.tol > 0.0 && st.active[p] && !(st.flags[p] & 1)) st.flags[p] |= 2;
    if (its) its[p] = st.kdone[p];
}

}  // namespace mstrsm
