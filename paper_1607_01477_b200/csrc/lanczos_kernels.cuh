// lanczos_kernels.cuh -- a.7 inverse-Lanczos step of the Van Loan / Lui pseudospectra driver
// (R14, R25).  One warp per grid point; all points advance in lockstep, each operator
// application being one op-N and one op-C multi-shift solve over all points.
#pragma once
#include "common.cuh"

namespace mstrsm {

struct LanczosState {
    cplx *V, *Vp, *W, *Y;        // m x npts each (column per point)
    double *alpha, *beta;        // iters x npts
    int *kdone, *active, *flags;
    double *amax, *beta_prev, *sigma;
    const int *e1, *e2;          // exponents of the two solves of this step
};

// copy src -> dst for active points (m x npts, column-major), one warp per point
__global__ void copy_cols_kernel(const cplx *__restrict__ src, cplx *__restrict__ dst, int64_t m,
                                 int64_t npts) {
    int lane = threadIdx.x & 31;
    int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t p = w; p < npts; p += nw) {
        const cplx *s = src + p * m;
        cplx *d = dst + p * m;
        for (int64_t i = lane; i < m; i += 32) d[i] = s[i];
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
            st.amax[p] = 0.0; st.beta_prev[p] = 0.0; st.sigma[p] = 0.0;
        }
    }
}

// One Lanczos step for every active point, after y = (U - zI)^{-1} v (in Y, exponent e1) and
// w = (U - zI)^{-H} y (in W, exponent e2).
__global__ void lanczos_step_kernel(LanczosState st, int64_t m, int64_t npts, int it, int iters) {
    int lane = threadIdx.x & 31;
    int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t p = w; p < npts; p += nw) {
        if (!st.active[p]) continue;
        cplx *V = st.V + p * m, *Vp = st.Vp + p * m, *W = st.W + p * m;
        const cplx *Y = st.Y + p * m;
        int e1 = st.e1[p], e2 = st.e2[p];
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
        if (!brk && it + 1 < iters) {
            double binv = 1.0 / b;
            for (int64_t i = lane; i < m; i += 32) {
                cplx wi = W[i];
                Vp[i] = V[i];
                V[i] = make_double2(wi.x * binv, wi.y * binv);
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

__global__ void bisect_sigma_kernel(LanczosState st, int64_t npts) {
    int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= npts || st.flags[p]) return;
    int k = st.kdone[p];
    const double *al = st.alpha + p, *be = st.beta + p;
    double lmax;
    if (k <= 0) { st.sigma[p] = __longlong_as_double(0x7ff0000000000000ll); return; }
    if (k == 1) {
        lmax = al[0];
    } else {
        double lo = 1.7976931348623157e308, hi = -1.7976931348623157e308, b2 = 0.0;
        for (int i = 0; i < k; i++) {
            double r = (i > 0 ? fabs(be[int64_t(i - 1) * npts]) : 0.0) + (i < k - 1 ? fabs(be[int64_t(i) * npts]) : 0.0);
            double ai = al[int64_t(i) * npts];
            lo = fmin(lo, ai - r);
            hi = fmax(hi, ai + r);
            if (i < k - 1) { double b = be[int64_t(i) * npts]; b2 = fmax(b2, b * b); }
        }
        double pivmin = 2.2250738585072014e-308 * fmax(b2, 1.0);
        for (int itb = 0; itb < 400; itb++) {
            double wd = fmax(fabs(lo), fabs(hi));
            if (hi - lo <= 4.0 * 0x1p-52 * wd) break;
            double mid = 0.5 * (lo + hi);
            if (mid <= lo || mid >= hi) break;
            if (sturm_below_dev(al, be, npts, k, mid, pivmin) == k) hi = mid; else lo = mid;
        }
        lmax = 0.5 * (lo + hi);
    }
    st.sigma[p] = lmax > 0.0 ? 1.0 / sqrt(lmax) : __longlong_as_double(0x7ff0000000000000ll);
}

}  // namespace mstrsm
