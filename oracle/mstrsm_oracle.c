/*
 * oracle/mstrsm_oracle.c -- plain, slow, obviously-correct CPU oracle for
 * the blocked (safe) multi-shift triangular solve of Moon & Poulson,
 * "Accelerating eigenvector and pseudospectra computation using blocked
 * multi-shift triangular solves", arXiv 1607.01477.
 *
 * *** TEST INFRASTRUCTURE ONLY ***
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
 * --impl reference) may load liboracle.so.  It shares no code, header,
 * constant table or helper with the CUDA product path in
 * paper_1607_01477_b200/, and neither side includes the other.
 *
 * What is here (each cited in place):
 *   oracle_mstrsm_{d,z}    Alg. 3 / Alg. 5 column by column, op N and op C
 *   oracle_norms_{d,z}     the norm pass
 *   oracle_trevc_{d,z}     Alg. 6 TriangEig with the P:503-508 shortcut
 *   oracle_pseudospectra_z Alg. "Van Loan/Lui" with a fixed
 *                          number of Lanczos steps on
 *                          (T - zI)^{-H} (T - zI)^{-1}
 *   oracle_tridiag_lmax    largest eigenvalue of a symmetric tridiagonal
 *                          matrix by Sturm-count bisection
 *
 * Parity pins: every function above is pinned by tests in
 * tests/test_oracle_pins.py; see DESIGN.md section 4 for the list.
 *
 * Build: gcc -O2 -ffp-contract=off -fPIC -shared -pthread (no -ffast-math,
 * no -march=native), see Makefile.
 */
#include <float.h>
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <unistd.h>

#include "oracle_scalar.h"

/* Omega = 2^970 = dlamch('P') / dlamch('S') (R1; "a machine-dependent
 * overflow constant"). */
#define OMEGA 0x1p+970

/* Smallest integer k >= 1 with 2^-k * a < L (R2: t = 2^-k, the smallest
 * power-of-two reduction that satisfies "t * M < Omega", P:285/P:303/P:396).
 * Exact: ldexp is exact or correctly rounded.  a non-finite -> k = 1100
 * (R8: cannot happen while max|U| <= 2^40). */
static int minpow2(double a, double L)
{
    if (!(a <= DBL_MAX)) return 1100;
    int k = ilogb(a) - ilogb(L);
    if (k < 1) k = 1;
    while (k > 1 && ldexp(a, -(k - 1)) < L) k--;
    while (!(ldexp(a, -k) < L)) k++;
    return k;
}

static void run_threads(void *(*fn)(void *), void *arg, int nthreads)
{
    if (nthreads <= 0) {
        long c = sysconf(_SC_NPROCESSORS_ONLN);
        nthreads = c > 0 ? (int)c : 1;
    }
    if (nthreads == 1) { fn(arg); return; }
    pthread_t *t = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    for (int i = 0; i < nthreads; i++) pthread_create(&t[i], NULL, fn, arg);
    for (int i = 0; i < nthreads; i++) pthread_join(t[i], NULL);
    free(t);
}

/* ---- real instantiation ---- */
#define S double
#define P_ d_
#define FN(name) name##_d
#include "oracle_algo.inc"
#include "oracle_gen.inc"
#undef S
#undef P_
#undef FN

/* ---- complex instantiation ---- */
#define S ozc
#define P_ z_
#define FN(name) name##_z
#include "oracle_algo.inc"
#include "oracle_gen.inc"
#undef S
#undef P_
#undef FN

/* ------------------------------------------------------------------ */
/* Largest eigenvalue of the k x k symmetric tridiagonal matrix with
 * diagonal a[0..k) and off-diagonal b[0..k-1), by bisection on Sturm
 * counts (R14).  Starts from the Gershgorin interval; stops when the
 * interval is <= 4 * 2^-52 * max(|lo|, |hi|) wide. */
static int sturm_below(const double *a, const double *b, int k, double x, double pivmin)
{
    int cnt = 0;
    double q = a[0] - x;
    if (fabs(q) < pivmin) q = -pivmin;
    if (q < 0) cnt++;
    for (int i = 1; i < k; i++) {
        q = (a[i] - x) - (b[i - 1] * b[i - 1]) / q;
        if (fabs(q) < pivmin) q = -pivmin;
        if (q < 0) cnt++;
    }
    return cnt;
}

double oracle_tridiag_lmax(const double *a, const double *b, int k)
{
    if (k <= 0) return 0.0;
    if (k == 1) return a[0];
    double lo = INFINITY, hi = -INFINITY, b2 = 0.0;
    for (int i = 0; i < k; i++) {
        double r = (i > 0 ? fabs(b[i - 1]) : 0.0) + (i < k - 1 ? fabs(b[i]) : 0.0);
        if (a[i] - r < lo) lo = a[i] - r;
        if (a[i] + r > hi) hi = a[i] + r;
        if (i < k - 1 && b[i] * b[i] > b2) b2 = b[i] * b[i];
    }
    double pivmin = DBL_MIN * (b2 > 1.0 ? b2 : 1.0);
    for (int it = 0; it < 400; it++) {
        double w = fabs(lo) > fabs(hi) ? fabs(lo) : fabs(hi);
        if (hi - lo <= 4.0 * 0x1p-52 * w) break;
        double mid = 0.5 * (lo + hi);
        if (mid <= lo || mid >= hi) break;
        if (sturm_below(a, b, k, mid, pivmin) == k) hi = mid; else lo = mid;
    }
    return 0.5 * (lo + hi);
}

/* ------------------------------------------------------------------ */
/* Van Loan / Lui pseudospectra: for every point z,
 * sigma_min(T - zI) = 1 / sqrt(lambda_max((T - zI)^{-H} (T - zI)^{-1}))
 * (P:600-604), lambda_max by `iters` Lanczos steps (P:634-638,
 * R14) from the shared unit start vector v0.  Each operator application is
 * one op-N and one op-C safe solve.
 * flags bit0: a solve rescaled (c < 1); sigma is then the rigorous upper
 * bound c1 / ||y||_2 from that step (R25). */
typedef struct {
    const ozc *U; int64_t ldu, m;
    const ozc *z; int64_t npts; int iters;
    const ozc *v0; double *sigma; int32_t *flags; int nb;
    double tol; int32_t *its;       /* SpectralCloud deflation (R33); tol = 0: fixed iters */
    const double *cnlN, *PN, *cnlC, *PC; double deltaN, deltaC;
    int64_t next; pthread_mutex_t mu;
} ps_job_t;

static double znorm2_scaled(const ozc *y, int64_t m)
{
    double s = 0.0;
    for (int64_t i = 0; i < m; i++) {
        double a = fabs(y[i].re) > fabs(y[i].im) ? fabs(y[i].re) : fabs(y[i].im);
        if (a > s) s = a;
    }
    if (s == 0.0) return 0.0;
    double acc = 0.0;
    for (int64_t i = 0; i < m; i++) {
        double p = y[i].re / s, q = y[i].im / s;
        acc = acc + (p * p + q * q);
    }
    return s * sqrt(acc);
}

static void *ps_worker(void *arg)
{
    ps_job_t *J = (ps_job_t *)arg;
    int64_t m = J->m;
    ozc *v = (ozc *)malloc(sizeof(ozc) * (size_t)m);
    ozc *vp = (ozc *)malloc(sizeof(ozc) * (size_t)m);
    ozc *y = (ozc *)malloc(sizeof(ozc) * (size_t)m);
    ozc *w = (ozc *)malloc(sizeof(ozc) * (size_t)m);
    double *al = (double *)malloc(sizeof(double) * (size_t)(J->iters + 1));
    double *be = (double *)malloc(sizeof(double) * (size_t)(J->iters + 1));
    for (;;) {
        pthread_mutex_lock(&J->mu);
        int64_t p = J->next++;
        pthread_mutex_unlock(&J->mu);
        if (p >= J->npts) break;
        ozc z = J->z[p];
        for (int64_t i = 0; i < m; i++) { v[i] = J->v0[i]; vp[i] = z_zero(); }
        double beta_prev = 0.0, amax = 0.0, sigma = 0.0, theta_prev = 0.0;
        int k = 0, flag = 0, conv = 0, brk = 0;
        for (int it = 0; it < J->iters; it++) {
            for (int64_t i = 0; i < m; i++) y[i] = v[i];
            int e1 = col_N_z(J->U, J->ldu, m, z, y, m, 1, J->nb, J->cnlN, J->PN, J->deltaN);
            int e2 = 0;
            if (e1 == 0) {
                for (int64_t i = 0; i < m; i++) w[i] = y[i];
                e2 = col_C_z(J->U, J->ldu, m, z, w, 1, J->nb, J->cnlC, J->PC, J->deltaC);
            }
            if (e1 < 0 || e2 < 0) {
                double ny = znorm2_scaled(y, m);
                sigma = ldexp(1.0 / ny, e1);
                flag = 1;
                break;
            }
            double a = 0.0;                                   /* alpha = Re(v^H w) */
            for (int64_t i = 0; i < m; i++) a = a + (v[i].re * w[i].re + v[i].im * w[i].im);
            for (int64_t i = 0; i < m; i++) {                 /* w -= alpha v + beta v_prev */
                w[i].re = (w[i].re - a * v[i].re) - beta_prev * vp[i].re;
                w[i].im = (w[i].im - a * v[i].im) - beta_prev * vp[i].im;
            }
            double bsq = 0.0;
            for (int64_t i = 0; i < m; i++) bsq = bsq + (w[i].re * w[i].re + w[i].im * w[i].im);
            double b = sqrt(bsq);
            al[k] = a; be[k] = b; k++;
            if (a > amax) amax = a;
            if (b <= (double)m * 0x1p-52 * amax) { brk = 1; break; }   /* Krylov space exhausted */
            if (J->tol > 0.0) {       /* R33: the point leaves the batch when its estimate settles */
                double theta = oracle_tridiag_lmax(al, be, k);
                if (k >= 2 && fabs(theta - theta_prev) <= J->tol * theta) { conv = 1; break; }
                theta_prev = theta;
            }
            for (int64_t i = 0; i < m; i++) {
                vp[i] = v[i];
                v[i].re = w[i].re / b;
                v[i].im = w[i].im / b;
            }
            beta_prev = b;
        }
        if (!flag) {
            double lmax = oracle_tridiag_lmax(al, be, k);
            sigma = lmax > 0.0 ? 1.0 / sqrt(lmax) : INFINITY;
        }
        J->sigma[p] = sigma;
        /* bit1: tol > 0 and neither converged nor exhausted within iters steps */
        if (J->tol > 0.0 && !flag && !conv && !brk) flag |= 2;
        if (J->flags) J->flags[p] = flag;
        if (J->its) J->its[p] = k;
    }
    free(v); free(vp); free(y); free(w); free(al); free(be);
    return NULL;
}

/* SpectralCloud: as oracle_pseudospectra_z, but with tol > 0 a point stops after
 * the first step k >= 2 with |theta_k - theta_{k-1}| <= tol theta_k, theta_k = lambda_max of the
 * k-step tridiagonal (R33); its[p] = Lanczos steps taken; flags bit1 = not settled in `iters`. */
int oracle_spectral_cloud_z(const ozc *U, int64_t ldu, int64_t m, const ozc *z,
                            int64_t npts, int iters, double tol, const ozc *v0, double *sigma,
                            int32_t *flags, int32_t *its, int nb, int nthreads)
{
    if (m < 1 || npts < 0 || iters < 1 || nb < 1) return -1;
    if (npts == 0) return 0;
    int64_t nblk = (m + nb - 1) / nb;
    double *cnlN = (double *)calloc((size_t)m, sizeof(double));
    double *cnlC = (double *)calloc((size_t)m, sizeof(double));
    double *PN = (double *)calloc((size_t)nblk, sizeof(double));
    double *PC = (double *)calloc((size_t)nblk, sizeof(double));
    double uN = 0.0, uC = 0.0;
    norms_z(0, U, ldu, m, nb, cnlN, PN, &uN);
    norms_z(1, U, ldu, m, nb, cnlC, PC, &uC);
    ps_job_t J;
    J.U = U; J.ldu = ldu; J.m = m; J.z = z; J.npts = npts; J.iters = iters;
    J.v0 = v0; J.sigma = sigma; J.flags = flags; J.nb = nb;
    J.tol = tol > 0.0 ? tol : 0.0; J.its = its;
    J.cnlN = cnlN; J.PN = PN; J.cnlC = cnlC; J.PC = PC;
    J.deltaN = uN > 0.0 ? ldexp(uN, -52) : DBL_MIN;
    J.deltaC = uC > 0.0 ? ldexp(uC, -52) : DBL_MIN;
    J.next = 0;
    pthread_mutex_init(&J.mu, NULL);
    run_threads(ps_worker, &J, nthreads);
    pthread_mutex_destroy(&J.mu);
    free(cnlN); free(cnlC); free(PN); free(PC);
    return 0;
}

int oracle_pseudospectra_z(const ozc *U, int64_t ldu, int64_t m, const ozc *z,
                           int64_t npts, int iters, const ozc *v0, double *sigma,
                           int32_t *flags, int nb, int nthreads)
{
    return oracle_spectral_cloud_z(U, ldu, m, z, npts, iters, 0.0, v0, sigma, flags, NULL, nb, nthreads);
}

/* Exposed for tests: the scalar helpers, so the pins can exercise them. */
double oracle_zmod(double re, double im) { return z_mod(z_make(re, im)); }
void oracle_zdiv(double ar, double ai, double br, double bi, double *out)
{
    ozc q = z_div(z_make(ar, ai), z_make(br, bi));
    out[0] = q.re; out[1] = q.im;
}
int oracle_minpow2(double a, double L) { return minpow2(a, L); }
