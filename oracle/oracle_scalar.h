/*
 * oracle/oracle_scalar.h -- scalar arithmetic used by the CPU oracle.
 *
 * TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load the oracle.
 * Shares no code with paper_1607_01477_b200/ (the CUDA product path).
 *
 * Conventions (readings R7, R24):
 *   - IEEE fp64, round-to-nearest, built with -ffp-contract=off (no FMA).
 *   - complex multiply: textbook (ac - bd) + (ad + bc) i.
 *   - complex divide: Smith's algorithm.
 *   - |z| = sqrt(re^2 + im^2) evaluated after a power-of-two prescale so
 *     that neither square can overflow or underflow (exact prescale, one
 *     correctly rounded sqrt).  For real scalars |x| = fabs(x).
 */
#ifndef ORACLE_SCALAR_H
#define ORACLE_SCALAR_H

#include <math.h>
#include <stdint.h>

typedef struct { double re, im; } ozc;   /* layout = double _Complex */

/* ---- real ---------------------------------------------------------- */
static inline double d_sub(double a, double b) { return a - b; }
static inline double d_mul(double a, double b) { return a * b; }
static inline double d_div(double a, double b) { return a / b; }
static inline double d_mod(double a) { return fabs(a); }
static inline double d_conj(double a) { return a; }
static inline double d_neg(double a) { return -a; }
static inline double d_real(double r) { return r; }
static inline int    d_is_zero(double a) { return a == 0.0; }
static inline double d_ldexp(double a, int k) { return ldexp(a, k); }
static inline double d_zero(void) { return 0.0; }

/* ---- complex ------------------------------------------------------- */
static inline ozc z_make(double re, double im) { ozc z; z.re = re; z.im = im; return z; }
static inline ozc z_sub(ozc a, ozc b) { return z_make(a.re - b.re, a.im - b.im); }
static inline ozc z_mul(ozc a, ozc b)
{
    return z_make(a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re);
}
/* Smith (1962): divide by the larger component first. */
static inline ozc z_div(ozc a, ozc b)
{
    if (fabs(b.im) <= fabs(b.re)) {
        double r = b.im / b.re;
        double den = b.re + b.im * r;
        return z_make((a.re + a.im * r) / den, (a.im - a.re * r) / den);
    } else {
        double r = b.re / b.im;
        double den = b.im + b.re * r;
        return z_make((a.re * r + a.im) / den, (a.im * r - a.re) / den);
    }
}
/* |z| with an exact power-of-two prescale (see header comment). */
static inline double z_mod(ozc a)
{
    double x = fabs(a.re), y = fabs(a.im);
    double big = x > y ? x : y;
    if (big == 0.0) return 0.0;
    if (!(big <= 1.7976931348623157e308)) {           /* Inf or NaN */
        if (isinf(x) || isinf(y)) return INFINITY;
        return NAN;
    }
    int s = 0;
    if (big > 0x1p+500) s = -600;                      /* avoid overflow  */
    else if (big < 0x1p-500) s = 600;                  /* avoid underflow */
    x = ldexp(x, s);
    y = ldexp(y, s);
    double r = sqrt(x * x + y * y);
    return ldexp(r, -s);
}
static inline ozc    z_conj(ozc a) { return z_make(a.re, -a.im); }
static inline ozc    z_neg(ozc a) { return z_make(-a.re, -a.im); }
static inline ozc    z_real(double r) { return z_make(r, 0.0); }
static inline int    z_is_zero(ozc a) { return a.re == 0.0 && a.im == 0.0; }
static inline ozc    z_ldexp(ozc a, int k) { return z_make(ldexp(a.re, k), ldexp(a.im, k)); }
static inline ozc    z_zero(void) { return z_make(0.0, 0.0); }

#endif
