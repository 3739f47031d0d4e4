// common.cuh -- scalar types and device arithmetic for libmstrsm (sm_100a).
//
// Written independently of oracle/ (which this code never includes).  The bound arithmetic
// follows the readings of DESIGN.md §3 so that, given bit-identical inputs, the GPU makes the
// same scaling decisions as the paper's Alg. 4/5:
//   |z|   : sqrt(re^2 + im^2) with an exact power-of-two prescale, no FMA        (R7)
//   a / b : Smith's algorithm for complex, no FMA                                (R7)
//   t     : 2^-k with the smallest k >= 1 such that 2^-k a < L                   (R2)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace mstrsm {

constexpr double kOmega = 0x1p+970;   // R1: dlamch('P') / dlamch('S')

typedef double2 cplx;                 // interleaved (re, im), 16-byte aligned

// ---------------------------------------------------------------- scalar traits
template <typename T> struct S;

template <> struct S<double> {
    static constexpr bool cplx_ = false;
    __device__ __forceinline__ static double zero() { return 0.0; }
    __device__ __forceinline__ static double sub(double a, double b) { return __dsub_rn(a, b); }
    __device__ __forceinline__ static double div(double a, double b) { return __ddiv_rn(a, b); }
    __device__ __forceinline__ static double mul(double a, double b) { return __dmul_rn(a, b); }
    __device__ __forceinline__ static double mod(double a) { return fabs(a); }
    __device__ __forceinline__ static double conj(double a) { return a; }
    __device__ __forceinline__ static double neg(double a) { return -a; }
    __device__ __forceinline__ static double real(double r) { return r; }
    __device__ __forceinline__ static bool is_zero(double a) { return a == 0.0; }
    __device__ __forceinline__ static double ldx(double a, int k) { return ldexp(a, k); }
    __device__ __forceinline__ static double shfl(double a, int src) { return __shfl_sync(0xffffffffu, a, src); }
    // y - x*u (fused; rounding-level differences vs the oracle are covered by R20/R24)
    __device__ __forceinline__ static double fnms(double y, double x, double u) { return fma(-x, u, y); }
};

template <> struct S<cplx> {
    static constexpr bool cplx_ = true;
    __device__ __forceinline__ static cplx mk(double r, double i) { return make_double2(r, i); }
    __device__ __forceinline__ static cplx zero() { return mk(0.0, 0.0); }
    __device__ __forceinline__ static cplx sub(cplx a, cplx b) { return mk(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y)); }
    __device__ __forceinline__ static cplx mul(cplx a, cplx b) {
        return mk(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)), __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
    }
    // Smith (1962), without FMA contraction.
    __device__ __forceinline__ static cplx div(cplx a, cplx b) {
        if (fabs(b.y) <= fabs(b.x)) {
            double r = __ddiv_rn(b.y, b.x);
            double den = __dadd_rn(b.x, __dmul_rn(b.y, r));
            return mk(__ddiv_rn(__dadd_rn(a.x, __dmul_rn(a.y, r)), den),
                      __ddiv_rn(__dsub_rn(a.y, __dmul_rn(a.x, r)), den));
        } else {
            double r = __ddiv_rn(b.x, b.y);
            double den = __dadd_rn(b.y, __dmul_rn(b.x, r));
            return mk(__ddiv_rn(__dadd_rn(__dmul_rn(a.x, r), a.y), den),
                      __ddiv_rn(__dsub_rn(__dmul_rn(a.y, r), a.x), den));
        }
    }
    __device__ __forceinline__ static double mod(cplx a) {
        double x = fabs(a.x), y = fabs(a.y);
        double big = x > y ? x : y;
        if (big == 0.0) return 0.0;
        if (!(big <= 1.7976931348623157e308)) {
            if (isinf(x) || isinf(y)) return __longlong_as_double(0x7ff0000000000000ll);
            return __longlong_as_double(0x7ff8000000000000ll);
        }
        double s = 1.0, sinv = 1.0;
        if (big > 0x1p+500) { s = 0x1p-600; sinv = 0x1p+600; }
        else if (big < 0x1p-500) { s = 0x1p+600; sinv = 0x1p-600; }
        x = __dmul_rn(x, s);
        y = __dmul_rn(y, s);
        double r = __dsqrt_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)));
        return __dmul_rn(r, sinv);
    }
    __device__ __forceinline__ static cplx conj(cplx a) { return mk(a.x, -a.y); }
    __device__ __forceinline__ static cplx neg(cplx a) { return mk(-a.x, -a.y); }
    __device__ __forceinline__ static cplx real(double r) { return mk(r, 0.0); }
    __device__ __forceinline__ static bool is_zero(cplx a) { return a.x == 0.0 && a.y == 0.0; }
    __device__ __forceinline__ static cplx ldx(cplx a, int k) { return mk(ldexp(a.x, k), ldexp(a.y, k)); }
    __device__ __forceinline__ static cplx shfl(cplx a, int src) {
        return mk(__shfl_sync(0xffffffffu, a.x, src), __shfl_sync(0xffffffffu, a.y, src));
    }
    // y - x*u, complex, fused.
    __device__ __forceinline__ static cplx fnms(cplx y, cplx x, cplx u) {
        double re = fma(-x.x, u.x, fma(x.y, u.y, y.x));
        double im = fma(-x.x, u.y, fma(-x.y, u.x, y.y));
        return mk(re, im);
    }
};

// Smallest integer k >= 1 with ldexp(a, -k) < L (R2); a non-finite -> 1100 (R8).
__device__ __forceinline__ int minpow2(double a, double L) {
    if (!(a <= 1.7976931348623157e308)) return 1100;
    int k = ilogb(a) - ilogb(L);
    if (k < 1) k = 1;
    while (k > 1 && ldexp(a, -(k - 1)) < L) k--;
    while (!(ldexp(a, -k) < L)) k++;
    return k;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// 2^d as a double for d >= -1074 (exact); callers handle smaller d via ldexp on the value.
__device__ __forceinline__ double pow2(int d) { return ldexp(1.0, d); }

__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
// cp.async with zero fill when !valid (src-size 0).
template <int BYTES>
__device__ __forceinline__ void cp_async(void *dst, const void *src, bool valid) {
    unsigned d = smem_u32(dst);
    int sz = valid ? BYTES : 0;
    if (BYTES == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(sz));
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(d), "l"(src), "n"(BYTES), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Block partition (R9).  op N: block b covers rows [max(0, m-(b+1)nb), m-b*nb).
//                        op C: block b covers rows [b*nb, min(m, (b+1)nb)).
struct Blk { int64_t lo, hi; };
__host__ __device__ __forceinline__ Blk block_rows(int op, int64_t m, int nb, int64_t b) {
    Blk r;
    if (op == 0) { r.hi = m - b * nb; r.lo = r.hi - nb < 0 ? 0 : r.hi - nb; }
    else { r.lo = b * nb; r.hi = r.lo + nb > m ? m : r.lo + nb; }
    return r;
}

}  // namespace mstrsm

namespace mstrsm {
// Programmatic dependent launch: wait for the preceding grid in the stream (a no-op when the
// kernel was launched without the attribute).
// Phase timing of the diagonal kernels (experiment builds only, -DMSTRSM_PHASE_TIMES,
// tools/build_phase.sh): PT_MARK(pt, k) stores clock64() in slot k of this CTA's row of pt (16
// slots per CTA, pass 0); slots 0 and 12-15 hold %globaltimer (entry, exits).
#ifdef MSTRSM_PHASE_TIMES
__device__ __forceinline__ long long pt_gtime() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define PT_MARK(pt, k, cond)                                                          \
    do {                                                                              \
        if ((pt) && (cond)) (pt)[blockIdx.x * 16 + (k)] = ((k) == 0 || (k) >= 12) ? pt_gtime() : clock64(); \
    } while (0)
#else
#define PT_MARK(pt, k, cond) do { } while (0)
#endif
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
// ... and let the next grid in the stream launch now (onto the SMs this grid leaves free) rather
// than when this one completes.  Its griddepcontrol.wait still waits for this grid's completion and
// memory, so a kernel may trigger at its very start as long as its dependents touch no global
// memory before their pdl_wait (the diagonal and update kernels stage only read-only U before it).
// Used by the complex diagonal and update kernels, whose shared memory keeps a waiting dependent
// CTA off their SMs; the real path's smaller CTAs would share an SM with a waiting dependent
// (c2 1.30 -> 1.35 ms with the trigger, c4 82.1 -> 80.9 ms, c5 155.6 -> 155.4 ms).
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
}  // namespace mstrsm
