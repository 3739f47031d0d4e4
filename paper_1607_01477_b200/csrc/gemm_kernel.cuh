// gemm_kernel.cuh -- a.5, the shift-free substitution step shared by every shift:
//
//     C(i,j) <- 2^{d_j} C(i,j) - sum_k A(i,k) X(k,j)
//
//   op N: C = B(0:lo, cols), A = U(0:lo, lo:hi),         X = B(lo:hi, cols)
//   op C: C = B(hi:m, cols), A = U(lo:hi, hi:m)^H,       X = B(lo:hi, cols)
//
// d_j <= 0 is the exponent change of column j in this block (safe variant, lazy form of the
// xSCAL rescales of P:378-380 and P:398 applied to rows I0); d = 0 / null for the plain solve.
//
// FP64 tensor cores: sm_100a has no tcgen05 f64 kind, so the contraction is the warp-level
// mma.sync.aligned.m8n8k4.f64 (SASS DMMA.8x8x4).  Complex = 4 real DMMA sub-products sharing
// the A/X fragments (Cr += Ar Xr - Ai Xi, Ci += Ar Xi + Ai Xr).  Operand tiles are staged by
// cp.async (LDGSTS) into a 3-stage shared-memory ring with XOR swizzles that make every fragment
// load conflict-free; 4 warps (2x2) per CTA, 2 CTAs per SM.
#pragma once
#include "common.cuh"

namespace mstrsm {

// Not volatile: the MMA is a pure function of its operands, so the compiler may interleave the
// independent accumulator chains.
__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(c0), "+d"(c1)
        : "d"(a), "d"(b));
}

template <typename T>
struct GemmArgs {
    const T *U; int64_t ldu;
    T *B; int64_t ldb;
    int64_t M, N; int K;
    int64_t a_r0, a_c0;    // op N: A(i,k) = U(a_r0+i, a_c0+k); op C: A(i,k) = conj(U(a_r0+k, a_c0+i))
    int64_t c_r0, x_r0;    // C rows start, X rows start
    const T *X; int64_t ldx;   // X(k,j) = X[(x_r0 + k) + (col0 + j) * ldx] (X = B for the U product;
                               // the generalized solve's V product reads C = -lambda X from a buffer)
    // complex 3M only (nullable): the sums Re + Im of the operands, precomputed:
    //   As indexed like A (op N: As[(a_r0+i) + (a_c0+k) ldas]; op C: As[(a_r0+k) + (a_c0+i) ldas],
    //   there holding Re - Im = Re(conj)), Xs(k,j) = Xs[k + (col0 + j) ldxs]
    const double *As; int64_t ldas;
    const double *Xsum; int64_t ldxs;
    int64_t col0;          // first column
    const int *dblk;       // per-column exponent delta (nullable)
    long long *pt;         // phase times (MSTRSM_PHASE_TIMES builds only; nullable)
    int early_a;           // gemm_update_kernel: the first stages' A tiles (read-only U) before the wait
    int trig;              // gemm_update_kernel: let the next grid launch at this one's start
};

// Tile geometry.  Complex: CTA 64 (rows) x 64 (cols), warp 32x32, BK = 16.
//                 Real:    CTA 64 x 64, warp 32x32, BK = 16.
template <typename T> struct GemmCfg;
template <> struct GemmCfg<cplx> { static constexpr int BM = 64, BN = 64, BK = 16, WM = 32, WN = 32; };
template <> struct GemmCfg<double> { static constexpr int BM = 64, BN = 64, BK = 16, WM = 32, WN = 32; };
constexpr int kGemmStages = 3;
constexpr int kGemmThreads = 128;

template <typename T>
__host__ __device__ constexpr int gemm_stage_elems() {
    return GemmCfg<T>::BM * GemmCfg<T>::BK + GemmCfg<T>::BN * GemmCfg<T>::BK;
}
template <typename T>
__host__ __device__ constexpr int gemm_smem_bytes() {
    return kGemmStages * gemm_stage_elems<T>() * int(sizeof(T));
}

// Swizzled smem offsets (in elements).
//  A, op N ("k-major", m contiguous): element (k, m) of a BK x BM tile.
//  A, op C and X ("row-major over the BM/BN index", k contiguous): element (r, k) of BMxBK / BNxBK.
template <typename T>
__device__ __forceinline__ int offA_kmajor(int k, int mm) {
    constexpr int BM = GemmCfg<T>::BM;
    if (S<T>::cplx_) return k * BM + (mm ^ ((k & 3) << 1));      // 16-B elements: 8 per 128 B
    else return k * BM + (mm ^ ((k & 3) << 2));                  // 8-B elements: 16 per 128 B
}
template <typename T>
__device__ __forceinline__ int offRK(int r, int k) {
    constexpr int BK = GemmCfg<T>::BK;
    if (S<T>::cplx_) return r * BK + (k ^ ((r & 1) << 2));
    else return r * BK + (k ^ ((r & 3) << 2));
}

template <typename T, bool OPC>
__global__ void __launch_bounds__(kGemmThreads, 2) gemm_update_kernel(GemmArgs<T> g) {
    constexpr int BM = GemmCfg<T>::BM, BN = GemmCfg<T>::BN, BK = GemmCfg<T>::BK;
    constexpr int WM = GemmCfg<T>::WM, WN = GemmCfg<T>::WN;
    constexpr int MI = WM / 8, NI = WN / 8;
    constexpr bool CPX = S<T>::cplx_;
    constexpr int ESZ = sizeof(T);
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T *smem = reinterpret_cast<T *>(smem_raw);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp & 1, wn = warp >> 1;
    const int gq = lane >> 2, tq = lane & 3;
    const int64_t m0 = int64_t(blockIdx.x) * BM;
    const int64_t n0 = int64_t(blockIdx.y) * BN;
    const int nk = (g.K + BK - 1) / BK;

    // per-column epilogue scale 2^{d_j} of this tile (the lazy xSCAL of P:378-380 / P:398), read
    // from dblk once per CTA while the pipeline fills
    __shared__ double s_sc[BN];
    __shared__ int s_d[BN];
    auto stageA = [&](int s) { return smem + s * gemm_stage_elems<T>(); };
    auto stageX = [&](int s) { return smem + s * gemm_stage_elems<T>() + BM * BK; };

    auto load_A = [&](int s, int kt) {
        T *As = stageA(s);
        const int k0 = kt * BK;
        if (!OPC) {
            // BK columns of U, BM contiguous rows each
#pragma unroll
            for (int it = 0; it < (BM * BK) / kGemmThreads; it++) {
                int idx = it * kGemmThreads + tid;
                int mm = idx % BM, k = idx / BM;
                int64_t gi = m0 + mm;
                int gk = k0 + k;
                bool v = gi < g.M && gk < g.K;
                const T *src = g.U + (v ? (g.a_r0 + gi) + (g.a_c0 + gk) * g.ldu : 0);
                cp_async<ESZ>(As + offA_kmajor<T>(k, mm), src, v);
            }
        } else {
            // A(i,k) = conj(U(a_r0+k, a_c0+i)): BM columns of U, BK contiguous rows each
#pragma unroll
            for (int it = 0; it < (BM * BK) / kGemmThreads; it++) {
                int idx = it * kGemmThreads + tid;
                int k = idx % BK, mm = idx / BK;
                int64_t gi = m0 + mm;
                int gk = k0 + k;
                bool v = gi < g.M && gk < g.K;
                const T *src = g.U + (v ? (g.a_r0 + gk) + (g.a_c0 + gi) * g.ldu : 0);
                cp_async<ESZ>(As + offRK<T>(mm, k), src, v);
            }
        }
    };
    auto load_X = [&](int s, int kt) {
        T *Xs = stageX(s);
        const int k0 = kt * BK;
        // X tile: BN columns of B, BK contiguous rows each
#pragma unroll
        for (int it = 0; it < (BN * BK) / kGemmThreads; it++) {
            int idx = it * kGemmThreads + tid;
            int k = idx % BK, nn = idx / BK;
            int64_t gj = n0 + nn;
            int gk = k0 + k;
            bool v = gj < g.N && gk < g.K;
            const T *src = g.X + (v ? (g.x_r0 + gk) + (g.col0 + gj) * g.ldx : 0);
            cp_async<ESZ>(Xs + offRK<T>(nn, k), src, v);
        }
    };
    auto load_stage = [&](int s, int kt) { load_A(s, kt); load_X(s, kt); };

    // U is read-only during a solve: with early_a the first stages' A tiles are issued before the
    // wait for the preceding grid (launched as a programmatic dependent), which X, C and d need.
    // They join the first stage's cp.async group, so the pipeline's group counting is unchanged.
    if (g.trig) pdl_trigger();
    if (g.early_a) {
#pragma unroll
        for (int s = 0; s < kGemmStages - 1; s++)
            if (s < nk) load_A(s, s);
    }
    pdl_wait();
    if (tid < BN) {
        const int64_t gj = n0 + tid;
        const int d = (g.dblk && gj < g.N) ? g.dblk[g.col0 + gj] : 0;
        s_d[tid] = d;
        s_sc[tid] = d >= -1022 ? __longlong_as_double((long long)(1023 + d) << 52) : 0.0;
    }

    // accumulators: real part (and imaginary part for complex), 2 doubles per 8x8 sub-tile
    double accR[MI][NI][2], accI[CPX ? MI : 1][CPX ? NI : 1][2];
#pragma unroll
    for (int i = 0; i < MI; i++)
#pragma unroll
        for (int jn = 0; jn < NI; jn++) {
            accR[i][jn][0] = accR[i][jn][1] = 0.0;
            if (CPX) accI[CPX ? i : 0][CPX ? jn : 0][0] = accI[CPX ? i : 0][CPX ? jn : 0][1] = 0.0;
        }

#pragma unroll
    for (int s = 0; s < kGemmStages - 1; s++) {
        if (s < nk) {
            if (g.early_a) load_X(s, s);
            else load_stage(s, s);
        }
        cp_async_commit();
    }

    // C tile prefetch: half h (columns [32h, 32h+32) of the tile) goes to the pipeline stage
    // (nk + h) % S, issued at iteration max(0, nk - 2 + h), when that stage is no longer needed by
    // the mainloop; the epilogue then reads C from shared memory.
    static_assert(kGemmStages == 3, "C prefetch assumes 3 stages");
    static_assert(BM * (BN / 2) <= gemm_stage_elems<T>(), "C half must fit in one stage");
    auto offC = [&](int row, int colh) {                  // swizzled [col][row] within a half
        if constexpr (CPX) return colh * BM + (row ^ (((colh >> 1) & 3) << 1));
        else return colh * BM + (row ^ (((colh >> 1) & 3) << 2));
    };
    auto load_c_half = [&](int h) {
        T *Cs = smem + ((nk + h) % kGemmStages) * gemm_stage_elems<T>();
#pragma unroll
        for (int it = 0; it < (BM * (BN / 2)) / kGemmThreads; it++) {
            int idx = it * kGemmThreads + tid;
            int row = idx % BM, colh = idx / BM;
            int64_t gi = m0 + row, gj = n0 + h * (BN / 2) + colh;
            bool v = gi < g.M && gj < g.N;
            const T *src = g.B + (v ? (g.c_r0 + gi) + (g.col0 + gj) * g.ldb : 0);
            cp_async<ESZ>(Cs + offC(row, colh), src, v);
        }
    };

    for (int kt = 0; kt < nk; kt++) {
        cp_async_wait<kGemmStages - 2>();
        __syncthreads();
        {
            int nxt = kt + kGemmStages - 1;
            if (nxt < nk) load_stage(nxt % kGemmStages, nxt);
            if (kt == (nk - 2 > 0 ? nk - 2 : 0)) load_c_half(0);
            if (kt == nk - 1) load_c_half(1);
            cp_async_commit();
        }
        const T *As = stageA(kt % kGemmStages);
        const T *Xs = stageX(kt % kGemmStages);
#pragma unroll
        for (int kk = 0; kk < BK / 4; kk++) {
            const int k = kk * 4 + tq;
            double ar[MI], ai[MI], nai[MI], br[NI], bi[NI];
#pragma unroll
            for (int i = 0; i < MI; i++) {
                int mm = wm * WM + i * 8 + gq;
                T v = OPC ? As[offRK<T>(mm, k)] : As[offA_kmajor<T>(k, mm)];
                if constexpr (CPX) { ar[i] = v.x; ai[i] = OPC ? -v.y : v.y; }
                else { ar[i] = v; ai[i] = 0.0; }
                nai[i] = -ai[i];
            }
#pragma unroll
            for (int jn = 0; jn < NI; jn++) {
                int nn = wn * WN + jn * 8 + gq;
                T v = Xs[offRK<T>(nn, k)];
                if constexpr (CPX) { br[jn] = v.x; bi[jn] = v.y; }
                else { br[jn] = v; bi[jn] = 0.0; }
            }
            // four passes over independent accumulators: consecutive DMMAs never depend on
            // each other (dependency distance MI*NI*2 instructions)
#pragma unroll
            for (int i = 0; i < MI; i++)
#pragma unroll
                for (int jn = 0; jn < NI; jn++) dmma(accR[i][jn][0], accR[i][jn][1], ar[i], br[jn]);
            if constexpr (CPX) {
#pragma unroll
                for (int i = 0; i < MI; i++)
#pragma unroll
                    for (int jn = 0; jn < NI; jn++) dmma(accI[i][jn][0], accI[i][jn][1], ar[i], bi[jn]);
#pragma unroll
                for (int i = 0; i < MI; i++)
#pragma unroll
                    for (int jn = 0; jn < NI; jn++) dmma(accR[i][jn][0], accR[i][jn][1], nai[i], bi[jn]);
#pragma unroll
                for (int i = 0; i < MI; i++)
#pragma unroll
                    for (int jn = 0; jn < NI; jn++) dmma(accI[i][jn][0], accI[i][jn][1], ai[i], br[jn]);
            }
        }
    }
    if (nk == 0) { load_c_half(0); load_c_half(1); cp_async_commit(); }
    cp_async_wait<0>();
    __syncthreads();

    // ---- epilogue: C = 2^d C - acc (C from shared memory); one FMA per element (2^0 = 1 is
    //      exact), bounds checks only on edge tiles; for d < -1022 (subnormal scale) 2^d in two exact
    //      normal factors, as gemm_ws_kernel ----
    const T *Cs = smem + ((nk + wn) % kGemmStages) * gemm_stage_elems<T>();   // this warp's half
    const bool full = m0 + BM <= g.M && n0 + BN <= g.N;
#pragma unroll
    for (int jn = 0; jn < NI; jn++) {
#pragma unroll
        for (int c = 0; c < 2; c++) {
            const int colh = jn * 8 + tq * 2 + c;
            const int64_t gj = n0 + wn * WN + colh;
            const double sc = s_sc[wn * WN + colh];
            const bool tiny = s_d[wn * WN + colh] < -1022;
            T *colp = g.B + g.c_r0 + (g.col0 + gj) * g.ldb;
#pragma unroll
            for (int i = 0; i < MI; i++) {
                const int row = wm * WM + i * 8 + gq;
                const int64_t gi = m0 + row;
                const T old = Cs[offC(row, colh)];
                T nv;
                if constexpr (CPX) {
                    nv.x = fma(old.x, sc, -accR[i][jn][c]);
                    nv.y = fma(old.y, sc, -accI[i][jn][c]);
                } else {
                    nv = fma(old, sc, -accR[i][jn][c]);
                }
                if (tiny) {     // 2^d as f1 * f2, both normal: the same roundings as gemm_ws_kernel
                    const int d = max(s_d[wn * WN + colh], -2044);
                    const double f1 = __longlong_as_double((long long)(1023 + d + 1022) << 52);
                    const double f2 = 0x1p-1022;
                    if constexpr (CPX) {
                        nv.x = fma(__dmul_rn(old.x, f1), f2, -accR[i][jn][c]);
                        nv.y = fma(__dmul_rn(old.y, f1), f2, -accI[i][jn][c]);
                    } else {
                        nv = fma(__dmul_rn(old, f1), f2, -accR[i][jn][c]);
                    }
                }
                if (full || (gi < g.M && gj < g.N)) colp[gi] = nv;
            }
        }
    }
}

}  // namespace mstrsm
