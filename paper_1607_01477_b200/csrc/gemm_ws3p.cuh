// gemm_ws3p.cuh -- the complex 3M update GEMM (gemm_ws3m.cuh) with the operand sums
// precomputed and every operand moved by the bulk-copy engine:
//
//     C(i,j) <- 2^{d_j} C(i,j) - (P1 - P2, P3 - P1 - P2),   P1 = Ar Xr, P2 = Ai Xi, P3 = A+ X+
//
// where A+ = Ar + Ai (the Usum plane, presum_kernel, once per solve) and X+ = Xr + Xi (written by
// the diagonal kernel next to X).  The sums are exactly the ones the register-sum kernel forms
// (the same __dadd_rn of the same operands), so the two kernels produce identical products.
// Without the in-register sums the consumer loop is LDS + DMMA only; the producers then move 1.5x
// the bytes, which per-element cp.async cannot issue fast enough -- so every contiguous segment
// (a 48-row column piece of A / A+ / C) is one
// cp.async.bulk (UBLKCP) completing on the stage's mbarrier with a byte count, and X / X+ (64
// columns of 8 rows each) are one tensor-map box each (UTMALDG, swizzled, zero fill past K and N).
// Bulk copies land unswizzled, so A / A+ / C use padded strides; X / X+ use the TMA swizzles with
// a column permutation of the B fragment (sig8) -- every fragment read is conflict-free
// (DESIGN §7.2).  Op C (A = conj(U)^T, k contiguous in U): A and A+ are tensor-map boxes too, with
// the same row permutation on the A fragment (sig8; the epilogue maps rows back).
#pragma once
#include <cuda.h>   // CUtensorMap

#include "gemm_ws3m.cuh"

namespace mstrsm {

// stage layout (bytes; stage base 1024-aligned):
//   X  [nn][8] cplx   dense 128-B rows, TMA SWIZZLE_128B (16-B chunk k at k ^ (nn & 7))
//   X+ [nn][8] f64    dense 64-B rows,  TMA SWIZZLE_64B  (16-B chunk k/2 at k/2 ^ ((nn >> 1) & 3))
//   A  [k][kPA] cplx  bulk copies, padded rows;  A+ [k][kPAs] f64 likewise
// A C quarter [colq][kPC] cplx (bulk copies) reuses a whole stage.
constexpr int kPA = 50, kPAs = 52;
// C quarter column stride: op N rows are lane groups 2p, 2p+1 (32p, 32p+16 B), op C rows are the
// sig8-permuted p, p+4 (16p, 16p+64 B); 800 B resp. 784 B columns keep the epilogue reads
// conflict-free.
template <bool OPC> constexpr int k3p_pc() { return OPC ? 49 : 50; }
constexpr int k3pOffXs = k3mBN * k3mBK * 16;                     // 8192
constexpr int k3pOffA = k3pOffXs + k3mBN * k3mBK * 8;            // 12288
constexpr int k3pOffAs = k3pOffA + k3mBK * kPA * 16;             // 18688
// op C: A (48 rows x 8 k, k contiguous) and A+ come as tensor-map boxes: A [mm][8] cplx dense
// 128-B rows (128-B swizzle), A+ [mm][8] f64 64-B rows (64-B swizzle), rows sig8-permuted
constexpr int k3pOffAsC = k3pOffA + k3mBM * k3mBK * 16;           // 18432
constexpr int k3pStage = (k3pOffAs + k3mBK * kPAs * 8 + 1023) & ~1023;
constexpr int k3pRing = (227 * 1024 - 4096 - 1024) / (2 * k3pStage);
constexpr int k3pSmemBytes = 2 * k3pRing * k3pStage + 1024;      // + 1024: base alignment
static_assert(16 * 50 * 16 <= k3pStage, "a C quarter must fit in one stage");
static_assert(k3pOffA % 1024 == 0 && k3pOffAsC % 512 == 0 && k3pOffAsC + k3mBM * k3mBK * 8 <= k3pStage, "");
static_assert(k3pOffA % 16 == 0 && k3pOffAs % 16 == 0 && k3pOffXs % 512 == 0, "");

// raise the barrier's expected transaction bytes without arriving
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes)
                 : "memory");
}
// one contiguous global -> shared copy (16-byte aligned, multiple of 16 bytes), completing on bar
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// one 2-D tensor-map box (out-of-range elements zero-filled), completing on bar
__device__ __forceinline__ void tma_2d(void *dst, const CUtensorMap *tm, int c0, int c1, uint64_t *bar) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                 " [%0], [%1, {%2, %3}], [%4];\n"
                 ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
                 : "memory");
}
// B-fragment column permutation: lane group gq reads column sig(gq) of each 8-column group, so
// the two row groups of a quarter-warp (gq = 2p, 2p+1 -> columns p, p+4) hit opposite halves of
// the swizzled 128-B / 64-B rows.  Accumulator column 2 tq + c is then column tq + 4 c.
__device__ __forceinline__ int sig8(int gq) { return (gq >> 1) | ((gq & 1) << 2); }

template <bool OPC>
__global__ void __launch_bounds__(kWsThreads, 1) gemm_ws3p_kernel(GemmArgs<cplx> g, int tiles_m, int ntiles,
                                                                  const __grid_constant__ CUtensorMap tmX,
                                                                  const __grid_constant__ CUtensorMap tmXs,
                                                                  const __grid_constant__ CUtensorMap tmA,
                                                                  const __grid_constant__ CUtensorMap tmAs,
                                                                  int phase) {
    constexpr int kPC = k3p_pc<OPC>();
    constexpr int BM = k3mBM, BN = k3mBN, BK = k3mBK, RS = k3pRing;
    constexpr int MI = k3mMI, NI = 4;
    extern __shared__ __align__(1024) unsigned char smem_dyn[];
    unsigned char *smem_raw = smem_dyn + ((1024 - (smem_u32(smem_dyn) & 1023)) & 1023);
    __shared__ uint64_t full_bar[2][RS], empty_bar[2][RS];
    __shared__ int s_d[2][BN];
    __shared__ int s_go;    // phase != 0: group 1 starts once group 0 is phase/4 through its first tile

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nk = (g.K + BK - 1) / BK;
    if (tid == 0) {
        for (int q = 0; q < 2; q++)
            for (int s = 0; s < RS; s++) {
                mbar_init(&full_bar[q][s], 64);     // every producer lane arrives (with its bytes)
                mbar_init(&empty_bar[q][s], 4);     // the 4 warps of the consuming group
            }
        s_go = (phase && nk > 0) ? 0 : 1;     // (K = 0: no k-tile would release group 1)
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    pdl_trigger();
    pdl_wait();

    if (warp < 4) {
        // ------------------------------------------------------------------ producers
        // warp 2q: A and A+ (lanes 0-7 / 8-15, one bulk copy per k) and the C quarters;
        // warp 2q+1: X and X+ (lane 0, one tensor-map box each) and d_j
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kWsProducerRegs));
        const int q = warp >> 1, half = warp & 1;
        int gk = 0, local = 0;
#pragma unroll 1
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, local++) {
            if ((local & 1) != q) continue;
            const int64_t m0 = int64_t(tile % tiles_m) * BM, n0 = int64_t(tile / tiles_m) * BN;
            const int rows = int(g.M - m0 < BM ? g.M - m0 : BM);
            const int cols = int(g.N - n0 < BN ? g.N - n0 : BN);
            if (half == 0) {   // warm L2 with this tile's C (read through the ring after the k-tiles)
#pragma unroll
                for (int c2 = 0; c2 < BN / 32; c2++) {
                    const int jn = c2 * 32 + lane;
                    if (jn < cols) {
                        const uintptr_t a0 = reinterpret_cast<uintptr_t>(g.B + (g.c_r0 + m0) + (g.col0 + n0 + jn) * g.ldb);
                        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(a0), "r"(unsigned(rows * 16))
                                     : "memory");
                    }
                }
            }
#pragma unroll 1
            for (int kt = 0; kt < nk; kt++, gk++) {
                const int s = gk % RS, r = gk / RS;
                mbar_wait(&empty_bar[q][s], (r & 1) ^ 1);
                unsigned char *st = smem_raw + (q * RS + s) * k3pStage;
                uint64_t *fb = &full_bar[q][s];
                const int k0 = kt * BK;
                if (half == 1) {                // X, X+: one tensor-map box each (zero fill past K, N)
                    if (lane == 0) {
                        mbar_arrive_expect_tx(fb, BN * BK * 24);
                        tma_2d(st, &tmX, 2 * k0, int(n0), fb);
                        tma_2d(st + k3pOffXs, &tmXs, k0, int(n0), fb);
                    } else {
                        mbar_arrive(fb);
                    }
                } else if (OPC) {               // A = conj(U)^T, A+: one tensor-map box each
                    if (lane == 0) {
                        mbar_arrive_expect_tx(fb, BM * BK * 24);
                        tma_2d(st + k3pOffA, &tmA, 2 * k0, int(m0), fb);
                        tma_2d(st + k3pOffAsC, &tmAs, k0, int(m0), fb);
                    } else {
                        mbar_arrive(fb);
                    }
                } else if (k0 + BK <= g.K) {    // A, A+: one bulk copy per k (rows contiguous)
                    if (lane < 2 * BK) {
                        const int k = lane & (BK - 1);
                        const uint32_t bytes = lane < BK ? uint32_t(rows) * 16 : uint32_t((rows * 8 + 15) & ~15);
                        mbar_arrive_expect_tx(fb, bytes);
                        if (lane < BK)
                            bulk_g2s(st + k3pOffA + k * kPA * 16, g.U + (g.a_r0 + m0) + (g.a_c0 + k0 + k) * g.ldu, bytes, fb);
                        else
                            bulk_g2s(st + k3pOffAs + k * kPAs * 8, g.As + (g.a_r0 + m0) + (g.a_c0 + k0 + k) * g.ldas,
                                     bytes, fb);
                    } else {
                        mbar_arrive(fb);
                    }
                } else {                        // ragged last k-tile (K % 8 != 0): zero-filled element copies
                    cplx *As = reinterpret_cast<cplx *>(st + k3pOffA);
                    double *Ass = reinterpret_cast<double *>(st + k3pOffAs);
                    for (int idx = lane; idx < BM * BK; idx += 32) {
                        const int mm = idx % BM, k = idx / BM;
                        const bool v = mm < rows && k0 + k < g.K;
                        As[k * kPA + mm] = v ? g.U[(g.a_r0 + m0 + mm) + (g.a_c0 + k0 + k) * g.ldu] : cplx{0.0, 0.0};
                        Ass[k * kPAs + mm] = v ? g.As[(g.a_r0 + m0 + mm) + (g.a_c0 + k0 + k) * g.ldas] : 0.0;
                    }
                    mbar_arrive(fb);
                }
            }
#pragma unroll 1
            for (int cq = 0; cq < 4; cq++, gk++) {    // C quarter cq (columns 16cq .. 16cq+15) and its d_j
                const int s = gk % RS, r = gk / RS;
                mbar_wait(&empty_bar[q][s], (r & 1) ^ 1);
                unsigned char *st = smem_raw + (q * RS + s) * k3pStage;
                uint64_t *fb = &full_bar[q][s];
                if (half == 0) {
                    const int jn = 16 * cq + (lane & 15);
                    const bool v = lane < 16 && jn < cols;
                    mbar_arrive_expect_tx(fb, v ? uint32_t(rows) * 16 : 0u);
                    if (v)
                        bulk_g2s(st + (lane & 15) * kPC * 16, g.B + (g.c_r0 + m0) + (g.col0 + n0 + jn) * g.ldb,
                                 uint32_t(rows) * 16, fb);
                } else {
                    if (g.dblk && lane < 16) {
                        const int jn = 16 * cq + lane;
                        s_d[q][jn] = jn < cols ? g.dblk[g.col0 + n0 + jn] : 0;
                    }
                    mbar_arrive(fb);
                }
            }
        }
        return;
    }

    // ---------------------------------------------------------------------- consumers
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kWsConsumerRegs));
    const int cw = warp - 4, grp = cw >> 2, wq = cw & 3;
    const int wm = wq & 1, wn = wq >> 1;          // rows 8 MI wm .. +8 MI-1, columns 32 wn .. +31
    const int gq = lane >> 2, tq = lane & 3, sg = sig8(gq);
    int local = 0, gk = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, local++) {
        if ((local & 1) != grp) continue;
        const int64_t m0 = int64_t(tile % tiles_m) * BM, n0 = int64_t(tile / tiles_m) * BN;
        if (local == 1)         // group 1's first tile: offset the two groups' epilogues (by half a tile: phase 2)
            while (*reinterpret_cast<volatile int *>(&s_go) == 0) __nanosleep(64);

        double p1[MI][NI][2], p2[MI][NI][2], p3[MI][NI][2];
#pragma unroll
        for (int i = 0; i < MI; i++)
#pragma unroll
            for (int jn = 0; jn < NI; jn++)
#pragma unroll
                for (int c = 0; c < 2; c++) p1[i][jn][c] = p2[i][jn][c] = p3[i][jn][c] = 0.0;

        for (int kt = 0; kt < nk; kt++, gk++) {
            const int s = gk % RS, r = gk / RS;
            mbar_wait(&full_bar[grp][s], r & 1);
            const unsigned char *st = smem_raw + (grp * RS + s) * k3pStage;
            const cplx *As = reinterpret_cast<const cplx *>(st + k3pOffA) + wm * 8 * MI + gq;
            const double *Ass = reinterpret_cast<const double *>(st + k3pOffAs) + wm * 8 * MI + gq;
            const unsigned char *Xb = st + (wn * 32 + sg) * 128, *Xsb = st + k3pOffXs + (wn * 32 + sg) * 64;
            const unsigned char *Ab = st + k3pOffA + (wm * 8 * MI + sg) * 128;
            const unsigned char *Asb = st + k3pOffAsC + (wm * 8 * MI + sg) * 64;
#pragma unroll
            for (int kk = 0; kk < BK / 4; kk++) {
                const int k = kk * 4 + tq;
                const int xo = (k ^ sg) << 4, xso = ((((k >> 1) ^ (sg >> 1)) & 3) << 4) | ((k & 1) << 3);
                double ar[MI], ai[MI], as[MI], br[NI], bi[NI], bs[NI];
#pragma unroll
                for (int i = 0; i < MI; i++) {
                    if constexpr (OPC) {        // rows wm 24 + 8 i + sig8(gq), conj at use
                        const cplx v = *reinterpret_cast<const cplx *>(Ab + i * 8 * 128 + xo);
                        ar[i] = v.x;
                        ai[i] = -v.y;
                        as[i] = *reinterpret_cast<const double *>(Asb + i * 8 * 64 + xso);
                    } else {
                        const cplx v = As[k * kPA + i * 8];
                        ar[i] = v.x;
                        ai[i] = v.y;
                        as[i] = Ass[k * kPAs + i * 8];
                    }
                }
#pragma unroll
                for (int jn = 0; jn < NI; jn++) {
                    const cplx v = *reinterpret_cast<const cplx *>(Xb + jn * 8 * 128 + xo);
                    br[jn] = v.x;
                    bi[jn] = v.y;
                    bs[jn] = *reinterpret_cast<const double *>(Xsb + jn * 8 * 64 + xso);
                }
#pragma unroll
                for (int i = 0; i < MI; i++)
#pragma unroll
                    for (int jn = 0; jn < NI; jn++) dmma(p1[i][jn][0], p1[i][jn][1], ar[i], br[jn]);
#pragma unroll
                for (int i = 0; i < MI; i++)
#pragma unroll
                    for (int jn = 0; jn < NI; jn++) dmma(p2[i][jn][0], p2[i][jn][1], ai[i], bi[jn]);
#pragma unroll
                for (int i = 0; i < MI; i++)
#pragma unroll
                    for (int jn = 0; jn < NI; jn++) dmma(p3[i][jn][0], p3[i][jn][1], as[i], bs[jn]);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty_bar[grp][s]);
            if (local == 0 && kt == (nk * phase) / 4 && cw == 0 && lane == 0) *reinterpret_cast<volatile int *>(&s_go) = 1;
        }

        // ---- epilogue (as gemm_ws3m_kernel): C = 2^d C - (P1 - P2, P3 - P1 - P2) ----
        auto sq = [&](int cq) { return (gk + cq) % RS; };
#pragma unroll
        for (int cq = 0; cq < 4; cq++) mbar_wait(&full_bar[grp][sq(cq)], ((gk + cq) / RS) & 1);
        __syncwarp();
        if (lane == 0) { mbar_arrive(&empty_bar[grp][sq(2 - 2 * wn)]); mbar_arrive(&empty_bar[grp][sq(3 - 2 * wn)]); }
        const bool full = m0 + BM <= g.M && n0 + BN <= g.N;
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const cplx *Cs = reinterpret_cast<const cplx *>(smem_raw + (grp * RS + sq(2 * wn + h)) * k3pStage);
#pragma unroll
            for (int jj = 0; jj < 2; jj++) {
                const int jn = 2 * h + jj;
#pragma unroll
                for (int c = 0; c < 2; c++) {
                    const int colq = jj * 8 + tq + 4 * c;      // accumulator column 2 tq + c (sig8)
                    const int colh = jn * 8 + tq + 4 * c;
                    const int64_t gj = n0 + wn * 32 + colh;
                    const int d = max(g.dblk ? s_d[grp][wn * 32 + colh] : 0, -2044);
                    const bool lo = d < -1022;
                    const double f1 = lo ? __longlong_as_double((long long)(1023 + d + 1022) << 52) : 1.0;
                    const double f2 = __longlong_as_double((long long)(1023 + (lo ? -1022 : d)) << 52);
                    cplx *colp = g.B + g.c_r0 + (g.col0 + gj) * g.ldb;
#pragma unroll
                    for (int i = 0; i < MI; i++) {
                        const int row = wm * 8 * MI + i * 8 + (OPC ? sg : gq);
                        const int64_t gi = m0 + row;
                        const cplx old = Cs[colq * kPC + row];
                        const double re = __dsub_rn(p1[i][jn][c], p2[i][jn][c]);
                        const double im = __dsub_rn(__dsub_rn(p3[i][jn][c], p1[i][jn][c]), p2[i][jn][c]);
                        cplx nv;
                        nv.x = fma(__dmul_rn(old.x, f1), f2, -re);
                        nv.y = fma(__dmul_rn(old.y, f1), f2, -im);
                        if (full || (gi < g.M && gj < g.N)) colp[gi] = nv;
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty_bar[grp][sq(2 * wn + h)]);
        }
        gk += 4;
    }
}

}  // namespace mstrsm
