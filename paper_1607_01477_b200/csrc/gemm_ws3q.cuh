// gemm_ws3q.cuh -- gemm_ws3p_kernel's contraction (3M with precomputed operand sums, P:177,
// P:408) with three consumer warpgroups instead of two: 12 consumer warps = 3 per SM
// sub-partition to hide the shared-memory and barrier latencies the two-group kernel exposes at
// k-tile boundaries (its consumer loop alone reaches 87.5 % of the DMMA peak).
// Registers: 512 threads, producer warpgroup at 56, consumers at 152 (96 accumulators: a warp
// owns 16 x 32, the group tile is 32 x 64).  One producer warp per group (A / A+ bulk copies or,
// for op C, tensor-map boxes; X / X+ tensor-map boxes; C halves by bulk copy); 3-stage ring per
// group; C comes through the ring in two 32-column halves.  Selected with MSTRSM_3M_GROUPS=3.
#pragma once
#include "gemm_ws3p.cuh"

namespace mstrsm {

constexpr int k3qThreads = 512, k3qProducerRegs = 56, k3qConsumerRegs = 152;
static_assert(128 * k3qProducerRegs + 384 * k3qConsumerRegs <= 65536, "register pool");
constexpr int k3qBM = 32, k3qBN = 64, k3qBK = 8, k3qMI = 2;
constexpr int kQA = 34, kQAs = 36;                                     // padded k-rows (A, A+)
constexpr int k3qOffXs = k3qBN * k3qBK * 16;                          // 8192
constexpr int k3qOffA = k3qOffXs + k3qBN * k3qBK * 8;                 // 12288 (1024-aligned)
constexpr int k3qOffAs = k3qOffA + k3qBK * kQA * 16;                  // 16640
constexpr int k3qOffAsC = k3qOffA + k3qBM * k3qBK * 16;               // 16384 (op C, 512-aligned)
constexpr int k3qStage = (k3qOffAs + k3qBK * kQAs * 8 + 1023) & ~1023; // 19456
constexpr int k3qRing = 3;
constexpr int k3qSmemBytes = 3 * k3qRing * k3qStage + 1024;
// C half [col][pc] cplx: op N rows 2p, 2p+1 -> 544 B columns, op C (sig8 rows p, p+4) -> 528 B
template <bool OPC> constexpr int k3q_pc() { return OPC ? 33 : 34; }
static_assert(32 * 34 * 16 <= k3qStage && k3qOffAsC + k3qBM * k3qBK * 8 <= k3qStage, "");

template <bool OPC>
__global__ void __launch_bounds__(k3qThreads, 1) gemm_ws3q_kernel(GemmArgs<cplx> g, int tiles_m, int ntiles,
                                                                  const __grid_constant__ CUtensorMap tmX,
                                                                  const __grid_constant__ CUtensorMap tmXs,
                                                                  const __grid_constant__ CUtensorMap tmA,
                                                                  const __grid_constant__ CUtensorMap tmAs,
                                                                  int phase, int early_a) {
    constexpr int kPC = k3q_pc<OPC>();
    constexpr int BM = k3qBM, BN = k3qBN, BK = k3qBK, RS = k3qRing, MI = k3qMI, NI = 4, NG = 3;
    extern __shared__ __align__(1024) unsigned char smem_dyn[];
    unsigned char *smem_raw = smem_dyn + ((1024 - (smem_u32(smem_dyn) & 1023)) & 1023);
    __shared__ uint64_t full_bar[NG][RS], empty_bar[NG][RS];
    __shared__ int s_d[NG][BN];
    __shared__ int s_go;    // phase != 0: group q starts its first tile once group 0 is q/3 through its own

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nk = (g.K + BK - 1) / BK;
    if (tid == 0) {
        for (int q = 0; q < NG; q++)
            for (int s = 0; s < RS; s++) {
                mbar_init(&full_bar[q][s], 32);     // the group's producer warp, every lane
                mbar_init(&empty_bar[q][s], 4);     // the 4 warps of the consuming group
            }
        s_go = (phase && nk > 0) ? 0 : NG;    // (K = 0: no k-tile would release the others)
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    pdl_trigger();
    PT_MARK(g.pt, 0, tid == 0);
    PT_MARK(g.pt, 1, tid == 0);
    __syncthreads();
    // early_a: the U operands (A, A+) of each group's first kE k-tiles are read-only during the
    // solve, so their copies into the (still empty) ring stages are issued before the wait for the
    // preceding grid, which only the X / X+ / C loads need (the stage's full barrier then expects
    // both parts).  The launcher sets it for short launches, where the pipeline fill weighs.
    const int kE = early_a ? (nk < RS ? nk : RS) : 0;
    if (warp < NG && kE > 0) {
        const int q = warp, tile = blockIdx.x + q * gridDim.x;
        if (tile < ntiles) {
            const int64_t m0 = int64_t(tile % tiles_m) * BM;
            const int rows = int(g.M - m0 < BM ? g.M - m0 : BM);
            for (int kt = 0; kt < kE; kt++) {
                const int k0 = kt * BK;
                if (!(OPC || k0 + BK <= g.K)) break;              // (ragged k-tile: written by hand later)
                unsigned char *st = smem_raw + (q * RS + kt) * k3qStage;
                uint64_t *fb = &full_bar[q][kt];
                if (OPC) {
                    if (lane == 16) {
                        mbar_expect_tx(fb, BM * BK * 24);
                        tma_2d(st + k3qOffA, &tmA, 2 * k0, int(m0), fb);
                        tma_2d(st + k3qOffAsC, &tmAs, k0, int(m0), fb);
                    }
                } else if (lane < 2 * BK) {
                    const uint32_t bytes = lane < BK ? uint32_t(rows) * 16 : uint32_t((rows * 8 + 15) & ~15);
                    mbar_expect_tx(fb, bytes);
                    const int k = lane & (BK - 1);
                    if (lane < BK)
                        bulk_g2s(st + k3qOffA + k * kQA * 16, g.U + (g.a_r0 + m0) + (g.a_c0 + k0 + k) * g.ldu, bytes, fb);
                    else
                        bulk_g2s(st + k3qOffAs + k * kQAs * 8, g.As + (g.a_r0 + m0) + (g.a_c0 + k0 + k) * g.ldas, bytes, fb);
                }
            }
        }
    }
    pdl_wait();
    PT_MARK(g.pt, 2, tid == 0);

    if (warp < 4) {
        // ------------------------------------------------------------------ producers
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(k3qProducerRegs));
        const int q = warp;
        if (q >= NG) return;
        int gk = 0, local = 0;
#pragma unroll 1
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, local++) {
            if (local % NG != q) continue;
            const int64_t m0 = int64_t(tile % tiles_m) * BM, n0 = int64_t(tile / tiles_m) * BN;
            const int rows = int(g.M - m0 < BM ? g.M - m0 : BM);
            const int cols = int(g.N - n0 < BN ? g.N - n0 : BN);
#pragma unroll
            for (int c2 = 0; c2 < BN / 32; c2++) {      // warm L2 with this tile's C
                const int jn = c2 * 32 + lane;
                if (jn < cols) {
                    const uintptr_t a0 = reinterpret_cast<uintptr_t>(g.B + (g.c_r0 + m0) + (g.col0 + n0 + jn) * g.ldb);
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(a0), "r"(unsigned(rows * 16))
                                 : "memory");
                }
            }
#pragma unroll 1
            for (int kt = 0; kt < nk; kt++, gk++) {
                const int s = gk % RS, r = gk / RS;
                mbar_wait(&empty_bar[q][s], (r & 1) ^ 1);
                unsigned char *st = smem_raw + (q * RS + s) * k3qStage;
                uint64_t *fb = &full_bar[q][s];
                const int k0 = kt * BK;
                if (OPC || k0 + BK <= g.K) {
                    const bool early = local == q && kt < kE;            // A, A+ already issued
                    uint32_t bytes = 0;
                    if (lane == 16) bytes = BN * BK * 24 + (OPC && !early ? BM * BK * 24 : 0);
                    if (!OPC && !early && lane < 2 * BK)
                        bytes = lane < BK ? uint32_t(rows) * 16 : uint32_t((rows * 8 + 15) & ~15);
                    mbar_arrive_expect_tx(fb, bytes);
                    if (lane == 16) {
                        tma_2d(st, &tmX, 2 * k0, int(n0), fb);
                        tma_2d(st + k3qOffXs, &tmXs, k0, int(n0), fb);
                        if (OPC && !early) {
                            tma_2d(st + k3qOffA, &tmA, 2 * k0, int(m0), fb);
                            tma_2d(st + k3qOffAsC, &tmAs, k0, int(m0), fb);
                        }
                    }
                    if (!OPC && !early && lane < 2 * BK) {
                        const int k = lane & (BK - 1);
                        if (lane < BK)
                            bulk_g2s(st + k3qOffA + k * kQA * 16, g.U + (g.a_r0 + m0) + (g.a_c0 + k0 + k) * g.ldu,
                                     bytes, fb);
                        else
                            bulk_g2s(st + k3qOffAs + k * kQAs * 8, g.As + (g.a_r0 + m0) + (g.a_c0 + k0 + k) * g.ldas,
                                     bytes, fb);
                    }
                } else {                        // op N ragged last k-tile: zero-filled A / A+, X by TMA
                    cplx *As = reinterpret_cast<cplx *>(st + k3qOffA);
                    double *Ass = reinterpret_cast<double *>(st + k3qOffAs);
                    for (int idx = lane; idx < BM * BK; idx += 32) {
                        const int mm = idx % BM, k = idx / BM;
                        const bool v = mm < rows && k0 + k < g.K;
                        As[k * kQA + mm] = v ? g.U[(g.a_r0 + m0 + mm) + (g.a_c0 + k0 + k) * g.ldu] : cplx{0.0, 0.0};
                        Ass[k * kQAs + mm] = v ? g.As[(g.a_r0 + m0 + mm) + (g.a_c0 + k0 + k) * g.ldas] : 0.0;
                    }
                    __syncwarp();
                    mbar_arrive_expect_tx(fb, lane == 16 ? uint32_t(BN * BK * 24) : 0u);
                    if (lane == 16) {
                        tma_2d(st, &tmX, 2 * k0, int(n0), fb);
                        tma_2d(st + k3qOffXs, &tmXs, k0, int(n0), fb);
                    }
                }
            }
#pragma unroll 1
            for (int h = 0; h < 2; h++, gk++) {         // C half h (columns 32h .. 32h+31) and its d_j
                const int s = gk % RS, r = gk / RS;
                mbar_wait(&empty_bar[q][s], (r & 1) ^ 1);
                unsigned char *st = smem_raw + (q * RS + s) * k3qStage;
                uint64_t *fb = &full_bar[q][s];
                const int jn = 32 * h + lane;
                const bool v = jn < cols;
                if (g.dblk) s_d[q][jn] = v ? g.dblk[g.col0 + n0 + jn] : 0;
                mbar_arrive_expect_tx(fb, v ? uint32_t(rows) * 16 : 0u);
                if (v)
                    bulk_g2s(st + lane * kPC * 16, g.B + (g.c_r0 + m0) + (g.col0 + n0 + jn) * g.ldb,
                             uint32_t(rows) * 16, fb);
            }
        }
        return;
    }

    // ---------------------------------------------------------------------- consumers
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(k3qConsumerRegs));
    const int cw = warp - 4, grp = cw >> 2, wq = cw & 3;
    const int wm = wq & 1, wn = wq >> 1;          // rows 16 wm .. +15, columns 32 wn .. +31
    const int gq = lane >> 2, tq = lane & 3, sg = sig8(gq);
    int local = 0, gk = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, local++) {
        if (local % NG != grp) continue;
        const int64_t m0 = int64_t(tile % tiles_m) * BM, n0 = int64_t(tile / tiles_m) * BN;
        if (local == grp && grp > 0)   // staggered start: the groups' epilogues do not coincide
            while (*reinterpret_cast<volatile int *>(&s_go) < grp) __nanosleep(64);

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
            PT_MARK(g.pt, grp == 0 ? 3 : 5 + grp, kt == 0 && local == grp && wq == 0 && lane == 0);
            const unsigned char *st = smem_raw + (grp * RS + s) * k3qStage;
            const cplx *As = reinterpret_cast<const cplx *>(st + k3qOffA) + wm * 8 * MI + gq;
            const double *Ass = reinterpret_cast<const double *>(st + k3qOffAs) + wm * 8 * MI + gq;
            const unsigned char *Xb = st + (wn * 32 + sg) * 128, *Xsb = st + k3qOffXs + (wn * 32 + sg) * 64;
            const unsigned char *Ab = st + k3qOffA + (wm * 8 * MI + sg) * 128;
            const unsigned char *Asb = st + k3qOffAsC + (wm * 8 * MI + sg) * 64;
#pragma unroll
            for (int kk = 0; kk < BK / 4; kk++) {
                const int k = kk * 4 + tq;
                const int xo = (k ^ sg) << 4, xso = ((((k >> 1) ^ (sg >> 1)) & 3) << 4) | ((k & 1) << 3);
                double ar[MI], ai[MI], as[MI], br[NI], bi[NI], bs[NI];
#pragma unroll
                for (int i = 0; i < MI; i++) {
                    if constexpr (OPC) {
                        const cplx v = *reinterpret_cast<const cplx *>(Ab + i * 8 * 128 + xo);
                        ar[i] = v.x;
                        ai[i] = -v.y;
                        as[i] = *reinterpret_cast<const double *>(Asb + i * 8 * 64 + xso);
                    } else {
                        const cplx v = As[k * kQA + i * 8];
                        ar[i] = v.x;
                        ai[i] = v.y;
                        as[i] = Ass[k * kQAs + i * 8];
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
            if (local == 0 && cw == 0 && lane == 0) {
                if (kt == nk / 3) *reinterpret_cast<volatile int *>(&s_go) = 1;
                if (kt == (2 * nk) / 3) *reinterpret_cast<volatile int *>(&s_go) = 2;
            }
        }

        PT_MARK(g.pt, 4, local == 0 && wq == 0 && lane == 0);
        // ---- epilogue: C = 2^d C - (P1 - P2, P3 - P1 - P2); warp (wm, wn) reads half wn ----
        const int s0 = gk % RS, s1 = (gk + 1) % RS;
        mbar_wait(&full_bar[grp][s0], (gk / RS) & 1);
        mbar_wait(&full_bar[grp][s1], ((gk + 1) / RS) & 1);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty_bar[grp][wn ? s0 : s1]);   // the half this warp does not read
        const bool full = m0 + BM <= g.M && n0 + BN <= g.N;
        const cplx *Cs = reinterpret_cast<const cplx *>(smem_raw + (grp * RS + (wn ? s1 : s0)) * k3qStage);
#pragma unroll
        for (int jn = 0; jn < NI; jn++) {
#pragma unroll
            for (int c = 0; c < 2; c++) {
                const int colh = jn * 8 + tq + 4 * c;          // accumulator column 2 tq + c (sig8)
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
                    const cplx old = Cs[colh * kPC + row];
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
        if (lane == 0) mbar_arrive(&empty_bar[grp][wn ? s1 : s0]);
        gk += 2;
        PT_MARK(g.pt, 5, local == 0 && wq == 0 && lane == 0);
        PT_MARK(g.pt, 8 + grp, wq == 0 && lane == 0);
        PT_MARK(g.pt, 12 + grp, wq == 0 && lane == 0);
    }
}

}  // namespace mstrsm
