// gemm_ws.cuh -- a.5 update GEMM, persistent warp-specialised ("ping-pong") form:
//
//     C(i,j) <- 2^{d_j} C(i,j) - sum_k A(i,k) X(k,j)        (lazy xSCAL P:378-380)
//
// Same operands, tile shapes, shared-memory swizzles and DMMA fragment code as gemm_update_kernel
// (gemm_kernel.cuh), organised for the short-K (K = n_b) shape of this method:
//   * one CTA per SM loops over output tiles (tile = blockIdx.x + i * gridDim.x);
//   * warpgroups 1 and 2 are two consumer groups that take alternate tiles (2x2 warps of 32x32 per
//     64x64 tile); one group's epilogue (C read from global, 2^d scale, store) overlaps the other
//     group's DMMA mainloop;
//   * warpgroup 0 holds the producers, two warps per consumer group: they stream the A/X k-tiles
//     of the group's tiles, in order, into the group's own kWsRingStages-deep shared-memory ring with
//     cp.async and signals each stage's "full" mbarrier through cp.async.mbarrier.arrive; the group
//     releases a stage through its "empty" mbarrier as soon as its four warps have read it, so the
//     producer runs ahead across tile boundaries (no __syncthreads anywhere in the loop).  After a
//     tile's K/8 k-tiles the ring carries the tile's C in four 16-column quarters (with the d_j),
//     released quarter by quarter by the epilogue, so the next tile's first k-tiles are already
//     in flight while the epilogue runs.  One
//     ring per group keeps every barrier's phases consumed in order (a shared ring would let one
//     group wait on a phase two rounds ahead, which a parity wait cannot tell apart).  This is what the one-tile-per-CTA kernel could not hide: with K = 128 a tile
//     has only 8 k-tiles, so pipeline fill and epilogue were a third of its time.
#pragma once
#include "gemm_kernel.cuh"

namespace mstrsm {

constexpr int kWsRingStages = 6;                   // per consumer group
constexpr int kWsStages = 2 * kWsRingStages;
constexpr int kWsBK = 8;                           // k-tile depth (a 64x64 tile has K/8 k-tiles)

// stage = A tile (BM x BK) + X tile (BN x BK); a C quarter (BM x 16 columns) has the same size
template <typename T>
__host__ __device__ constexpr int gemm_ws_stage_elems() { return (GemmCfg<T>::BM + GemmCfg<T>::BN) * kWsBK; }
// 12 warps = 3 warpgroups: producer WG (setmaxnreg 56) + 2 consumer WGs (setmaxnreg 224).  Each SM
// sub-partition holds one warp of every WG: 56 + 2 * 224 registers x 32 lanes fits its 16K file.
constexpr int kWsThreads = 384;
constexpr int kWsProducerRegs = 56, kWsConsumerRegs = 224;
// The CTA starts with 168 registers per thread (65536 / 384, rounded down); the consumers' increase
// is served only from what the producer warpgroup releases: (168 - 56) * 128 >= (224 - 168) * 256.
static_assert((168 - kWsProducerRegs) * 128 >= (kWsConsumerRegs - 168) * 256, "setmaxnreg pool");

template <typename T>
__host__ __device__ constexpr int gemm_ws_smem_bytes() {
    return kWsStages * gemm_ws_stage_elems<T>() * int(sizeof(T));
}

__device__ __forceinline__ void mbar_init(uint64_t *b, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
// arrive once all cp.async issued so far by this thread have landed
__device__ __forceinline__ void mbar_arrive_cpasync(uint64_t *b) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, int parity) {
    uint32_t done = 0;
    do {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                     " selp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(done) : "r"(smem_u32(b)), "r"(parity) : "memory");
    } while (!done);
}

// swizzled positions (element units) inside a stage
//  A, op N: (k, m) of a BK x BM tile, m contiguous (16-B slots rotated by k)
template <typename T> __device__ __forceinline__ int ws_offA_km(int k, int mm) {
    if constexpr (S<T>::cplx_) return k * 64 + (mm ^ ((k & 3) << 1));
    else return k * 64 + (mm ^ ((k & 3) << 2));
}
//  A, op C and X: (r, k) of a 64 x BK tile, k contiguous (BK = 8)
template <typename T> __device__ __forceinline__ int ws_offRK(int r, int k) {
    if constexpr (S<T>::cplx_) return r * kWsBK + (k ^ ((r & 1) << 2));
    else return r * kWsBK + (k ^ ((r & 3) << 1));
}
//  C quarter: (row, column) of a 64 x 16 block, rows contiguous
template <typename T> __device__ __forceinline__ int ws_offC(int row, int colq) {
    if constexpr (S<T>::cplx_) return colq * 64 + (row ^ (((colq >> 1) & 3) << 1));
    else return colq * 64 + (row ^ (((colq >> 1) & 3) << 2));
}

template <typename T, bool OPC>
__global__ void __launch_bounds__(kWsThreads, 1) gemm_ws_kernel(GemmArgs<T> g, int tiles_m, int ntiles, int early_a) {
    constexpr int BM = GemmCfg<T>::BM, BN = GemmCfg<T>::BN, BK = kWsBK;
    constexpr int WM = GemmCfg<T>::WM, WN = GemmCfg<T>::WN;
    constexpr int MI = WM / 8, NI = WN / 8;
    constexpr bool CPX = S<T>::cplx_;
    constexpr int ESZ = sizeof(T);
    constexpr int SE = gemm_ws_stage_elems<T>();
    static_assert(BM == 64 && BN == 64 && WM == 32 && WN == 32, "addressing below assumes 64x64 tiles");
    static_assert(BM * 16 <= SE, "a C quarter must fit in one stage");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T *smem = reinterpret_cast<T *>(smem_raw);
    __shared__ uint64_t full_bar[2][kWsRingStages], empty_bar[2][kWsRingStages];
    __shared__ int s_d[2][BN];                 // d_j of the group's current tile

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nk = (g.K + BK - 1) / BK;
    if (tid == 0) {
        for (int q = 0; q < 2; q++)
            for (int s = 0; s < kWsRingStages; s++) {
                mbar_init(&full_bar[q][s], 64);     // the two producer warps' cp.async arrivals
                mbar_init(&empty_bar[q][s], 4);     // the 4 warps of the consuming group
            }
    }
    __syncthreads();
    // A(mm, k) tile of k-tile k0 into As (the A warp of a ring; fully predicated unless interior)
    auto load_A = [&](T *As, int64_t m0, int k0, bool interior) {
        const int kl = lane & 7, nl = lane >> 3;
        const bool vm0 = m0 + lane < g.M, vm1 = m0 + lane + 32 < g.M;
        if (!OPC) {                 // A(mm,k) = U(a_r0+m0+mm, a_c0+k0+k): rows contiguous
            const T *ua = g.U + (g.a_r0 + m0 + lane) + (g.a_c0 + k0) * g.ldu;
            if (interior) {
#pragma unroll
                for (int k = 0; k < BK; k++) {
                    cp_async<ESZ>(As + ws_offA_km<T>(k, lane), ua + k * g.ldu, true);
                    cp_async<ESZ>(As + ws_offA_km<T>(k, lane + 32), ua + k * g.ldu + 32, true);
                }
            } else {
#pragma unroll
                for (int k = 0; k < BK; k++) {
                    const bool vk = k0 + k < g.K;
                    const T *col = ua + k * g.ldu;
                    cp_async<ESZ>(As + ws_offA_km<T>(k, lane), vk && vm0 ? col : g.U, vk && vm0);
                    cp_async<ESZ>(As + ws_offA_km<T>(k, lane + 32), vk && vm1 ? col + 32 : g.U, vk && vm1);
                }
            }
        } else {                    // A(mm,k) = conj(U(a_r0+k0+k, a_c0+m0+mm)): k contiguous
            const bool vk = k0 + kl < g.K;
            const T *ua = g.U + (g.a_r0 + k0 + kl) + (g.a_c0 + m0 + nl) * g.ldu;
#pragma unroll 4
            for (int it = 0; it < BM / 4; it++) {
                const int mm = 4 * it + nl;
                const bool v = vk && m0 + mm < g.M;
                cp_async<ESZ>(As + ws_offRK<T>(mm, kl), v ? ua + (4 * it) * g.ldu : g.U, v);
            }
        }
    };
    // early_a: U is read-only during the solve, so the A warps copy the A tiles of their group's
    // first kE k-tiles into the (still empty) ring stages and arrive on those stages' full
    // barriers before the wait for the preceding grid, which only the X and C loads need (as in
    // gemm_ws3q_kernel; the launcher sets it for short launches).
    const int kE = early_a ? (nk < kWsRingStages ? nk : kWsRingStages) : 0;
    if (warp < 4 && (warp & 1) == 0 && kE > 0) {
        const int q = warp >> 1, tile = blockIdx.x + q * gridDim.x;
        if (tile < ntiles) {
            const int64_t m0 = int64_t(tile % tiles_m) * BM;
            for (int kt = 0; kt < kE; kt++) {
                load_A(smem + (q * kWsRingStages + kt) * SE, m0, kt * BK,
                       m0 + BM <= g.M && kt * BK + BK <= g.K);
                mbar_arrive_cpasync(&full_bar[q][kt]);
            }
        }
    }
    pdl_wait();

    if (warp < 4) {
        // ------------------------------------------------------------------ producers
        // Two warps per ring: warp 2q+0 loads the A tiles and C columns 0-7 of each quarter,
        // warp 2q+1 the X tiles and C columns 8-15 (and the d_j).  Interior k-tiles take an
        // unpredicated path.
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kWsProducerRegs));
        const int q = warp >> 1, half = warp & 1;
        int gk = 0, local = 0;
        auto next_slot = [&]() -> T * {
            const int s = gk % kWsRingStages, r = gk / kWsRingStages;
            mbar_wait(&empty_bar[q][s], (r & 1) ^ 1);
            return smem + (q * kWsRingStages + s) * SE;
        };
        auto commit_slot = [&]() { mbar_arrive_cpasync(&full_bar[q][gk % kWsRingStages]); gk++; };
        const int kl = lane & 7, nl = lane >> 3;            // k-contiguous tiles: k = kl, column nl + 4 it
#pragma unroll 1
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, local++) {
            if ((local & 1) != q) continue;
            const int64_t m0 = int64_t(tile % tiles_m) * BM, n0 = int64_t(tile / tiles_m) * BN;
            const bool vm0 = m0 + lane < g.M, vm1 = m0 + lane + 32 < g.M;
            const bool mn_in = m0 + BM <= g.M && n0 + BN <= g.N;
            if (half == 0) {   // warm L2 with this tile's C (read through the ring after the k-tiles)
                const int64_t rows = g.M - m0 < BM ? g.M - m0 : int64_t(BM);
#pragma unroll
                for (int c2 = 0; c2 < BN / 32; c2++) {
                    const int64_t gj = n0 + c2 * 32 + lane;
                    if (gj < g.N && rows > 0) {
                        // 16-byte aligned start and length (bulk-copy rules)
                        const uintptr_t a0 = reinterpret_cast<uintptr_t>(g.B + (g.c_r0 + m0) + (g.col0 + gj) * g.ldb);
                        const uintptr_t al = a0 & ~uintptr_t(15);
                        const unsigned len = unsigned((a0 - al + rows * ESZ + 15) & ~uintptr_t(15));
                        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(al), "r"(len) : "memory");
                    }
                }
            }
#pragma unroll 1
            for (int kt = 0; kt < nk; kt++) {
                if (half == 0 && local == q && kt < kE) { gk++; continue; }   // A issued and arrived early
                T *As = next_slot(), *Xs = As + BM * BK;
                const int k0 = kt * BK;
                const bool interior = mn_in && k0 + BK <= g.K;
                if (half == 0) {
                    load_A(As, m0, k0, interior);
                } else {                        // X(k,nn) = X(x_r0+k0+k, col0+n0+nn): k contiguous
                    const T *xb = g.X + (g.x_r0 + k0 + kl) + (g.col0 + n0 + nl) * g.ldx;
                    if (interior) {
#pragma unroll 4
                        for (int it = 0; it < BN / 4; it++)
                            cp_async<ESZ>(Xs + ws_offRK<T>(4 * it + nl, kl), xb + (4 * it) * g.ldx, true);
                    } else {
                        const bool vk = k0 + kl < g.K;
#pragma unroll 4
                        for (int it = 0; it < BN / 4; it++) {
                            const int nn = 4 * it + nl;
                            const bool v = vk && n0 + nn < g.N;
                            cp_async<ESZ>(Xs + ws_offRK<T>(nn, kl), v ? xb + (4 * it) * g.ldx : g.X, v);
                        }
                    }
                }
                commit_slot();
            }
#pragma unroll 1
            for (int cq = 0; cq < 4; cq++) {    // C quarter cq (columns 16cq .. 16cq+15) and its d_j
                T *Cs = next_slot();
                const T *cb = g.B + (g.c_r0 + m0 + lane) + (g.col0 + n0 + 16 * cq + 8 * half) * g.ldb;
#pragma unroll 4
                for (int c8 = 0; c8 < 8; c8++) {
                    const int colq = 8 * half + c8;
                    const bool vn = n0 + 16 * cq + colq < g.N;
                    const T *col = cb + c8 * g.ldb;
                    cp_async<ESZ>(Cs + ws_offC<T>(lane, colq), vn && vm0 ? col : g.B, vn && vm0);
                    cp_async<ESZ>(Cs + ws_offC<T>(lane + 32, colq), vn && vm1 ? col + 32 : g.B, vn && vm1);
                }
                if (half == 1 && g.dblk && lane < 16) {
                    const bool vn = n0 + 16 * cq + lane < g.N;
                    cp_async<4>(&s_d[q][16 * cq + lane], vn ? g.dblk + g.col0 + n0 + 16 * cq + lane : g.dblk, vn);
                }
                commit_slot();
            }
        }
        return;
    }

    // ---------------------------------------------------------------------- consumers
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kWsConsumerRegs));
    const int cw = warp - 4, grp = cw >> 2, wq = cw & 3;
    const int wm = wq & 1, wn = wq >> 1;
    const int gq = lane >> 2, tq = lane & 3;
    int local = 0, gk = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, local++) {
        if ((local & 1) != grp) continue;
        const int64_t m0 = int64_t(tile % tiles_m) * BM, n0 = int64_t(tile / tiles_m) * BN;

        double accR[MI][NI][2], accI[CPX ? MI : 1][CPX ? NI : 1][2];
#pragma unroll
        for (int i = 0; i < MI; i++)
#pragma unroll
            for (int jn = 0; jn < NI; jn++) {
                accR[i][jn][0] = accR[i][jn][1] = 0.0;
                if (CPX) accI[CPX ? i : 0][CPX ? jn : 0][0] = accI[CPX ? i : 0][CPX ? jn : 0][1] = 0.0;
            }

        for (int kt = 0; kt < nk; kt++, gk++) {
            const int s = gk % kWsRingStages, r = gk / kWsRingStages;
            mbar_wait(&full_bar[grp][s], r & 1);
            const T *As = smem + (grp * kWsRingStages + s) * SE, *Xs = As + BM * BK;
#pragma unroll
            for (int kk = 0; kk < BK / 4; kk++) {
                const int k = kk * 4 + tq;
                double ar[MI], ai[MI], nai[MI], br[NI], bi[NI];
#pragma unroll
                for (int i = 0; i < MI; i++) {
                    const int mm = wm * WM + i * 8 + gq;
                    const T v = OPC ? As[ws_offRK<T>(mm, k)] : As[ws_offA_km<T>(k, mm)];
                    if constexpr (CPX) { ar[i] = v.x; ai[i] = OPC ? -v.y : v.y; }
                    else { ar[i] = v; ai[i] = 0.0; }
                    nai[i] = -ai[i];
                }
#pragma unroll
                for (int jn = 0; jn < NI; jn++) {
                    const int nn = wn * WN + jn * 8 + gq;
                    const T v = Xs[ws_offRK<T>(nn, k)];
                    if constexpr (CPX) { br[jn] = v.x; bi[jn] = v.y; }
                    else { br[jn] = v; bi[jn] = 0.0; }
                }
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
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty_bar[grp][s]);
        }

        // ---- epilogue: C = 2^d C - acc, C and d from the four C-quarter slots.  Every warp waits
        //      for all four (the ring's 4-arrival count), releases the two it does not read at once
        //      and each of its own two as soon as it is done with it. ----
        auto sq = [&](int cq) { return (gk + cq) % kWsRingStages; };
#pragma unroll
        for (int cq = 0; cq < 4; cq++) mbar_wait(&full_bar[grp][sq(cq)], ((gk + cq) / kWsRingStages) & 1);
        __syncwarp();
        if (lane == 0) { mbar_arrive(&empty_bar[grp][sq(2 - 2 * wn)]); mbar_arrive(&empty_bar[grp][sq(3 - 2 * wn)]); }
        const bool full = m0 + BM <= g.M && n0 + BN <= g.N;
#pragma unroll
        for (int h = 0; h < 2; h++) {           // own quarters 2 wn + h: columns jn = 2h, 2h+1
            const T *Cs = smem + (grp * kWsRingStages + sq(2 * wn + h)) * SE;
#pragma unroll
            for (int jj = 0; jj < 2; jj++) {
                const int jn = 2 * h + jj;
#pragma unroll
                for (int c = 0; c < 2; c++) {
                    const int colq = jj * 8 + tq * 2 + c;            // column inside the quarter
                    const int colh = jn * 8 + tq * 2 + c;            // column inside the warp tile
                    const int64_t gj = n0 + wn * WN + colh;
                    // 2^d as f1 * f2 with both factors normal doubles (d < -1022 happens when a
                    // column underflows; the scale is then applied in two exact steps, no ldexp)
                    const int d = max(g.dblk ? s_d[grp][wn * WN + colh] : 0, -2044);
                    const bool lo = d < -1022;
                    const double f1 = lo ? __longlong_as_double((long long)(1023 + d + 1022) << 52) : 1.0;
                    const double f2 = __longlong_as_double((long long)(1023 + (lo ? -1022 : d)) << 52);
                    T *colp = g.B + g.c_r0 + (g.col0 + gj) * g.ldb;
#pragma unroll
                    for (int i = 0; i < MI; i++) {
                        const int row = wm * WM + i * 8 + gq;
                        const int64_t gi = m0 + row;
                        const T old = Cs[ws_offC<T>(row, colq)];
                        T nv;
                        if constexpr (CPX) {
                            nv.x = fma(__dmul_rn(old.x, f1), f2, -accR[i][jn][c]);
                            nv.y = fma(__dmul_rn(old.y, f1), f2, -accI[i][jn][c]);
                        } else {
                            nv = fma(__dmul_rn(old, f1), f2, -accR[i][jn][c]);
                        }
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
