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
//   * warps 0 and 1 of warpgroup 0 are the producers, one per consumer group: each streams the A/X
//     k-tiles of its group's tiles, in order, into its own kWsRingStages-deep shared-memory ring with
//     cp.async and signals each stage's "full" mbarrier through cp.async.mbarrier.arrive; the group
//     releases a stage through its "empty" mbarrier as soon as its four warps have read it, so the
//     producer runs ahead across tile boundaries (no __syncthreads anywhere in the loop).  One
//     ring per group keeps every barrier's phases consumed in order (a shared ring would let one
//     group wait on a phase two rounds ahead, which a parity wait cannot tell apart).  This is what the one-tile-per-CTA kernel could not hide: with K = 128 a tile
//     has only 8 k-tiles, so pipeline fill and epilogue were a third of its time.
#pragma once
#include "gemm_kernel.cuh"

namespace mstrsm {

constexpr int kWsRingStages = 3;                   // per consumer group
constexpr int kWsStages = 2 * kWsRingStages;
// 12 warps = 3 warpgroups: producer WG (setmaxnreg 56) + 2 consumer WGs (setmaxnreg 224).  Each SM
// sub-partition holds one warp of every WG: 56 + 2 * 224 registers x 32 lanes fits its 16K file.
constexpr int kWsThreads = 384;
constexpr int kWsProducerRegs = 56, kWsConsumerRegs = 224;

template <typename T>
__host__ __device__ constexpr int gemm_ws_smem_bytes() {
    return kWsStages * gemm_stage_elems<T>() * int(sizeof(T));
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

template <typename T, bool OPC>
__global__ void __launch_bounds__(kWsThreads, 1) gemm_ws_kernel(GemmArgs<T> g, int tiles_m, int ntiles) {
    constexpr int BM = GemmCfg<T>::BM, BN = GemmCfg<T>::BN, BK = GemmCfg<T>::BK;
    constexpr int WM = GemmCfg<T>::WM, WN = GemmCfg<T>::WN;
    constexpr int MI = WM / 8, NI = WN / 8;
    constexpr bool CPX = S<T>::cplx_;
    constexpr int ESZ = sizeof(T);
    constexpr int SE = gemm_stage_elems<T>();
    static_assert(BM == 64 && BN == 64 && BK == 16 && WN == 32, "addressing below assumes 64x64x16 tiles");
    static_assert(BM * (BN / 2) <= SE, "a C half must fit in one stage");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T *smem = reinterpret_cast<T *>(smem_raw);
    __shared__ uint64_t full_bar[2][kWsRingStages], empty_bar[2][kWsRingStages];
    __shared__ int s_d[2][BN];                 // 2^d_j exponents of the group's current tile

    // swizzled [column][row] position of C element (row, colh) inside a C-half stage
    auto offC = [](int row, int colh) {
        if constexpr (CPX) return colh * BM + (row ^ (((colh >> 1) & 3) << 1));
        else return colh * BM + (row ^ (((colh >> 1) & 3) << 2));
    };

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nk = (g.K + BK - 1) / BK;
    if (tid == 0) {
        for (int q = 0; q < 2; q++)
            for (int s = 0; s < kWsRingStages; s++) {
                mbar_init(&full_bar[q][s], 32);     // the producer warp's cp.async arrivals
                mbar_init(&empty_bar[q][s], 4);     // the 4 warps of the consuming group
            }
    }
    __syncthreads();

    if (warp < 4) {
        // ------------------------------------------------------------------ producers
        // Per tile of its group: nk k-tile slots, then two C-half slots (C(:, 32h .. 32h+31) and the
        // matching d_j) so that the epilogue reads C from shared memory.
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kWsProducerRegs));
        if (warp >= 2) return;
        const int q = warp;
        int gk = 0, local = 0;
        auto next_slot = [&]() -> T * {
            const int s = gk % kWsRingStages, r = gk / kWsRingStages;
            mbar_wait(&empty_bar[q][s], (r & 1) ^ 1);
            return smem + (q * kWsRingStages + s) * SE;
        };
        auto commit_slot = [&]() { mbar_arrive_cpasync(&full_bar[q][gk % kWsRingStages]); gk++; };
        const int kl = lane & 15, nl = lane >> 4;           // X / A(op C): k = kl, column pair nl
#pragma unroll 1
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, local++) {
            if ((local & 1) != q) continue;
            const int64_t m0 = int64_t(tile % tiles_m) * BM, n0 = int64_t(tile / tiles_m) * BN;
            const bool vm0 = m0 + lane < g.M, vm1 = m0 + lane + 32 < g.M;
            {   // warm L2 with this tile's C (read by the C-half slots after the k-tiles)
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
                T *As = next_slot(), *Xs = As + BM * BK;
                const int k0 = kt * BK;
                if (!OPC) {                     // A(mm,k) = U(a_r0+m0+mm, a_c0+k0+k): rows contiguous
                    const T *ua = g.U + (g.a_r0 + m0 + lane) + (g.a_c0 + k0) * g.ldu;
#pragma unroll 4
                    for (int k = 0; k < BK; k++) {
                        const bool vk = k0 + k < g.K;
                        const T *col = ua + k * g.ldu;
                        cp_async<ESZ>(As + offA_kmajor<T>(k, lane), vk && vm0 ? col : g.U, vk && vm0);
                        cp_async<ESZ>(As + offA_kmajor<T>(k, lane + 32), vk && vm1 ? col + 32 : g.U, vk && vm1);
                    }
                } else {                        // A(mm,k) = conj(U(a_r0+k0+k, a_c0+m0+mm)): k contiguous
                    const bool vk = k0 + kl < g.K;
                    const T *ua = g.U + (g.a_r0 + k0 + kl) + (g.a_c0 + m0 + nl) * g.ldu;
#pragma unroll 4
                    for (int it = 0; it < BM / 2; it++) {
                        const int mm = 2 * it + nl;
                        const bool v = vk && m0 + mm < g.M;
                        cp_async<ESZ>(As + offRK<T>(mm, kl), v ? ua + (2 * it) * g.ldu : g.U, v);
                    }
                }
                {                               // X(k,nn) = B(x_r0+k0+k, col0+n0+nn): k contiguous
                    const bool vk = k0 + kl < g.K;
                    const T *xb = g.B + (g.x_r0 + k0 + kl) + (g.col0 + n0 + nl) * g.ldb;
#pragma unroll 4
                    for (int it = 0; it < BN / 2; it++) {
                        const int nn = 2 * it + nl;
                        const bool v = vk && n0 + nn < g.N;
                        cp_async<ESZ>(Xs + offRK<T>(nn, kl), v ? xb + (2 * it) * g.ldb : g.B, v);
                    }
                }
                commit_slot();
            }
#pragma unroll 1
            for (int h = 0; h < 2; h++) {       // C half h and its exponents
                T *Cs = next_slot();
                const T *cb = g.B + (g.c_r0 + m0 + lane) + (g.col0 + n0 + 32 * h) * g.ldb;
#pragma unroll 4
                for (int colh = 0; colh < 32; colh++) {
                    const bool vn = n0 + 32 * h + colh < g.N;
                    const T *col = cb + colh * g.ldb;
                    cp_async<ESZ>(Cs + offC(lane, colh), vn && vm0 ? col : g.B, vn && vm0);
                    cp_async<ESZ>(Cs + offC(lane + 32, colh), vn && vm1 ? col + 32 : g.B, vn && vm1);
                }
                if (g.dblk) {
                    const bool vn = n0 + 32 * h + lane < g.N;
                    cp_async<4>(&s_d[q][32 * h + lane], vn ? g.dblk + g.col0 + n0 + 32 * h + lane : g.dblk, vn);
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
                    const T v = OPC ? As[offRK<T>(mm, k)] : As[offA_kmajor<T>(k, mm)];
                    if constexpr (CPX) { ar[i] = v.x; ai[i] = OPC ? -v.y : v.y; }
                    else { ar[i] = v; ai[i] = 0.0; }
                    nai[i] = -ai[i];
                }
#pragma unroll
                for (int jn = 0; jn < NI; jn++) {
                    const int nn = wn * WN + jn * 8 + gq;
                    const T v = Xs[offRK<T>(nn, k)];
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

        // ---- epilogue: C = 2^d C - acc with C and d from the two C-half slots (every warp waits
        //      for both and releases both, keeping the 4-arrival count of the ring) ----
        const int s0 = gk % kWsRingStages, s1 = (gk + 1) % kWsRingStages;
        mbar_wait(&full_bar[grp][s0], (gk / kWsRingStages) & 1);
        mbar_wait(&full_bar[grp][s1], ((gk + 1) / kWsRingStages) & 1);
        const T *Cs = smem + (grp * kWsRingStages + (wn ? s1 : s0)) * SE;     // this warp's half
        const bool full = m0 + BM <= g.M && n0 + BN <= g.N;
#pragma unroll
        for (int jn = 0; jn < NI; jn++) {
#pragma unroll
            for (int c = 0; c < 2; c++) {
                const int colh = jn * 8 + tq * 2 + c;
                const int64_t gj = n0 + wn * WN + colh;
                // 2^d as f1 * f2 with both factors normal doubles (d < -1022 happens when a column
                // underflows; the scale is then applied in two exact steps, no ldexp)
                const int d = max(g.dblk ? s_d[grp][wn * WN + colh] : 0, -2044);
                const bool lo = d < -1022;
                const double f1 = lo ? __longlong_as_double((long long)(1023 + d + 1022) << 52) : 1.0;
                const double f2 = __longlong_as_double((long long)(1023 + (lo ? -1022 : d)) << 52);
                T *colp = g.B + g.c_r0 + (g.col0 + gj) * g.ldb;
#pragma unroll
                for (int i = 0; i < MI; i++) {
                    const int row = wm * WM + i * 8 + gq;
                    const int64_t gi = m0 + row;
                    const T old = Cs[offC(row, colh)];
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
        if (lane == 0) { mbar_arrive(&empty_bar[grp][s0]); mbar_arrive(&empty_bar[grp][s1]); }
        gk += 2;
    }
}

}  // namespace mstrsm
