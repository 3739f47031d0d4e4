// gemm_ws3m.cuh -- a.5 update GEMM for complex operands with three real products ("3M"):
//
//     C(i,j) <- 2^{d_j} C(i,j) - sum_k A(i,k) X(k,j)        (lazy xSCAL P:378-380)
//
//     P1 = Ar Xr,  P2 = Ai Xi,  P3 = (Ar + Ai)(Xr + Xi)   ->   Re = P1 - P2,  Im = P3 - P1 - P2
//
// The same contraction as the four-product form (Re = Ar Xr - Ai Xi, Im = Ar Xi + Ai Xr) with a
// quarter fewer DMMAs; it is normwise stable with an error bound of the same order (the sums
// Ar + Ai, Xr + Xi are formed in registers, exactly as cgemm3m-style kernels do), so the results
// agree with the oracle to rounding (R24, R29).  Structure as gemm_ws_kernel (gemm_ws.cuh):
// persistent, one CTA per SM, producer warpgroup (2 cp.async warps per ring) + two consumer
// warpgroups on alternate tiles, one mbarrier ring per group, C staged through the ring in
// quarters.  Three accumulator sets do not fit a 32x32 complex warp tile, so a warp owns
// (8 MI) x 32 (MI = 3: 24 x 32, 144 accumulator registers) and a group's tile is 16 MI x 64.
#pragma once
#include "gemm_ws.cuh"

namespace mstrsm {

#ifndef MSTRSM_3M_MI
#define MSTRSM_3M_MI 3
#endif
constexpr int k3mMI = MSTRSM_3M_MI;                                      // warp tile (8 MI) x 32
constexpr int k3mBM = 16 * k3mMI, k3mBN = 64, k3mBK = 8;
constexpr int k3mStageElems = (k3mBM + k3mBN) * k3mBK;                 // (BM + 64) x 8 complex
constexpr int k3mRing = (227 * 1024 - 2048) / (2 * k3mStageElems * 16); // deepest ring that fits
constexpr int k3mSmemBytes = 2 * k3mRing * k3mStageElems * 16;

__device__ __forceinline__ int m3_offA_km(int k, int mm) { return k * k3mBM + (mm ^ ((k & 3) << 1)); }
__device__ __forceinline__ int m3_offRK(int r, int k) { return r * k3mBK + (k ^ ((r & 1) << 2)); }
__device__ __forceinline__ int m3_offC(int row, int colq) { return colq * k3mBM + (row ^ (((colq >> 1) & 3) << 1)); }

template <bool OPC>
__global__ void __launch_bounds__(kWsThreads, 1) gemm_ws3m_kernel(GemmArgs<cplx> g, int tiles_m, int ntiles) {
    constexpr int BM = k3mBM, BN = k3mBN, BK = k3mBK, SE = k3mStageElems, RS = k3mRing;
    constexpr int MI = k3mMI, NI = 4;             // warp tile 8 MI x 32
    static_assert(BM * 16 <= SE, "a C quarter must fit in one stage");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    cplx *smem = reinterpret_cast<cplx *>(smem_raw);
    __shared__ uint64_t full_bar[2][RS], empty_bar[2][RS];
    __shared__ int s_d[2][BN];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nk = (g.K + BK - 1) / BK;
    if (tid == 0) {
        for (int q = 0; q < 2; q++)
            for (int s = 0; s < RS; s++) {
                mbar_init(&full_bar[q][s], 64);     // the two producer warps' cp.async arrivals
                mbar_init(&empty_bar[q][s], 4);     // the 4 warps of the consuming group
            }
    }
    __syncthreads();

    if (warp < 4) {
        // ------------------------------------------------------------------ producers
        // warp 2q: A tiles + C columns 0-7 of each quarter; warp 2q+1: X tiles + C columns 8-15 + d_j
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kWsProducerRegs));
        const int q = warp >> 1, half = warp & 1;
        int gk = 0, local = 0;
        auto next_slot = [&]() -> cplx * {
            const int s = gk % RS, r = gk / RS;
            mbar_wait(&empty_bar[q][s], (r & 1) ^ 1);
            return smem + (q * RS + s) * SE;
        };
        auto commit_slot = [&]() { mbar_arrive_cpasync(&full_bar[q][gk % RS]); gk++; };
        const int kl = lane & 7, nl = lane >> 3;
#pragma unroll 1
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, local++) {
            if ((local & 1) != q) continue;
            const int64_t m0 = int64_t(tile % tiles_m) * BM, n0 = int64_t(tile / tiles_m) * BN;
            const bool vm = m0 + lane < g.M, vm2 = lane + 32 < BM && m0 + lane + 32 < g.M;
            const bool mn_in = m0 + BM <= g.M && n0 + BN <= g.N;
            if (half == 0) {   // warm L2 with this tile's C (read through the ring after the k-tiles)
                const int64_t rows = g.M - m0 < BM ? g.M - m0 : int64_t(BM);
#pragma unroll
                for (int c2 = 0; c2 < BN / 32; c2++) {
                    const int64_t gj = n0 + c2 * 32 + lane;
                    if (gj < g.N && rows > 0) {
                        const uintptr_t a0 = reinterpret_cast<uintptr_t>(g.B + (g.c_r0 + m0) + (g.col0 + gj) * g.ldb);
                        const uintptr_t al = a0 & ~uintptr_t(15);
                        const unsigned len = unsigned((a0 - al + rows * 16 + 15) & ~uintptr_t(15));
                        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(al), "r"(len) : "memory");
                    }
                }
            }
#pragma unroll 1
            for (int kt = 0; kt < nk; kt++) {
                cplx *As = next_slot(), *Xs = As + BM * BK;
                const int k0 = kt * BK;
                const bool interior = mn_in && k0 + BK <= g.K;
                if (half == 0) {
                    if (!OPC) {                 // A(mm,k) = U(a_r0+m0+mm, a_c0+k0+k): lane = row
                        const cplx *ua = g.U + (g.a_r0 + m0 + lane) + (g.a_c0 + k0) * g.ldu;
#pragma unroll
                        for (int k = 0; k < BK; k++) {
                            const bool v = interior || (vm && k0 + k < g.K);
                            cp_async<16>(As + m3_offA_km(k, lane), v ? ua + k * g.ldu : g.U, v);
                            if (BM > 32 && lane + 32 < BM) {
                                const bool v2 = (interior || k0 + k < g.K) && vm2;
                                cp_async<16>(As + m3_offA_km(k, lane + 32), v2 ? ua + k * g.ldu + 32 : g.U, v2);
                            }
                        }
                    } else {                    // A(mm,k) = conj(U(a_r0+k0+k, a_c0+m0+mm)): k contiguous
                        const bool vk = k0 + kl < g.K;
                        const cplx *ua = g.U + (g.a_r0 + k0 + kl) + (g.a_c0 + m0 + nl) * g.ldu;
#pragma unroll
                        for (int it = 0; it < BM / 4; it++) {
                            const int mm = 4 * it + nl;
                            const bool v = vk && m0 + mm < g.M;
                            cp_async<16>(As + m3_offRK(mm, kl), v ? ua + (4 * it) * g.ldu : g.U, v);
                        }
                    }
                } else {                        // X(k,nn) = X(x_r0+k0+k, col0+n0+nn): k contiguous
                    const cplx *xb = g.X + (g.x_r0 + k0 + kl) + (g.col0 + n0 + nl) * g.ldx;
                    if (interior) {
#pragma unroll 4
                        for (int it = 0; it < BN / 4; it++)
                            cp_async<16>(Xs + m3_offRK(4 * it + nl, kl), xb + (4 * it) * g.ldx, true);
                    } else {
                        const bool vk = k0 + kl < g.K;
#pragma unroll 4
                        for (int it = 0; it < BN / 4; it++) {
                            const int nn = 4 * it + nl;
                            const bool v = vk && n0 + nn < g.N;
                            cp_async<16>(Xs + m3_offRK(nn, kl), v ? xb + (4 * it) * g.ldx : g.X, v);
                        }
                    }
                }
                commit_slot();
            }
#pragma unroll 1
            for (int cq = 0; cq < 4; cq++) {    // C quarter cq (columns 16cq .. 16cq+15) and its d_j
                cplx *Cs = next_slot();
                const cplx *cb = g.B + (g.c_r0 + m0 + lane) + (g.col0 + n0 + 16 * cq + 8 * half) * g.ldb;
#pragma unroll 4
                for (int c8 = 0; c8 < 8; c8++) {
                    const int colq = 8 * half + c8;
                    const bool vn = n0 + 16 * cq + colq < g.N;
                    cp_async<16>(Cs + m3_offC(lane, colq), vm && vn ? cb + c8 * g.ldb : g.B, vm && vn);
                    if (BM > 32 && lane + 32 < BM)
                        cp_async<16>(Cs + m3_offC(lane + 32, colq), vm2 && vn ? cb + c8 * g.ldb + 32 : g.B, vm2 && vn);
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
    const int wm = wq & 1, wn = wq >> 1;          // rows 8 MI wm .. +8 MI-1, columns 32 wn .. +31
    const int gq = lane >> 2, tq = lane & 3;
    int local = 0, gk = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, local++) {
        if ((local & 1) != grp) continue;
        const int64_t m0 = int64_t(tile % tiles_m) * BM, n0 = int64_t(tile / tiles_m) * BN;

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
            const cplx *As = smem + (grp * RS + s) * SE, *Xs = As + BM * BK;
#pragma unroll
            for (int kk = 0; kk < BK / 4; kk++) {
                const int k = kk * 4 + tq;
                double ar[MI], ai[MI], as[MI], br[NI], bi[NI], bs[NI];
#pragma unroll
                for (int i = 0; i < MI; i++) {
                    const int mm = wm * 8 * MI + i * 8 + gq;
                    const cplx v = OPC ? As[m3_offRK(mm, k)] : As[m3_offA_km(k, mm)];
                    ar[i] = v.x;
                    ai[i] = OPC ? -v.y : v.y;
                    as[i] = __dadd_rn(ar[i], ai[i]);
                }
#pragma unroll
                for (int jn = 0; jn < NI; jn++) {
                    const cplx v = Xs[m3_offRK(wn * 32 + jn * 8 + gq, k)];
                    br[jn] = v.x;
                    bi[jn] = v.y;
                    bs[jn] = __dadd_rn(v.x, v.y);
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
        }

        // ---- epilogue: C = 2^d C - (P1 - P2, P3 - P1 - P2); C and d from the four C quarters
        //      (every warp waits for all four, releases the two it does not read at once and its
        //      own two as it finishes them) ----
        auto sq = [&](int cq) { return (gk + cq) % RS; };
#pragma unroll
        for (int cq = 0; cq < 4; cq++) mbar_wait(&full_bar[grp][sq(cq)], ((gk + cq) / RS) & 1);
        __syncwarp();
        if (lane == 0) { mbar_arrive(&empty_bar[grp][sq(2 - 2 * wn)]); mbar_arrive(&empty_bar[grp][sq(3 - 2 * wn)]); }
        const bool full = m0 + BM <= g.M && n0 + BN <= g.N;
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const cplx *Cs = smem + (grp * RS + sq(2 * wn + h)) * SE;
#pragma unroll
            for (int jj = 0; jj < 2; jj++) {
                const int jn = 2 * h + jj;
#pragma unroll
                for (int c = 0; c < 2; c++) {
                    const int colq = jj * 8 + tq * 2 + c;
                    const int colh = jn * 8 + tq * 2 + c;
                    const int64_t gj = n0 + wn * 32 + colh;
                    const int d = max(g.dblk ? s_d[grp][wn * 32 + colh] : 0, -2044);
                    const bool lo = d < -1022;
                    const double f1 = lo ? __longlong_as_double((long long)(1023 + d + 1022) << 52) : 1.0;
                    const double f2 = __longlong_as_double((long long)(1023 + (lo ? -1022 : d)) << 52);
                    cplx *colp = g.B + g.c_r0 + (g.col0 + gj) * g.ldb;
#pragma unroll
                    for (int i = 0; i < MI; i++) {
                        const int row = wm * 8 * MI + i * 8 + gq;
                        const int64_t gi = m0 + row;
                        const cplx old = Cs[m3_offC(row, colq)];
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
