// mstrsm.cu -- libmstrsm.so: C ABI (include/mstrsm.h) + host orchestration of the blocked
// (safe) multi-shift triangular solve (arXiv 1607.01477, Alg. 3 / Alg. 5) on sm_100a.
//
// Per solve, all on the library stream, no host synchronisation:
//   a.2 norm pass (safe)            norm_cols_n / norm_rows_c, panel_sum, rowsum, delta
//   a.1 init                        init_rhs / init_trevc
//   for every block b (op N bottom-up, op C top-down; P:162-180 / P:362-411):
//     a.3+a.4 diag_kernel           per-column diagonal-block solve, bounds, rescale decision
//     a.5     gemm_update_kernel    B(I0,act) = 2^d B(I0,act) - U(I0,I1) X(I1,act)  (DMMA)
//   a.6 finalize                    lazy exponent fix-up, scales, diag(Z)
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <functional>
#include <thread>
#include <chrono>
#include <vector>

#include "../../include/mstrsm.h"
#include "aux_kernels.cuh"
#include "runtime.cuh"
#include "lanczos_kernels.cuh"

using namespace mstrsm;
using namespace mstrsm::rt;

namespace {

// Device workspace for one solve, carved out of one stream-ordered allocation.
// Caller-provided workspace (mstrsm_*_ex_ws): while a call runs with an arena, every device
// allocation of the solve is carved from it (256-B aligned) and never freed; otherwise
// allocations are stream-ordered from the device pool.
struct Arena {
    char *base = nullptr;
    size_t size = 0, off = 0;
    bool active = false;
};
thread_local Arena g_arena;
cudaError_t ws_malloc(void **p, size_t bytes) {
    if (g_arena.active) {
        const size_t o = (g_arena.off + 255) & ~size_t(255);
        if (o + bytes > g_arena.size) return cudaErrorMemoryAllocation;
        *p = g_arena.base + o;
        g_arena.off = o + bytes;
        return cudaSuccess;
    }
    return cudaMallocAsync(p, bytes, g_stream);
}
void ws_free(void *p, cudaStream_t st) {
    if (!p) return;
    const char *c = static_cast<const char *>(p);
    if (g_arena.active && c >= g_arena.base && c < g_arena.base + g_arena.size) return;
    cudaFreeAsync(p, st);
}

struct Work {
    void *base = nullptr;
    double *cnl = nullptr, *part = nullptr, *P = nullptr, *delta = nullptr, *G = nullptr;
    int *e = nullptr, *dblk = nullptr, *dblk2 = nullptr, *Etab = nullptr;
    int *fb_list = nullptr, *fb_count = nullptr;   // diag fallback: column list, count per block
    int64_t *rowend = nullptr;
    void *shifts = nullptr;            // trevc: gathered diag(T)
    void *xscr = nullptr;              // diagl_kernel scratch: n_b rounded up to 8 rows x n columns
    int64_t ldscr = 0;
    cudaStream_t st = nullptr;
    ~Work() { ws_free(base, st); }
};

template <typename T>
int alloc_work(Work &w, int64_t m, int64_t n, int nb, bool need_rowend, bool need_shifts, size_t *bytes_only = nullptr) {
    int64_t nblk = cdiv(m, nb);
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~size_t(255); return o; };
    size_t o_cnl = take(m * 8), o_part = take(m * 8), o_P = take(std::max<int64_t>(nblk, 1) * 8),
           o_delta = take(16), o_G = take(n * 8), o_e = take(n * 4), o_d = take(n * 4), o_d2 = take(n * 4),
           o_E = take(std::max<int64_t>(nblk, 1) * n * 4), o_r = take(need_rowend ? n * 8 : 0),
           o_fl = take(n * 4), o_fc = take(std::max<int64_t>(nblk, 1) * 4),
           o_s = take(need_shifts ? n * sizeof(T) : 0);
    const int64_t ldscr = (std::min(nb, 128) + 7) / 8 * 8;
    const size_t o_x = take(size_t(ldscr) * std::max<int64_t>(n, 1) * sizeof(T));
    if (bytes_only) { *bytes_only = off; return 0; }
    w.st = g_stream;
    CK(ws_malloc(&w.base, off));
    char *b = static_cast<char *>(w.base);
    w.cnl = (double *)(b + o_cnl); w.part = (double *)(b + o_part); w.P = (double *)(b + o_P);
    w.delta = (double *)(b + o_delta); w.G = (double *)(b + o_G); w.e = (int *)(b + o_e);
    w.dblk = (int *)(b + o_d); w.dblk2 = (int *)(b + o_d2); w.Etab = (int *)(b + o_E);
    w.fb_list = (int *)(b + o_fl); w.fb_count = (int *)(b + o_fc);
    w.rowend = need_rowend ? (int64_t *)(b + o_r) : nullptr;
    w.shifts = need_shifts ? (void *)(b + o_s) : nullptr;
    w.xscr = (void *)(b + o_x);
    w.ldscr = ldscr;
    return 0;
}

template <typename K>
int occupancy(K kern, int threads, size_t smem) {
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, threads, smem) != cudaSuccess) nb = 1;
    return std::max(nb, 1);
}

// ---------------------------------------------------------------- norm pass (a.2)
template <typename T>
int norm_pass(int op, const T *U, int64_t ldu, int64_t m, int nb, Work &w, bool cols_done = false) {
    int64_t nblk = cdiv(m, nb);
    if (op == 0) {
        int blocks = int(std::min<int64_t>(cdiv(m, 8), int64_t(g_num_sms) * 16));
        if (!cols_done) {       // (trevc's fused prepass has produced cnl / pcol already)
            norm_cols_n_kernel<T><<<blocks, 256, 0, g_stream>>>(U, ldu, m, nb, w.cnl, w.part, g_flag);
            CK_LAUNCH("norm_cols_n_kernel");
        }
        panel_sum_kernel<<<int(cdiv(nblk, 128)), 128, 0, g_stream>>>(0, m, nb, nblk, w.part, w.P);
        CK_LAUNCH("panel_sum_kernel");
        int64_t nch = cdiv(m, kRowsumChunk);
        double *part2 = nullptr;
        CK(ws_malloc((void **)&part2, size_t(nch) * m * 8));
        rowsum_n_kernel<T><<<dim3(unsigned(cdiv(m, 128)), unsigned(nch)), 128, 0, g_stream>>>(U, ldu, m, part2);
        CK_LAUNCH("rowsum_n_kernel");
        rowsum_reduce_kernel<<<int(cdiv(m, 128)), 128, 0, g_stream>>>(m, nch, part2, w.part);
        CK_LAUNCH("rowsum_reduce_kernel");
        ws_free(part2, g_stream);
    } else {
        CK(cudaMemsetAsync(w.cnl, 0, size_t(m) * 8, g_stream));
        CK(cudaMemsetAsync(w.part, 0, size_t(m) * 8, g_stream));
        norm_rows_c_chunk_kernel<T><<<dim3(unsigned(cdiv(m, 128)), unsigned(cdiv(m, kRowsumChunk))), 128, 0,
                                      g_stream>>>(U, ldu, m, nb, w.cnl, w.part, g_flag);
        CK_LAUNCH("norm_rows_c_chunk_kernel");
        panel_sum_kernel<<<int(cdiv(nblk, 128)), 128, 0, g_stream>>>(1, m, nb, nblk, w.part, w.P);
        CK_LAUNCH("panel_sum_kernel");
        colsum_c_tiled_kernel<T><<<int(cdiv(m, 32)), 256, 0, g_stream>>>(U, ldu, m, w.part);
        CK_LAUNCH("colsum_c_tiled_kernel");
    }
    delta_kernel<<<1, 1024, 0, g_stream>>>(m, w.part, w.delta);
    CK_LAUNCH("delta_kernel");
    return 0;
}

// ||U||_inf of op N for delta (R4) into delta[0..1] (rowsum + ordered reduction + max).
template <typename T>
int compute_delta_n(const T *U, int64_t ldu, int64_t m, double *rs, double *delta) {
    const int64_t nch = cdiv(m, kRowsumChunk);
    double *part2 = nullptr;
    CK(ws_malloc((void **)&part2, size_t(nch) * m * 8));
    rowsum_n_kernel<T><<<dim3(unsigned(cdiv(m, 128)), unsigned(nch)), 128, 0, g_stream>>>(U, ldu, m, part2);
    CK_LAUNCH("rowsum_n_kernel");
    rowsum_reduce_kernel<<<int(cdiv(m, 128)), 128, 0, g_stream>>>(m, nch, part2, rs);
    CK_LAUNCH("rowsum_reduce_kernel");
    ws_free(part2, g_stream);
    delta_kernel<<<1, 1024, 0, g_stream>>>(m, rs, delta);
    CK_LAUNCH("delta_kernel");
    return 0;
}

// Per-block hook of the blocked solve (this thread's): called at the top of block b, before its
// diagonal step, on the library stream.  The multi-GPU path uses it to wait for T's panel b and run
// that panel's prepass as the panels arrive (trevc_impl with panel_ready).
thread_local const std::function<int(int64_t)> *t_pre_block = nullptr;
// ... and may point block b at its own copy of the triangle's panel b (columns [lo_b, hi_b), rows
// 0 .. hi_b): U(i, k) of block b is t_blk_U[i + k * t_blk_ld] (nullptr: the solve's U, ldu).
thread_local const void *t_blk_U = nullptr;
thread_local int64_t t_blk_ld = 0;
// ... and may be told when block b's diagonal step has been launched (its rows are then final up to
// the lazy exponent fix-up: the multi-GPU path gathers them behind the compute front)
thread_local const std::function<int(int64_t)> *t_after_diag = nullptr;
// With the per-block hook: the panel sums P_b are formed by the diagonal kernel from these
// per-column panel maxima (the same ascending sum panel_sum_kernel does) instead of a launch.
thread_local const double *t_panel_part = nullptr;

// ---------------------------------------------------------------- look-ahead (op N, safe)
// Look-ahead (MSTRSM_LOOKAHEAD=1 enables; off by default since round 2's diagonal kernels: c3 22.2
// ms without vs 22.3 with, the 8-GPU shard 25.2 vs 25.6, c5 equal -- profiles/r02/exp_la_r02.txt,
// the diagonal step is now short enough that confining it to a few SMs costs what the overlap
// saves): block b's update is split into its top n_b rows (the next diagonal block,
// on the library stream) and the rest (on a side stream, on fewer SMs), so that the next
// diagonal step -- latency-bound, and the per-block floor of a multi-GPU shard -- runs on the
// SMs the rest leaves free.  dblk and the X+ plane are double-buffered by block
// parity (the rest of block b still reads them while the diagonal step of b+1 writes).  A block
// overlaps only when the model says it pays (the next diagonal pass outlasts what the rest loses
// on the SMs it gives up); the others run as in blocked_solve.
bool lookahead_enabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("MSTRSM_LOOKAHEAD");
        v = (e && !strcmp(e, "1")) ? 1 : 0;
    }
    return v == 1;
}
template <typename T>
int blocked_solve_la(const T *U, int64_t ldu, int64_t m, const T *shifts, int64_t sstride, T *B, int64_t ldb,
                     int64_t n, const int64_t *rowend_dev, const std::vector<int64_t> *rowend_sorted_host, int nb,
                     Work &w, const double *Usum, double *Xsum, int64_t ldus, int ldxs);

// ---------------------------------------------------------------- the blocked solve
// Paired blocks (pair_blocks below): blocks 2q and 2q+1 (solve order) form a pair.
// After the first block's diagonal step only the second block's rows are updated (a GEMM with
// M = K = n_b); after the second's, the rows beyond both are updated by one GEMM with K = 2 n_b
// (pair_fix in diag_kernel.cuh keeps the exponent bookkeeping of Alg. 5 exact).  The long update
// GEMMs then run at twice the K: at K = n_b = 64 (c4) the per-tile epilogue and pipeline fill weigh
// on the DMMA rate.  The X+ plane holds both blocks of a pair (ld = 2 x n_b rounded).
// Measured (profiles/r02/exp_pair_r02.txt, single vs paired): complex n_b = 64 pays (c4 87.7 ->
// 83.2 ms, c4d 74.1 -> 71.1: its K = 64 updates become K = 128 ones); at n_b = 128 the K = 128
// update is already efficient and the extra launch per pair costs what K = 256 saves (c5 155.7 vs
// 156.3, the 8-GPU shard 25.6 vs 26.0); real data loses (c2 1.30 vs 1.46: the diagonal step
// dominates and the update is one more latency-bound launch).  So: complex with n_b <= 64.
// MSTRSM_PAIR=0 never, =2 always (tests), default by that rule; even n_b only.
template <typename T>
bool pair_blocks(int nb) {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("MSTRSM_PAIR");
        const char *o = getenv("MSTRSM_DIAG_OLD");              // (round 1's kernel has no pair_fix)
        v = (o && o[0] == '1') ? 0 : (e && (e[0] == '0' || e[0] == '2') && !e[1]) ? e[0] - '0' : 1;
    }
    // (even n_b: the two blocks' X+ rows must be contiguous in the plane, and every block's first
    // X+ row 16-byte aligned for the tensor maps)
    return nb % 2 == 0 && (v == 2 || (v == 1 && S<T>::cplx_ && nb <= 64));
}

// State (G, e) must be initialised by the caller (init kernels).  active_from(b) gives the first
// active column of block b when row ends are known on the host and sorted.
template <typename T, bool SAFE>
int blocked_solve(int op, const T *U, int64_t ldu, int64_t m, const T *shifts, int64_t sstride,
                  T *B, int64_t ldb, int64_t n, const int64_t *rowend_dev,
                  const std::vector<int64_t> *rowend_sorted_host, int nb, Work &w,
                  const double *Usum = nullptr, double *Xsum = nullptr, int64_t ldus = 0, int ldxs = 0) {
    int64_t nblk = cdiv(m, nb);
    const bool pair = pair_blocks<T>(nb) && nblk >= 2;
    if constexpr (SAFE) {
        // (small solves: stream/event overhead; real data: the update is cheap next to the diagonal
        // step, which the split would confine to a few SMs -- c2 1.36 ms with, 1.30 ms without)
        if (!pair && op == 0 && m >= 1024 && S<T>::cplx_ && lookahead_enabled())
            return blocked_solve_la<T>(U, ldu, m, shifts, sstride, B, ldb, n, rowend_dev, rowend_sorted_host, nb, w,
                                       Usum, Xsum, ldus, ldxs);
    }
    if (SAFE) CK(cudaMemsetAsync(w.fb_count, 0, nblk * 4, g_stream));   // diag fallback counts
    auto c0_of = [&](const Blk &bl) -> int64_t {
        if (op != 0 || !rowend_sorted_host) return 0;
        const auto &re = *rowend_sorted_host;
        return std::upper_bound(re.begin(), re.end(), bl.lo) - re.begin();   // first r > lo
    };
    const int64_t ldxh = ldxs / 2;             // X+ rows per block of a pair
    // X+ rows of block b within its pair's plane: op N, the second block (above) ends where the
    // first begins (offset ldxh); op C, the first block (above) at 0, the second after it
    auto xs_off = [&](int64_t b, bool second) -> int64_t {
        if (!pair) return 0;
        const Blk bl = block_rows(op, m, nb, b);
        if (op == 0) return second ? ldxh - (bl.hi - bl.lo) : ldxh;
        return second ? ldxh : 0;
    };
    auto after_diag = [&](int64_t b) -> int { return t_after_diag ? (*t_after_diag)(b) : 0; };
    auto debug = [&](int64_t b, const char *what) {
        if (!g_debug_sync) return;
        cudaError_t e = cudaStreamSynchronize(g_stream);
        fprintf(stderr, "[mstrsm debug] block %lld %s done (%s)\n", (long long)b, what, cudaGetErrorString(e));
    };
    int early = 0;                             // U / cnl ready: later launches stage before the wait
    bool first_ran = false;                    // pair: the first block of the current pair ran its step
    int64_t c0_first = 0;
    for (int64_t b = 0; b < nblk; b++) {
        if (t_pre_block) {
            if (int rc = (*t_pre_block)(b)) return rc;
        }
        const T *Ub = t_blk_U ? static_cast<const T *>(t_blk_U) : U;   // this block's view of U
        const int64_t ldub = t_blk_U ? t_blk_ld : ldu;
        // (the pairing depends on the block index only, never on which columns are active, so a
        // column's arithmetic is the same in every column subset: multi-GPU shards reproduce the
        // single-GPU solve bit for bit.  A first block without active columns has X = 0 and no
        // exponent deltas; its pair's second block still runs the merged update.)
        const bool is_first = pair && (b % 2 == 0) && b + 1 < nblk;
        const bool is_second = pair && (b % 2 == 1);
        const Blk bl = block_rows(op, m, nb, b);
        const int64_t c0 = c0_of(bl);
        const int64_t ncols = n - c0;
        if (ncols <= 0) {                      // (the after-diag hook's collectives run on every rank)
            if (is_first) { first_ran = false; c0_first = n; }
            if (is_second && first_ran) {
                // (not reached with sorted row ends: a block's active columns include those of the
                // block solved before it) the first block's update of the rows beyond the pair alone
                first_ran = false;
                if (int rc = after_diag(b - 1)) return rc;
                const Blk bp = block_rows(op, m, nb, b - 1);
                GemmArgs<T> g{};
                g.U = Ub; g.ldu = ldub; g.B = B; g.ldb = ldb; g.X = B; g.ldx = ldb;
                g.dblk = SAFE ? w.dblk : nullptr;
                g.M = op == 0 ? bl.lo : m - bl.hi; g.N = n - c0_first; g.K = int(bp.hi - bp.lo);
                if (op == 0) { g.a_r0 = 0; g.a_c0 = bp.lo; g.c_r0 = 0; }
                else { g.a_r0 = bp.lo; g.a_c0 = bl.hi; g.c_r0 = bl.hi; }
                g.x_r0 = bp.lo; g.col0 = c0_first;
                if (Usum && Xsum) { g.As = Usum; g.ldas = ldus; g.Xsum = Xsum + xs_off(b - 1, false); g.ldxs = ldxs; }
                if (g.M > 0 && g.N > 0) {
                    if (int rc = op == 0 ? launch_gemm<T, false>(g) : launch_gemm<T, true>(g)) return rc;
                }
            }
            if (int rc = after_diag(b)) return rc;
            continue;
        }
        double *xs = Xsum ? Xsum + xs_off(b, is_second) : nullptr;
        DiagArgs<T> a{};
        a.U = Ub; a.ldu = ldub; a.m = m; a.shifts = shifts; a.sstride = sstride;
        a.B = B; a.ldb = ldb; a.c0 = c0; a.ncols = ncols; a.n = n;
        a.rowend = op == 0 ? rowend_dev : nullptr;
        a.lo = bl.lo; a.hi = bl.hi; a.b = b;
        a.cnl = w.cnl; a.P = w.P; a.delta = w.delta;
        a.G = w.G; a.e = w.e; a.dblk = is_second ? w.dblk2 : w.dblk; a.Etab = w.Etab;
        a.fb_list = w.fb_list; a.fb_count = w.fb_count + b;
        a.force_fb = g_diag_force_fb;
        a.early = early;
        a.Xscr = static_cast<T *>(w.xscr); a.ldscr = w.ldscr;
        a.Ppart = t_panel_part;
        a.Xsum = xs; a.ldxs = ldxs;
        if (SAFE && is_second && first_ran) {
            const Blk bp = block_rows(op, m, nb, b - 1);
            a.dprev = w.dblk; a.c0prev = c0_first; a.plo = bp.lo; a.phi = bp.hi; a.bprev = b - 1;
            a.xsprev = Xsum ? Xsum + xs_off(b - 1, false) : nullptr;
        }
        if (xs && rowend_dev && !rowend_sorted_host)          // inactive columns in range: zero rows
            CK(cudaMemset2DAsync(xs + c0 * ldxs, size_t(ldxs) * 8, 0, size_t(bl.hi - bl.lo) * 8, size_t(ncols),
                                 g_stream));
        int rc = op == 0 ? launch_diag<T, SAFE, 0>(a, nb) : launch_diag<T, SAFE, 1>(a, nb);
        early = t_pre_block ? 0 : 1;           // (a per-block prepass writes cnl right before the diag)
        if (rc) return rc;
        // the after-diag hook sees final rows only: a pair's first block's rows may still be
        // rescaled by the second block's step
        if (!is_first) {
            if (is_second && first_ran && (rc = after_diag(b - 1))) return rc;
            if ((rc = after_diag(b))) return rc;
        }
        debug(b, "diag");
        GemmArgs<T> g{};
        g.U = Ub; g.ldu = ldub; g.B = B; g.ldb = ldb;
        g.X = B; g.ldx = ldb;
        g.dblk = SAFE ? a.dblk : nullptr;
        if (is_first) {
            // the second block's rows only, K = K_b
            const Blk bn = block_rows(op, m, nb, b + 1);
            g.M = bn.hi - bn.lo; g.N = ncols; g.K = int(bl.hi - bl.lo);
            if (op == 0) { g.a_r0 = bn.lo; g.a_c0 = bl.lo; g.c_r0 = bn.lo; }
            else { g.a_r0 = bl.lo; g.a_c0 = bn.lo; g.c_r0 = bn.lo; }
            g.x_r0 = bl.lo; g.col0 = c0;
            if (Usum && xs) { g.As = Usum; g.ldas = ldus; g.Xsum = xs; g.ldxs = ldxs; }
            first_ran = true;
            c0_first = c0;
        } else if (is_second) {
            // the rows beyond both blocks, K = K_p + K_b over rows [lo, hi) of the pair
            const Blk bp = block_rows(op, m, nb, b - 1);
            const int64_t plo = std::min(bl.lo, bp.lo), phi = std::max(bl.hi, bp.hi);
            g.M = op == 0 ? plo : m - phi; g.N = ncols; g.K = int(phi - plo);
            if (op == 0) { g.a_r0 = 0; g.a_c0 = plo; g.c_r0 = 0; }
            else { g.a_r0 = plo; g.a_c0 = phi; g.c_r0 = phi; }
            g.x_r0 = plo; g.col0 = c0;
            first_ran = false;
            if (g.M <= 0) continue;
            if (Usum && Xsum) {
                double *xsp = Xsum + (op == 0 ? xs_off(b, true) : 0);
                // the first block's X+ rows of the columns its step did not cover (X = 0 there)
                if (c0_first > c0)
                    CK(cudaMemset2DAsync(Xsum + xs_off(b - 1, false) + c0 * ldxs, size_t(ldxs) * 8, 0,
                                         size_t(bp.hi - bp.lo) * 8, size_t(c0_first - c0), g_stream));
                g.As = Usum; g.ldas = ldus; g.Xsum = xsp; g.ldxs = ldxs;
            }
        } else {
            g.M = op == 0 ? bl.lo : m - bl.hi; g.N = ncols; g.K = int(bl.hi - bl.lo);
            if (g.M <= 0) continue;
            if (op == 0) { g.a_r0 = 0; g.a_c0 = bl.lo; g.c_r0 = 0; }
            else { g.a_r0 = bl.lo; g.a_c0 = bl.hi; g.c_r0 = bl.hi; }
            g.x_r0 = bl.lo; g.col0 = c0;
            if (Usum && xs) { g.As = Usum; g.ldas = ldus; g.Xsum = xs; g.ldxs = ldxs; }
        }
        if (g.M > 0) {
            rc = op == 0 ? launch_gemm<T, false>(g) : launch_gemm<T, true>(g);
            if (rc) return rc;
            debug(b, "gemm");
        }
    }
    return 0;
}

template <typename T>
int blocked_solve_la(const T *U, int64_t ldu, int64_t m, const T *shifts, int64_t sstride, T *B, int64_t ldb,
                     int64_t n, const int64_t *rowend_dev, const std::vector<int64_t> *rowend_sorted_host, int nb,
                     Work &w, const double *Usum, double *Xsum, int64_t ldus, int ldxs) {
    DevRes *res = dev_res();                    // this thread's side stream and events on this device
    if (!res) return 1;
    const cudaStream_t side = res->side;
    const cudaEvent_t ev_d = res->ev_d, ev_rest = res->ev_rest;
    const cudaStream_t main_st = g_stream;
    const int64_t nblk = cdiv(m, nb);
    CK(cudaMemsetAsync(w.fb_count, 0, nblk * 4, g_stream));
    double *Xsum2 = nullptr;
    if (Xsum) CK(ws_malloc((void **)&Xsum2, size_t(ldxs) * std::max<int64_t>(n, 1) * 8));
    auto c0_of = [&](const Blk &bl) -> int64_t {
        if (!rowend_sorted_host) return 0;
        const auto &re = *rowend_sorted_host;
        return std::upper_bound(re.begin(), re.end(), bl.lo) - re.begin();
    };
    // columns one CTA of the next diagonal step covers in one pass: the n_b > 64 complex layout
    // (16, 8) has 15 substitution warps of 2 columns (diag_launch.cuh); MSTRSM_LA_COLS overrides
    static const int kColsPerCta = [] { const char *e = getenv("MSTRSM_LA_COLS"); const int v = e ? atoi(e) : 0; return v > 0 ? v : 30; }();
    const int cap_max = g_num_sms / 3;
    bool rest_pending = false;
    int diag_cap = 0;                          // CTAs the next diagonal step may use (0: all)
    int early = 0;
    int rc = 0;
    for (int64_t b = 0; b < nblk && !rc; b++) {
        if (t_pre_block) {
            if ((rc = (*t_pre_block)(b))) break;
        }
        const T *Ub = t_blk_U ? static_cast<const T *>(t_blk_U) : U;   // this block's view of U
        const int64_t ldub = t_blk_U ? t_blk_ld : ldu;
        const Blk bl = block_rows(0, m, nb, b);
        const int64_t c0 = c0_of(bl), ncols = n - c0;
        if (ncols <= 0) {
            diag_cap = 0;
            if (t_after_diag && (rc = (*t_after_diag)(b))) break;
            continue;
        }
        const int par = int(b & 1);
        int *dblk = par ? w.dblk2 : w.dblk;
        double *xs = Xsum ? (par ? Xsum2 : Xsum) : nullptr;
        DiagArgs<T> a{};
        a.U = Ub; a.ldu = ldub; a.m = m; a.shifts = shifts; a.sstride = sstride;
        a.B = B; a.ldb = ldb; a.c0 = c0; a.ncols = ncols; a.n = n;
        a.rowend = rowend_dev;
        a.lo = bl.lo; a.hi = bl.hi; a.b = b;
        a.cnl = w.cnl; a.P = w.P; a.delta = w.delta;
        a.G = w.G; a.e = w.e; a.dblk = dblk; a.Etab = w.Etab;
        a.fb_list = w.fb_list; a.fb_count = w.fb_count + b;
        a.force_fb = g_diag_force_fb;
        a.early = early;
        a.Xscr = static_cast<T *>(w.xscr); a.ldscr = w.ldscr;
        a.Ppart = t_panel_part;
        a.Xsum = xs; a.ldxs = ldxs;
        if (xs && rowend_dev && !rowend_sorted_host)          // inactive columns in range: zero rows
            CK(cudaMemsetAsync(xs + c0 * ldxs, 0, size_t(ncols) * ldxs * 8, g_stream));
        g_cta_cap = diag_cap;
        rc = launch_diag<T, true, 0>(a, nb);
        g_cta_cap = 0;
        early = t_pre_block ? 0 : 1;
        if (rc) break;
        if (t_after_diag && (rc = (*t_after_diag)(b))) break;
        diag_cap = 0;
        const int64_t M = bl.lo;
        if (M <= 0) continue;
        GemmArgs<T> g{};
        g.U = Ub; g.ldu = ldub; g.B = B; g.ldb = ldb;
        g.N = ncols; g.K = int(bl.hi - bl.lo);
        g.a_c0 = bl.lo; g.x_r0 = bl.lo; g.col0 = c0;
        g.X = B; g.ldx = ldb;
        if (Usum && xs) { g.As = Usum; g.ldas = ldus; g.Xsum = xs; g.ldxs = ldxs; }
        g.dblk = dblk;
        // the next block: rows [bn.lo, M) of this update; how many SMs would its diagonal step need?
        const Blk bn = block_rows(0, m, nb, b + 1);
        const int64_t Mtop = M - bn.lo;
        const int64_t ncols_next = n - c0_of(bn);
        const int X = int(cdiv(std::max<int64_t>(ncols_next, 1), kColsPerCta));
        // pays when the next diagonal step (one pass, ~100 us at n_b = 128) outlasts what the rest
        // of this update loses on the SMs it gives up (update at ~30 TF/s executed on all SMs)
        const double t_gemm = 6.0 * double(M) * double(ncols) * double(g.K) / 30e12;
        const double t_diag = 100e-6 * double(bn.hi - bn.lo) / 128.0;
        const bool overlap = Mtop < M && X <= cap_max && X < g_num_sms &&
                             t_diag > t_gemm * double(X) / double(g_num_sms - X) + 10e-6;
        if (!overlap) {                        // as blocked_solve
            if (rest_pending) { CK(cudaStreamWaitEvent(main_st, ev_rest, 0)); rest_pending = false; }
            g.M = M; g.a_r0 = 0; g.c_r0 = 0;
            rc = launch_gemm<T, false>(g);
            continue;
        }
        CK(cudaEventRecord(ev_d, main_st));                 // diagonal step b done
        if (rest_pending) CK(cudaStreamWaitEvent(main_st, ev_rest, 0));   // rows of b+1 fully updated
        // top: the next diagonal block's rows, on the SMs its diagonal step will use
        GemmArgs<T> gt = g;
        gt.M = Mtop; gt.a_r0 = M - Mtop; gt.c_r0 = M - Mtop;
        g_cta_cap = X;
        rc = launch_gemm<T, false>(gt);
        g_cta_cap = 0;
        if (rc) break;
        // rest: rows [0, M - Mtop) on the side stream, on the other SMs
        CK(cudaStreamWaitEvent(side, ev_d, 0));
        GemmArgs<T> gr = g;
        gr.M = M - Mtop; gr.a_r0 = 0; gr.c_r0 = 0;
        g_stream = side;
        g_cta_cap = g_num_sms - X;
        rc = launch_gemm<T, false>(gr);
        g_cta_cap = 0;
        g_stream = main_st;
        if (rc) break;
        CK(cudaEventRecord(ev_rest, side));
        rest_pending = true;
        diag_cap = X;
    }
    g_stream = main_st;
    g_cta_cap = 0;
    if (rest_pending) CK(cudaStreamWaitEvent(main_st, ev_rest, 0));
    if (Xsum2) ws_free(Xsum2, main_st);
    return rc;
}

// Sum planes for the complex 3M update (nullptr when the 3-product kernel is not in use or T is
// real): Usum (m x m doubles, strictly upper part) for operator op, Xsum (nb x n doubles).
struct SumPlanes {
    double *U = nullptr, *X = nullptr;
    int64_t ldu = 0;
    int ldx = 0;
    cudaStream_t st = nullptr;
    ~SumPlanes() { ws_free(U, st); ws_free(X, st); }
};
template <typename T>
int make_sum_planes(SumPlanes &sp, int op, const T *U, int64_t ldu, int64_t m, int64_t n, int nb, bool fill = true) {
    if constexpr (!S<T>::cplx_) return 0;
    else {
        if (gemm_variant() != 0 || m == 0 || !gemm_presum_enabled()) return 0;
        sp.st = g_stream;
        // even leading dimensions (16-byte aligned bulk copies), ldu > m so that a copy rounded
        // up to 16 bytes past the last row of a column stays inside that column
        sp.ldu = (m + 2) & ~int64_t(1);
        sp.ldx = 2 * ((nb + 1) & ~1);              // both blocks of a pair (blocked_solve)
        CK(ws_malloc((void **)&sp.U, size_t(sp.ldu) * m * 8));
        CK(ws_malloc((void **)&sp.X, size_t(sp.ldx) * std::max<int64_t>(n, 1) * 8));
        if (!fill) return 0;                        // the caller's kernel writes the plane
        int blocks = int(std::min<int64_t>(cdiv(m, 8), int64_t(g_num_sms) * 16));
        presum_kernel<<<blocks, 256, 0, g_stream>>>(U, ldu, m, sp.U, sp.ldu, op == 0 ? 1.0 : -1.0);
        CK_LAUNCH("presum_kernel");
        return 0;
    }
}

template <typename T>
int finalize(int op, int safe, T *B, int64_t ldb, int64_t m, int64_t n, int nb,
             const int64_t *rowend_dev, double *scales, int *scale_exp, const int64_t *diag_row,
             Work &w) {
    int blocks = int(std::min<int64_t>(cdiv(n, 8), int64_t(g_num_sms) * 16));
    if (blocks < 1) blocks = 1;
    CK(launch_k_lvl(2, finalize_kernel<T>, dim3(blocks), dim3(256), 0, g_stream, op, B, ldb, m, n, nb, cdiv(m, nb),
                rowend_dev, safe ? (const int *)w.e : nullptr, safe ? (const int *)w.Etab : nullptr, scales,
                scale_exp, diag_row));
    CK_LAUNCH("finalize_kernel");
    return 0;
}

bool is_sorted_nondecreasing(const int64_t *v, int64_t n) {
    for (int64_t i = 1; i < n; i++)
        if (v[i] < v[i - 1]) return false;
    return true;
}

// row_end (a device array; host memory accepted too).  The values are needed on the host
// to skip inactive columns per block when they are non-decreasing, so a device row_end is read back
// with one copy on the caller's stream (which waits for the work already enqueued on it).  The
// clamped values go to w.rowend.  Returns 0 or 1 (CUDA error).
int load_row_end(const int64_t *row_end, int64_t n, int64_t m, int64_t *rowend_dev,
                 std::vector<int64_t> &re_host, bool &sorted) {
    cudaPointerAttributes at{};
    cudaError_t e = cudaPointerGetAttributes(&at, row_end);
    if (e != cudaSuccess) {
        (void)cudaGetLastError();
        at.type = cudaMemoryTypeUnregistered;
    }
    re_host.resize(size_t(n));
    if (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) {
        CK(cudaMemcpyAsync(re_host.data(), row_end, size_t(n) * 8, cudaMemcpyDeviceToHost, g_stream));
        CK(cudaStreamSynchronize(g_stream));
    } else {
        std::copy(row_end, row_end + n, re_host.begin());
    }
    for (auto &v : re_host) v = v < 0 ? 0 : (v > m ? m : v);
    sorted = is_sorted_nondecreasing(re_host.data(), n);
    CK(cudaMemcpyAsync(rowend_dev, re_host.data(), size_t(n) * 8, cudaMemcpyHostToDevice, g_stream));
    return 0;  // (a copy from pageable memory has consumed its source when it returns)
}

template <typename T>
int mstrsm_ex_impl(int safe, int op, const T *U, int64_t ldu, int64_t m, const T *shifts,
                   int64_t sstride, T *B, int64_t ldb, int64_t n, const int64_t *row_end,
                   double *scales, int32_t *scale_exp, int nb) {
    if (safe != 0 && safe != 1) return -1;
    if (op != 0 && op != 1) return -2;
    if (m < 0) return -5;
    if (ldu < std::max<int64_t>(1, m)) return -4;
    if (sstride < 0) return -7;
    if (ldb < std::max<int64_t>(1, m)) return -9;
    if (n < 0) return -10;
    if (nb == 0) nb = 64;
    if (nb < 1 || nb > 128) return -14;
    if (op == 1 && row_end) return -11;
    if (m == 0 || n == 0) return 0;
    if (!U) return -3;
    if (!shifts) return -6;
    if (!B) return -8;
    if (safe && !scales) return -12;
    if (int rc = ensure_init()) return rc;

    Work w;
    if (int rc = alloc_work<T>(w, m, n, nb, row_end != nullptr, false)) return rc;
    std::vector<int64_t> re_host;
    bool sorted = false;
    if (row_end)
        if (int rc = load_row_end(row_end, n, m, w.rowend, re_host, sorted)) return rc;
    int blocks = int(std::min<int64_t>(cdiv(n, 8), int64_t(g_num_sms) * 16));
    if (safe) {
        if (int rc = norm_pass<T>(op, U, ldu, m, nb, w)) return rc;
        init_rhs_kernel<T><<<blocks, 256, 0, g_stream>>>(B, ldb, m, n, w.rowend, shifts, sstride, w.G, w.e, g_flag);
        CK_LAUNCH("init_rhs_kernel");
        SumPlanes sp;
        if (int rc = make_sum_planes<T>(sp, op, U, ldu, m, n, nb)) return rc;
        int rc = blocked_solve<T, true>(op, U, ldu, m, shifts, sstride, B, ldb, n, w.rowend,
                                        sorted ? &re_host : nullptr, nb, w, sp.U, sp.X, sp.ldu, sp.ldx);
        if (rc) return rc;
    } else {
        if (w.rowend) {
            init_rhs_kernel<T><<<blocks, 256, 0, g_stream>>>(B, ldb, m, n, w.rowend, nullptr, 0, nullptr, nullptr, nullptr);
            CK_LAUNCH("init_rhs_kernel");
        }
        SumPlanes sp;
        if (int rc = make_sum_planes<T>(sp, op, U, ldu, m, n, nb)) return rc;
        int rc = blocked_solve<T, false>(op, U, ldu, m, shifts, sstride, B, ldb, n, w.rowend,
                                         sorted ? &re_host : nullptr, nb, w, sp.U, sp.X, sp.ldu, sp.ldx);
        if (rc) return rc;
    }
    if (scales || scale_exp || safe)
        if (int rc = finalize<T>(op, safe, B, ldb, m, n, nb, w.rowend, scales, scale_exp, nullptr, w)) return rc;
    return 0;
}

// T fed panel by panel (the multi-GPU path): `enqueue(b)` puts the arrival of panel b -- columns
// [lo_b, hi_b) of T, rows 0 .. hi_b, op N block order (b = 0: the last columns) -- on stream cs;
// delta[0..1] (R4) is valid on cs before panel 0.  trevc_impl puts each panel's prepass on cs
// right behind its arrival and makes block b wait only for that.
struct PanelFeed {
    cudaStream_t cs;
    std::function<int(int64_t)> enqueue;
    const double *delta;
    std::function<void(int64_t, const void **, int64_t *)> view;   // nullable: block b's copy of panel b
    std::function<int(int64_t)> after_diag;   // nullable: block b's diagonal step launched (library stream)
    int *etab_out = nullptr;    // non-null: no lazy fix-up here; E (nblk x ncols) copied to etab_out,
    int64_t ld_etab = 0;        //   row b at etab_out + b * ld_etab, for the receiver's fix-up
};

template <typename T>
int trevc_impl(const T *Tm, int64_t ldt, int64_t m, const int64_t *cols_host, int64_t ncols,
               T *Z, int64_t ldz, double *scales, int32_t *scale_exp, int nb, const PanelFeed *feed = nullptr) {
    if (m < 0) return -3;
    if (ldt < std::max<int64_t>(1, m)) return -2;
    if (ncols < 0) return -5;
    if (ldz < std::max<int64_t>(1, m)) return -7;
    if (nb == 0) nb = 64;
    if (nb < 1 || nb > 128) return -10;
    if (m == 0 || ncols == 0) return 0;
    if (!Tm) return -1;
    if (!Z) return -6;
    std::vector<int64_t> cols(ncols);
    for (int64_t q = 0; q < ncols; q++) {
        cols[q] = cols_host ? cols_host[q] : q;
        if (cols[q] < 0 || cols[q] >= m || (q > 0 && cols[q] <= cols[q - 1])) return -4;
    }
    if (int rc = ensure_init()) return rc;
    Work w;
    if (int rc = alloc_work<T>(w, m, ncols, nb, true, true)) return rc;
    T *sh = static_cast<T *>(w.shifts);
    SumPlanes sp;
    // one pass over T for the column norms (all columns), Z / G / row_end / shifts of the requested
    // columns and the 3M sum plane
    const bool all_cols = ncols == m && cols.back() == m - 1;      // strictly increasing: the identity
    int *qof = nullptr;
    std::vector<int> qh;
    if (!all_cols) {                    // eigenvector k -> column q of Z (or -1)
        qh.assign(m, -1);
        for (int64_t q = 0; q < ncols; q++) qh[cols[q]] = int(q);
        CK(cudaMallocAsync(&qof, size_t(m) * 4, g_stream));
        CK(cudaMemcpyAsync(qof, qh.data(), size_t(m) * 4, cudaMemcpyHostToDevice, g_stream));
    }
    if (int rc = make_sum_planes<T>(sp, 0, Tm, ldt, m, ncols, nb, /*fill=*/false)) return rc;
    std::function<int(int64_t)> hook;
    std::vector<cudaEvent_t> pev;               // panel b's arrival + prepass done (feed mode)
    struct PevGuard {
        std::vector<cudaEvent_t> &v;
        ~PevGuard() { for (auto e : v) cudaEventDestroy(e); }
    } pevg{pev};
    if (!feed) {
        int blocks = int(std::min<int64_t>(cdiv(m, 8), int64_t(g_num_sms) * 16));
        trevc_prepass_kernel<T><<<blocks, 256, 0, g_stream>>>(Tm, ldt, m, nb, w.cnl, w.part, Z, ldz, sh, w.rowend,
                                                               w.G, w.e, sp.U, sp.ldu, g_flag, qof);
        CK_LAUNCH("trevc_prepass_kernel");
        if (int rc = norm_pass<T>(0, Tm, ldt, m, nb, w, /*cols_done=*/true)) return rc;
    } else {
        // T arrives panel by panel (right to left, the order the blocks consume it): every block
        // waits for its own panel and computes that panel's part of the prepass (column norms,
        // panel sum P_b, Z / G / row_end / shifts of the requested columns, 3M sum plane)
        CK(cudaMemsetAsync(w.cnl, 0, size_t(m) * 8, g_stream));        // (atomic maxima below)
        CK(cudaMemsetAsync(w.part, 0, size_t(m) * 8, g_stream));
        CK(cudaMemsetAsync(w.G, 0, size_t(ncols) * 8, g_stream));
        const int64_t nblk = cdiv(m, nb);
        pev.resize(size_t(nblk) + 1);
        for (auto &e : pev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CK(cudaEventRecord(pev[nblk], g_stream));                      // workspace ready
        CK(cudaStreamWaitEvent(feed->cs, pev[nblk], 0));
        for (int64_t b = 0; b < nblk; b++) {                           // everything on the comm stream
            if (int rc = feed->enqueue(b)) return rc;
            const Blk bl = block_rows(0, m, nb, b);
            const T *Tb = Tm;
            int64_t ldtb = ldt;
            if (feed->view) {
                const void *pv = nullptr;
                feed->view(b, &pv, &ldtb);
                Tb = static_cast<const T *>(pv);
            }
            const int64_t rchunk = 1024;                               // one panel over the whole GPU
            const dim3 grid(unsigned(cdiv(bl.hi - bl.lo, 8)), unsigned(cdiv(bl.hi, rchunk)));
            trevc_prepass_panel_kernel<T><<<grid, 256, 0, feed->cs>>>(Tb, ldtb, m, nb, w.cnl, w.part, Z, ldz, sh,
                                                                       w.rowend, w.G, w.e, sp.U, sp.ldu, g_flag, qof,
                                                                       bl.lo, bl.hi, rchunk);
            CK_LAUNCH("trevc_prepass_panel_kernel");
            CK(cudaEventRecord(pev[b], feed->cs));
        }
        CK(cudaStreamWaitEvent(g_stream, pev[0], 0));
        CK(cudaMemcpyAsync(w.delta, feed->delta, 2 * sizeof(double), cudaMemcpyDeviceToDevice, g_stream));
        t_panel_part = w.part;                 // the diagonal kernel forms P_b from the panel's pcol
        hook = [&](int64_t b) -> int {
            CK(cudaStreamWaitEvent(g_stream, pev[b], 0));
            if (feed->view) feed->view(b, &t_blk_U, &t_blk_ld);
            return 0;
        };
        if (feed->after_diag) t_after_diag = &feed->after_diag;
        t_pre_block = &hook;
    }
    int rc = blocked_solve<T, true>(0, Tm, ldt, m, sh, 1, Z, ldz, ncols, w.rowend, &cols, nb, w, sp.U, sp.X, sp.ldu, sp.ldx);
    t_pre_block = nullptr;
    t_panel_part = nullptr;
    t_blk_U = nullptr;
    t_after_diag = nullptr;
    if (qof) cudaFreeAsync(qof, g_stream);
    if (!rc && feed && feed->etab_out) {       // the receiver applies the fix-up (a.6) itself
        const int blocks = int(std::min<int64_t>(cdiv(ncols, 8), int64_t(g_num_sms) * 16));
        CK(launch_k_lvl(2, finalize_kernel<T>, dim3(std::max(blocks, 1)), dim3(256), 0, g_stream, 0, Z, ldz, m,
                        ncols, nb, cdiv(m, nb), (const int64_t *)w.rowend, (const int *)w.e, (const int *)nullptr,
                        scales, scale_exp, (const int64_t *)nullptr));
        CK_LAUNCH("finalize_kernel");
        CK(cudaMemcpy2DAsync(feed->etab_out, size_t(feed->ld_etab) * 4, w.Etab, size_t(ncols) * 4, size_t(ncols) * 4,
                             size_t(cdiv(m, nb)), cudaMemcpyDeviceToDevice, g_stream));
        return 0;
    }
    if (!rc) rc = finalize<T>(0, 1, Z, ldz, m, ncols, nb, w.rowend, scales, scale_exp, w.rowend, w);
    return rc;
}

// ---------------------------------------------------------------- side / triangle variants (f4)
// The footnote family of P:58-62 on top of the two kernels the path has (op N: back substitution
// on U; op C: forward substitution on U^H = lower):
//   left  lower  (A - sI) x = c b            ==  op C on U = A^H,      shifts conj(s)
//   right upper  x^T (A - sI) = c b^T        ==  op C on U = conj(A),  shifts conj(s), on B^T
//   right lower  x^T (A - sI) = c b^T        ==  op N on U = A^T,      shifts s,       on B^T
// (right: row j of the n x m array B is b_j^T).  The operand transforms are one tiled pass over
// the triangle (and two over B for the right cases) into workspace; the solves are the hot path.
template <typename T>
int side_impl(int safe, int side, int uplo, const T *A, int64_t lda, int64_t m, const T *shifts, int64_t sstride,
              T *B, int64_t ldb, int64_t n, double *scales, int32_t *scale_exp, int nb) {
    if (safe != 0 && safe != 1) return -1;
    if (side != 0 && side != 1) return -2;
    if (uplo != 0 && uplo != 1) return -3;
    if (m < 0) return -6;
    if (lda < std::max<int64_t>(1, m)) return -5;
    if (sstride < 0) return -8;
    if (n < 0) return -11;
    if (ldb < std::max<int64_t>(1, side == 0 ? m : n)) return -10;
    if (nb != 0 && (nb < 1 || nb > 128)) return -14;
    if (m == 0 || n == 0) return 0;
    if (!A) return -4;
    if (!shifts) return -7;
    if (!B) return -9;
    if (safe && !scales) return -12;
    if (side == 0 && uplo == 0)
        return mstrsm_ex_impl<T>(safe, 0, A, lda, m, shifts, sstride, B, ldb, n, nullptr, scales, scale_exp, nb);
    if (int rc = ensure_init()) return rc;
    const bool cplx_t = S<T>::cplx_;
    // transformed triangle (real right-upper needs none: conj(A) = A)
    const bool need_u = !(side == 1 && uplo == 0 && !cplx_t);
    const int mode = (side == 0) ? 0 : (uplo == 0 ? 2 : 1);
    const int op = (side == 1 && uplo == 1) ? 0 : 1;
    const bool conj_s = op == 1 && cplx_t;
    T *Uw = nullptr, *sw = nullptr, *Bt = nullptr;
    auto cleanup = [&]() {
        if (Uw) cudaFreeAsync(Uw, g_stream);
        if (sw) cudaFreeAsync(sw, g_stream);
        if (Bt) cudaFreeAsync(Bt, g_stream);
    };
    const T *Uuse = A;
    int64_t lduse = lda;
    if (need_u) {
        CK(cudaMallocAsync(&Uw, size_t(m) * m * sizeof(T), g_stream));
        const dim3 g(unsigned(cdiv(m, 32)), unsigned(cdiv(m, 32)));
        tri_upper_kernel<T><<<g, dim3(32, 8), 0, g_stream>>>(A, lda, m, Uw, m, mode);
        CK_LAUNCH("tri_upper_kernel");
        Uuse = Uw;
        lduse = m;
    }
    const T *suse = shifts;
    int64_t sst = sstride;
    if (conj_s) {
        CK(cudaMallocAsync(&sw, size_t(n) * sizeof(T), g_stream));
        conj_strided_kernel<T><<<int(cdiv(n, 256)), 256, 0, g_stream>>>(shifts, sstride, n, sw);
        CK_LAUNCH("conj_strided_kernel");
        suse = sw;
        sst = 1;
    }
    T *Buse = B;
    int64_t ldbuse = ldb;
    if (side == 1) {                    // B is n x m: solve on B^T (m x n)
        CK(cudaMallocAsync(&Bt, size_t(m) * n * sizeof(T), g_stream));
        transpose_kernel<T><<<dim3(unsigned(cdiv(n, 32)), unsigned(cdiv(m, 32))), dim3(32, 8), 0, g_stream>>>(
            B, ldb, n, m, Bt, m);
        CK_LAUNCH("transpose_kernel");
        Buse = Bt;
        ldbuse = m;
    }
    int rc = mstrsm_ex_impl<T>(safe, op, Uuse, lduse, m, suse, sst, Buse, ldbuse, n, nullptr, scales, scale_exp, nb);
    if (rc < 0) rc = 1;                 // arguments were validated above
    if (!rc && side == 1) {
        transpose_kernel<T><<<dim3(unsigned(cdiv(m, 32)), unsigned(cdiv(n, 32))), dim3(32, 8), 0, g_stream>>>(
            Bt, m, m, n, B, ldb);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) rc = set_cuda_error(e, "transpose_kernel");
    }
    cleanup();
    return rc;
}

// ---------------------------------------------------------------- back-transformation (f2)
// X := Q Z.  The update GEMM computes C <- C - A X, so X is zeroed, receives -Q Z
// panel by panel and is negated once.  Panel p (columns [p0, p1)) only needs rows 0..cols[p1-1]
// of Z (zero below, TRMM shape): K = cols[p1-1] + 1, about m/(2 W) extra flops over the exact
// triangle for W = 1024-column panels.
template <typename T>
int backtransform_impl(const T *Q, int64_t ldq, int64_t m, const T *Z, int64_t ldz, int64_t n,
                       const int64_t *cols_host, T *X, int64_t ldx) {
    if (m < 0) return -3;
    if (ldq < std::max<int64_t>(1, m)) return -2;
    if (ldz < std::max<int64_t>(1, m)) return -5;
    if (n < 0 || (!cols_host && n > m)) return -6;
    if (ldx < std::max<int64_t>(1, m)) return -9;
    if (m == 0 || n == 0) return 0;
    if (!Q) return -1;
    if (!Z) return -4;
    if (!X) return -8;
    if (cols_host)
        for (int64_t q = 0; q < n; q++)
            if (cols_host[q] < 0 || cols_host[q] >= m || (q > 0 && cols_host[q] <= cols_host[q - 1])) return -7;
    if (int rc = ensure_init()) return rc;
    CK(cudaMemset2DAsync(X, size_t(ldx) * sizeof(T), 0, size_t(m) * sizeof(T), size_t(n), g_stream));
    SumPlanes sp;                       // complex: operand sums of Q and Z for the 3M kernel
    if constexpr (S<T>::cplx_) {
        if (gemm_variant() == 0 && gemm_presum_enabled()) {
            sp.st = g_stream;
            sp.ldu = (m + 2) & ~int64_t(1);
            sp.ldx = int((m + 2) & ~int64_t(1));
            CK(cudaMallocAsync(&sp.U, size_t(sp.ldu) * m * 8, g_stream));
            CK(cudaMallocAsync(&sp.X, size_t(sp.ldx) * n * 8, g_stream));
            presum_kernel<<<int(std::min<int64_t>(cdiv(m, 8), int64_t(g_num_sms) * 16)), 256, 0, g_stream>>>(
                Q, ldq, m, sp.U, sp.ldu, 1.0, m);
            CK_LAUNCH("presum_kernel");
            presum_kernel<<<int(std::min<int64_t>(cdiv(n, 8), int64_t(g_num_sms) * 16)), 256, 0, g_stream>>>(
                Z, ldz, n, sp.X, sp.ldx, 1.0, m);
            CK_LAUNCH("presum_kernel");
        }
    }
    constexpr int64_t W = 1024;
    for (int64_t p0 = 0; p0 < n; p0 += W) {
        const int64_t p1 = std::min(n, p0 + W);
        const int64_t K = (cols_host ? cols_host[p1 - 1] : p1 - 1) + 1;
        GemmArgs<T> g{};
        g.U = Q; g.ldu = ldq; g.B = X; g.ldb = ldx;
        g.M = m; g.N = p1 - p0; g.K = int(K);
        g.a_r0 = 0; g.a_c0 = 0; g.c_r0 = 0; g.x_r0 = 0; g.col0 = p0;
        g.X = Z; g.ldx = ldz;
        g.dblk = nullptr;
        if (sp.U) { g.As = sp.U; g.ldas = sp.ldu; g.Xsum = sp.X; g.ldxs = sp.ldx; }
        if (int rc = launch_gemm<T, false>(g)) return rc;
    }
    const int blocks = int(std::min<int64_t>(cdiv(m * n, 256), int64_t(g_num_sms) * 16));
    negate_kernel<T><<<blocks, 256, 0, g_stream>>>(X, ldx, m, n);
    CK_LAUNCH("negate_kernel");
    return 0;
}

template <typename T>
int trevc_qz_impl(const T *Tm, int64_t ldt, int64_t m, const T *Q, int64_t ldq, T *X, int64_t ldx,
                  double *scales, int32_t *scale_exp, int nb) {
    if (m < 0) return -3;
    if (ldt < std::max<int64_t>(1, m)) return -2;
    if (ldq < std::max<int64_t>(1, m)) return -5;
    if (ldx < std::max<int64_t>(1, m)) return -7;
    if (nb != 0 && (nb < 1 || nb > 128)) return -10;
    if (m == 0) return 0;
    if (!Tm) return -1;
    if (!Q) return -4;
    if (!X) return -6;
    if (int rc = ensure_init()) return rc;
    T *Z = nullptr;
    CK(cudaMallocAsync(&Z, size_t(m) * m * sizeof(T), g_stream));
    int rc = trevc_impl<T>(Tm, ldt, m, nullptr, m, Z, m, scales, scale_exp, nb);
    if (rc < 0) rc = 1;                       // arguments were validated above
    if (!rc) rc = backtransform_impl<T>(Q, ldq, m, Z, m, m, nullptr, X, ldx);
    if (rc < 0) rc = 1;
    cudaFreeAsync(Z, g_stream);
    return rc;
}

// ---------------------------------------------------------------- generalized solve (Alg. 7/8)
// Per block: the generalized diagonal kernel (U' = U - lambda_j V on the fly, C = -lambda_j X(I1)),
// then the update B(I0,act) = 2^d B(I0,act) - U(I0,I1) X(I1,act) - V(I0,I1) C (P:893-896 /
// P:970-974) as two launches of the DMMA update GEMM (the second with d = 0, X = C).
template <typename T, bool SAFE>
int blocked_solve_gen(const T *U, int64_t ldu, const T *V, int64_t ldv, int64_t m, const T *shifts,
                      int64_t sstride, T *B, int64_t ldb, int64_t n, const int64_t *rowend_dev,
                      const std::vector<int64_t> *rowend_sorted_host, bool zero_c, int nb, Work &w,
                      Work &wv, T *Cbuf) {
    int64_t nblk = cdiv(m, nb);
    if (SAFE) CK(cudaMemsetAsync(w.fb_count, 0, nblk * 4, g_stream));
    for (int64_t b = 0; b < nblk; b++) {
        Blk bl = block_rows(0, m, nb, b);
        int64_t c0 = 0;
        if (rowend_sorted_host) {
            const auto &re = *rowend_sorted_host;
            c0 = std::upper_bound(re.begin(), re.end(), bl.lo) - re.begin();
        }
        int64_t ncols = n - c0;
        if (ncols <= 0) continue;
        if (zero_c) CK(cudaMemsetAsync(Cbuf + c0 * nb, 0, size_t(ncols) * nb * sizeof(T), g_stream));
        DiagArgs<T> a{};
        a.U = U; a.ldu = ldu; a.m = m; a.shifts = shifts; a.sstride = sstride;
        a.B = B; a.ldb = ldb; a.c0 = c0; a.ncols = ncols; a.n = n;
        a.rowend = rowend_dev;
        a.lo = bl.lo; a.hi = bl.hi; a.b = b;
        a.cnl = w.cnl; a.P = w.P; a.delta = w.delta;
        a.G = w.G; a.e = w.e; a.dblk = w.dblk; a.Etab = w.Etab;
        a.fb_list = w.fb_list; a.fb_count = w.fb_count + b;
        a.force_fb = g_diag_force_fb;
        a.V = V; a.ldv = ldv; a.cnlV = wv.cnl; a.PV = wv.P; a.deltaV = wv.delta;
        a.Cbuf = Cbuf; a.ldc = nb;
        if (int rc = launch_diag_gen<T, SAFE>(a, nb)) return rc;
        const int64_t M = bl.lo;
        if (M <= 0) continue;
        GemmArgs<T> g{};
        g.U = U; g.ldu = ldu; g.B = B; g.ldb = ldb;
        g.M = M; g.N = ncols; g.K = int(bl.hi - bl.lo);
        g.a_r0 = 0; g.a_c0 = bl.lo; g.c_r0 = 0;
        g.x_r0 = bl.lo; g.col0 = c0;
        g.X = B; g.ldx = ldb;
        g.dblk = SAFE ? w.dblk : nullptr;
        if (int rc = launch_gemm<T, false>(g)) return rc;               // - U(I0,I1) X(I1)
        GemmArgs<T> g2 = g;
        g2.U = V; g2.ldu = ldv; g2.X = Cbuf; g2.ldx = nb; g2.x_r0 = 0; g2.dblk = nullptr;
        if (int rc = launch_gemm<T, false>(g2)) return rc;              // - V(I0,I1) C, C = -lambda X
    }
    return 0;
}

template <typename T>
int mstrsm_gen_impl(int safe, const T *U, int64_t ldu, const T *V, int64_t ldv, int64_t m, const T *shifts,
                    int64_t sstride, T *B, int64_t ldb, int64_t n, const int64_t *row_end,
                    double *scales, int32_t *scale_exp, int nb) {
    if (safe != 0 && safe != 1) return -1;
    if (m < 0) return -6;
    if (ldu < std::max<int64_t>(1, m)) return -3;
    if (ldv < std::max<int64_t>(1, m)) return -5;
    if (sstride < 0) return -8;
    if (ldb < std::max<int64_t>(1, m)) return -10;
    if (n < 0) return -11;
    if (nb == 0) nb = 64;
    if (nb < 1 || nb > 64) return -15;
    if (m == 0 || n == 0) return 0;
    if (!U) return -2;
    if (!V) return -4;
    if (!shifts) return -7;
    if (!B) return -9;
    if (safe && !scales) return -13;
    if (int rc = ensure_init()) return rc;
    Work w, wv;
    if (int rc = alloc_work<T>(w, m, n, nb, row_end != nullptr, false)) return rc;
    if (int rc = alloc_work<T>(wv, m, 1, nb, false, false)) return rc;
    std::vector<int64_t> re_host;
    bool sorted = false;
    if (row_end)
        if (int rc = load_row_end(row_end, n, m, w.rowend, re_host, sorted)) return rc;
    T *Cbuf = nullptr;
    CK(cudaMallocAsync(&Cbuf, size_t(nb) * n * sizeof(T), g_stream));
    int blocks = int(std::min<int64_t>(cdiv(n, 8), int64_t(g_num_sms) * 16));
    int rc = 0;
    if (safe) {
        if ((rc = norm_pass<T>(0, U, ldu, m, nb, w)) == 0) rc = norm_pass<T>(0, V, ldv, m, nb, wv);
        if (!rc) {
            init_rhs_kernel<T><<<blocks, 256, 0, g_stream>>>(B, ldb, m, n, w.rowend, shifts, sstride, w.G, w.e, g_flag);
            CK_LAUNCH("init_rhs_kernel");
            rc = blocked_solve_gen<T, true>(U, ldu, V, ldv, m, shifts, sstride, B, ldb, n, w.rowend,
                                            sorted ? &re_host : nullptr, row_end && !sorted, nb, w, wv, Cbuf);
        }
    } else {
        if (w.rowend) {
            init_rhs_kernel<T><<<blocks, 256, 0, g_stream>>>(B, ldb, m, n, w.rowend, nullptr, 0, nullptr, nullptr, nullptr);
            CK_LAUNCH("init_rhs_kernel");
        }
        rc = blocked_solve_gen<T, false>(U, ldu, V, ldv, m, shifts, sstride, B, ldb, n, w.rowend,
                                         sorted ? &re_host : nullptr, row_end && !sorted, nb, w, wv, Cbuf);
    }
    if (!rc && (scales || scale_exp || safe))
        rc = finalize<T>(0, safe, B, ldb, m, n, nb, w.rowend, scales, scale_exp, nullptr, w);
    cudaFreeAsync(Cbuf, g_stream);
    return rc;
}

// GeneralizedTriangEig, Alg. 9 first function with the P:503-508 shortcut.
template <typename T>
int tgevc_impl(const T *Tm, int64_t ldt, const T *Sm, int64_t lds, int64_t m, T *Z, int64_t ldz,
               T *lambda, double *scales, int32_t *scale_exp, int nb) {
    if (m < 0) return -5;
    if (ldt < std::max<int64_t>(1, m)) return -2;
    if (lds < std::max<int64_t>(1, m)) return -4;
    if (ldz < std::max<int64_t>(1, m)) return -7;
    if (nb == 0) nb = 64;
    if (nb < 1 || nb > 64) return -11;
    if (m == 0) return 0;
    if (!Tm) return -1;
    if (!Sm) return -3;
    if (!Z) return -6;
    if (int rc = ensure_init()) return rc;
    Work w, wv;
    if (int rc = alloc_work<T>(w, m, m, nb, true, true)) return rc;
    if (int rc = alloc_work<T>(wv, m, 1, nb, false, false)) return rc;
    T *lam = static_cast<T *>(w.shifts);
    T *Cbuf = nullptr;
    CK(cudaMallocAsync(&Cbuf, size_t(nb) * m * sizeof(T), g_stream));
    int rc = norm_pass<T>(0, Tm, ldt, m, nb, w);
    if (!rc) rc = norm_pass<T>(0, Sm, lds, m, nb, wv);
    if (!rc) {
        int blocks = int(std::min<int64_t>(cdiv(m, 8), int64_t(g_num_sms) * 16));
        init_tgevc_kernel<T><<<blocks, 256, 0, g_stream>>>(Tm, ldt, Sm, lds, m, Z, ldz, lam, w.rowend, w.G,
                                                            w.e, g_flag);
        CK_LAUNCH("init_tgevc_kernel");
        std::vector<int64_t> cols(m);
        for (int64_t k = 0; k < m; k++) cols[k] = k;
        rc = blocked_solve_gen<T, true>(Tm, ldt, Sm, lds, m, lam, 1, Z, ldz, m, w.rowend, &cols, false, nb,
                                        w, wv, Cbuf);
    }
    if (!rc) rc = finalize<T>(0, 1, Z, ldz, m, m, nb, w.rowend, scales, scale_exp, w.rowend, w);
    if (!rc && lambda) CK(cudaMemcpyAsync(lambda, lam, m * sizeof(T), cudaMemcpyDeviceToDevice, g_stream));
    cudaFreeAsync(Cbuf, g_stream);
    return rc;
}

// ---------------------------------------------------------------- pseudospectra driver (a.7)
// Alg. VL batched over all points.  tol > 0: SpectralCloud deflation
// (R33) -- after every step the points whose Ritz value settled leave the batch and the remaining
// columns are compacted (stable), so later solves run on fewer shifts; per-point results are
// unchanged by the compaction (columns are independent).
int spectral_cloud_impl(const cplx *U, int64_t ldu, int64_t m, const cplx *z, int64_t npts, int iters,
                        double tol, const cplx *v0, double *sigma, int32_t *flags, int32_t *its, int nb) {
    if (m < 0) return -3;
    if (ldu < std::max<int64_t>(1, m)) return -2;
    if (npts < 0) return -5;
    if (iters < 1) return -6;
    if (!(tol >= 0.0)) return -7;
    if (nb == 0) nb = 64;
    if (nb < 1 || nb > 128) return -12;
    if (m == 0 || npts == 0) return 0;
    if (!U) return -1;
    if (!z) return -4;
    if (!v0) return -8;
    if (!sigma) return -9;
    if (int rc = ensure_init()) return rc;
    Work wN, wC;
    if (int rc = alloc_work<cplx>(wN, m, npts, nb, false, false)) return rc;
    if (int rc = alloc_work<cplx>(wC, m, npts, nb, false, false)) return rc;
    if (int rc = norm_pass<cplx>(0, U, ldu, m, nb, wN)) return rc;
    if (int rc = norm_pass<cplx>(1, U, ldu, m, nb, wC)) return rc;
    SumPlanes spN, spC;
    if (int rc = make_sum_planes<cplx>(spN, 0, U, ldu, m, npts, nb)) return rc;
    if (int rc = make_sum_planes<cplx>(spC, 1, U, ldu, m, npts, nb)) return rc;
    size_t vec = size_t(m) * npts * sizeof(cplx);
    size_t small = size_t(npts) * 8;
    size_t total = 4 * vec + 2 * size_t(iters) * small + 16 * small + 4096;
    char *buf = nullptr;
    CK(cudaMallocAsync(&buf, total, g_stream));
    size_t off = 0;
    auto take = [&](size_t bytes) { char *p = buf + off; off += (bytes + 255) & ~size_t(255); return p; };
    LanczosState st;
    st.V = (cplx *)take(vec); st.Vp = (cplx *)take(vec); st.W = (cplx *)take(vec); st.Y = (cplx *)take(vec);
    st.alpha = (double *)take(iters * small); st.beta = (double *)take(iters * small);
    st.kdone = (int *)take(npts * 4); st.active = (int *)take(npts * 4);
    st.flags = flags ? (int *)flags : (int *)take(npts * 4);
    st.amax = (double *)take(small); st.beta_prev = (double *)take(small); st.sigma = sigma;
    st.theta_prev = (double *)take(small);
    int *e1 = (int *)take(npts * 4), *e2 = (int *)take(npts * 4);
    st.e1 = e1; st.e2 = e2;
    int *pid = (int *)take(npts * 4), *pid2 = (int *)take(npts * 4), *src = (int *)take(npts * 4);
    int *count = (int *)take(64);
    cplx *zc = (cplx *)take(npts * 16), *zc2 = (cplx *)take(npts * 16);
    st.pid = pid; st.npts = npts; st.tol = tol;
    int blocks = int(std::min<int64_t>(cdiv(npts, 8), int64_t(g_num_sms) * 16));
    if (blocks < 1) blocks = 1;
    const int pblocks = int(cdiv(npts, 256));
    lanczos_init_kernel<<<blocks, 256, 0, g_stream>>>(v0, st, m, npts);
    CK_LAUNCH("lanczos_init_kernel");
    iota_kernel<<<pblocks, 256, 0, g_stream>>>(pid, npts);
    CK_LAUNCH("iota_kernel");
    CK(cudaMemcpyAsync(zc, z, npts * 16, cudaMemcpyDeviceToDevice, g_stream));
    int64_t nact = npts;
    int rc = 0;
    for (int it = 0; it < iters && !rc && nact > 0; it++) {
        const int ab = int(std::min<int64_t>(cdiv(nact, 8), int64_t(g_num_sms) * 16));
        CK(launch_k_lvl(2, copy_init_rhs_kernel, dim3(ab), dim3(256), 0, g_stream, (const cplx *)st.V, st.Y, m, nact,
                    (const cplx *)zc, wN.G, wN.e, g_flag));
        CK_LAUNCH("copy_init_rhs_kernel");
        rc = blocked_solve<cplx, true>(0, U, ldu, m, zc, 1, st.Y, m, nact, nullptr, nullptr, nb, wN, spN.U, spN.X, spN.ldu, spN.ldx);
        if (!rc) rc = finalize<cplx>(0, 1, st.Y, m, m, nact, nb, nullptr, nullptr, e1, nullptr, wN);
        if (rc) break;
        CK(launch_k_lvl(2, copy_init_rhs_kernel, dim3(ab), dim3(256), 0, g_stream, (const cplx *)st.Y, st.W, m, nact,
                    (const cplx *)nullptr, wC.G, wC.e, (int *)nullptr));
        CK_LAUNCH("copy_init_rhs_kernel");
        rc = blocked_solve<cplx, true>(1, U, ldu, m, zc, 1, st.W, m, nact, nullptr, nullptr, nb, wC, spC.U, spC.X, spC.ldu, spC.ldx);
        if (!rc) rc = finalize<cplx>(1, 1, st.W, m, m, nact, nb, nullptr, nullptr, e2, nullptr, wC);
        if (rc) break;
        if (m <= int64_t(kLsThreads) * kLsR) {    // vectors in registers: one pass over memory
            const int sb = int(std::min<int64_t>(nact, int64_t(g_num_sms) * 16));
            CK(launch_k_lvl(2, lanczos_step_reg_kernel, dim3(sb), dim3(kLsThreads), 0, g_stream, st, m, nact, it, iters));
            CK_LAUNCH("lanczos_step_reg_kernel");
        } else {
            CK(launch_k_lvl(2, lanczos_step_kernel, dim3(ab), dim3(256), 0, g_stream, st, m, nact, it, iters));
            CK_LAUNCH("lanczos_step_kernel");
        }
        if (it + 1 < iters) {           // the step left v_next in W: rotate (V, V_prev, W) <- (W, V, V_prev)
            cplx *t = st.Vp;
            st.Vp = st.V;
            st.V = st.W;
            st.W = t;
        }
        if (tol > 0.0 && it + 1 < iters) {
            converge_kernel<<<int(cdiv(nact, 128)), 128, 0, g_stream>>>(st, nact);
            CK_LAUNCH("converge_kernel");
            compact_slots_kernel<<<1, 1024, 0, g_stream>>>(pid, st.active, nact, pid2, src, count);
            CK_LAUNCH("compact_slots_kernel");
            int nnew = 0;
            CK(cudaMemcpyAsync(&nnew, count, 4, cudaMemcpyDeviceToHost, g_stream));
            CK(cudaStreamSynchronize(g_stream));
            if (nnew < nact) {          // V -> Y, Vp -> W (scratch until the next step), then swap
                const int gb = int(std::min<int64_t>(cdiv(std::max(nnew, 1), 8), int64_t(g_num_sms) * 16));
                if (nnew > 0) {
                    gather_cols_kernel<<<gb, 256, 0, g_stream>>>(st.V, st.Y, src, m, nnew);
                    CK_LAUNCH("gather_cols_kernel");
                    gather_cols_kernel<<<gb, 256, 0, g_stream>>>(st.Vp, st.W, src, m, nnew);
                    CK_LAUNCH("gather_cols_kernel");
                    gather_z_kernel<<<int(cdiv(nnew, 256)), 256, 0, g_stream>>>(z, pid2, zc2, nnew);
                    CK_LAUNCH("gather_z_kernel");
                }
                std::swap(st.V, st.Y);
                std::swap(st.Vp, st.W);
                std::swap(pid, pid2);
                std::swap(zc, zc2);
                st.pid = pid;
                nact = nnew;
            }
        } else if (tol > 0.0) {
            converge_kernel<<<int(cdiv(nact, 128)), 128, 0, g_stream>>>(st, nact);
            CK_LAUNCH("converge_kernel");
        }
    }
    if (!rc) {
        bisect_sigma_kernel<<<int(cdiv(npts, 128)), 128, 0, g_stream>>>(st, npts);
        CK_LAUNCH("bisect_sigma_kernel");
        cloud_finish_kernel<<<pblocks, 256, 0, g_stream>>>(st, npts, its);
        CK_LAUNCH("cloud_finish_kernel");
    }
    cudaFreeAsync(buf, g_stream);
    return rc;
}

int pseudospectra_impl(const cplx *U, int64_t ldu, int64_t m, const cplx *z, int64_t npts, int iters,
                       const cplx *v0, double *sigma, int32_t *flags, int nb) {
    int rc = spectral_cloud_impl(U, ldu, m, z, npts, iters, 0.0, v0, sigma, flags, nullptr, nb);
    if (rc < 0) rc = rc == -12 ? -10 : (rc == -7 ? -6 : (rc <= -8 ? rc + 1 : rc));   // pseudospectra_z positions
    return rc;
}

// SpectralWindow grid (R15, as numpy.linspace): x_i = i * step + x0 (no FMA), last point = x1
__global__ void window_grid_kernel(double x0, double x1, int64_t nx, double y0, double y1, int64_t ny, cplx *z) {
    int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= nx * ny) return;
    const int64_t ix = q % nx, iy = q / nx;
    auto lin = [](double a, double b, int64_t n, int64_t i) {
        if (n > 1 && i == n - 1) return b;
        const double step = n > 1 ? (b - a) / double(n - 1) : 0.0;
        return __dadd_rn(__dmul_rn(double(i), step), a);
    };
    z[q] = make_double2(lin(x0, x1, nx, ix), lin(y0, y1, ny, iy));
}

int spectral_window_impl(const cplx *U, int64_t ldu, int64_t m, double x0, double x1, int64_t nx, double y0,
                         double y1, int64_t ny, int iters, double tol, const cplx *v0, double *sigma,
                         int32_t *flags, int32_t *its, int nb) {
    if (nx < 0) return -6;
    if (ny < 0) return -9;
    if (!(std::isfinite(x0) && std::isfinite(x1))) return -4;
    if (!(std::isfinite(y0) && std::isfinite(y1))) return -7;
    if (m == 0 || nx == 0 || ny == 0) return m < 0 ? -3 : 0;
    if (int rc = ensure_init()) return rc;
    const int64_t npts = nx * ny;
    cplx *z = nullptr;
    CK(cudaMallocAsync(&z, npts * 16, g_stream));
    window_grid_kernel<<<int(cdiv(npts, 256)), 256, 0, g_stream>>>(x0, x1, nx, y0, y1, ny, z);
    CK_LAUNCH("window_grid_kernel");
    int rc = spectral_cloud_impl(U, ldu, m, z, npts, iters, tol, v0, sigma, flags, its, nb);
    if (rc < 0) {                                 // map spectral_cloud positions to spectral_window's
        const int map[13] = {0, -1, -2, -3, -4, -5, -10, -11, -12, -13, -14, -15, -16};
        rc = -rc < 13 ? map[-rc] : rc;
    }
    cudaFreeAsync(z, g_stream);
    return rc;
}

// SpectralPortrait window (R34): bounding box of diag(U) padded by 0.25 max(width, height,
// 1e-2 ||U||_inf) (||U||_inf as R4: max row sum of |U(i,k)|, k >= i).  Host synchronising.
int portrait_window(const cplx *U, int64_t ldu, int64_t m, double win[4]) {
    std::vector<cplx> d(m);
    CK(cudaMemcpy2DAsync(d.data(), sizeof(cplx), U, size_t(ldu + 1) * sizeof(cplx), sizeof(cplx), size_t(m),
                         cudaMemcpyDeviceToHost, g_stream));
    const int64_t nchunks = cdiv(m, kRowsumChunk);
    double *part = nullptr, *rs = nullptr;
    CK(cudaMallocAsync(&part, size_t(nchunks) * m * 8, g_stream));
    CK(cudaMallocAsync(&rs, size_t(m) * 8, g_stream));
    rowsum_n_kernel<cplx><<<dim3(unsigned(cdiv(m, 128)), unsigned(nchunks)), 128, 0, g_stream>>>(U, ldu, m, part);
    CK_LAUNCH("rowsum_n_kernel");
    rowsum_reduce_kernel<<<int(cdiv(m, 256)), 256, 0, g_stream>>>(m, nchunks, part, rs);
    CK_LAUNCH("rowsum_reduce_kernel");
    std::vector<double> rsh(m);
    CK(cudaMemcpyAsync(rsh.data(), rs, size_t(m) * 8, cudaMemcpyDeviceToHost, g_stream));
    CK(cudaStreamSynchronize(g_stream));
    cudaFreeAsync(part, g_stream);
    cudaFreeAsync(rs, g_stream);
    double xa = d[0].x, xb = d[0].x, ya = d[0].y, yb = d[0].y, un = 0.0;
    for (int64_t i = 0; i < m; i++) {
        xa = std::min(xa, d[i].x); xb = std::max(xb, d[i].x);
        ya = std::min(ya, d[i].y); yb = std::max(yb, d[i].y);
        un = std::max(un, rsh[i]);
    }
    const double pad = 0.25 * std::max(std::max(xb - xa, yb - ya), 1e-2 * un);
    win[0] = xa - pad; win[1] = xb + pad; win[2] = ya - pad; win[3] = yb + pad;
    return 0;
}

}  // namespace

// ============================================================================ C ABI
// Map an invalid-argument position of mstrsm_*_ex to the short prototypes
// (U, ldu, m, shifts, B, ldb, n, scales, nb).
static int short_pos(int rc) {
    if (rc >= 0) return rc;
    switch (-rc) {
        case 3: return -1; case 4: return -2; case 5: return -3; case 6: return -4; case 8: return -5;
        case 9: return -6; case 10: return -7; case 12: return -8; case 14: return -9; default: return rc;
    }
}

template <typename T>
int ex_ws_impl(int safe, int op, const T *U, int64_t ldu, int64_t m, const T *shifts, int64_t sstride, T *B,
               int64_t ldb, int64_t n, const int64_t *row_end, double *scales, int32_t *scale_exp, int nb,
               void *workspace, size_t workspace_bytes) {
    if (!workspace)                                  // NULL: the library allocates (as mstrsm_*_ex)
        return mstrsm_ex_impl<T>(safe, op, U, ldu, m, shifts, sstride, B, ldb, n, row_end, scales,
                                 scale_exp, nb);
    if (reinterpret_cast<uintptr_t>(workspace) % 256) return -15;
    g_arena.base = static_cast<char *>(workspace);
    g_arena.size = workspace_bytes;
    g_arena.off = 0;
    g_arena.active = true;
    int rc = mstrsm_ex_impl<T>(safe, op, U, ldu, m, shifts, sstride, B, ldb, n, row_end, scales, scale_exp, nb);
    g_arena.active = false;
    if (rc == 1 && last_cuda_error() == cudaErrorMemoryAllocation) rc = -16;   // workspace too small
    return rc;
}

// mstrsm_set_sync_status(1): the calls that can see a non-finite input synchronise the caller's
// stream before returning and report code 2 themselves (the flag is then cleared, as mstrsm_status
// does).  Per calling thread; off by default (the calls stay asynchronous).
static thread_local bool t_sync_status = false;
static int sync_status(int rc) {
    if (rc != 0 || !t_sync_status) return rc;
    CK(cudaStreamSynchronize(g_stream));
    int h = 0;
    CK(cudaMemcpy(&h, g_flag, sizeof(int), cudaMemcpyDeviceToHost));
    if (h) CK(cudaMemset(g_flag, 0, sizeof(int)));
    return h ? 2 : 0;
}

extern "C" {

int mstrsm_d(const double *U, int64_t ldu, int64_t m, const double *shifts, double *B, int64_t ldb,
             int64_t n, double *scales, int nb) {
    return short_pos(mstrsm_ex_impl<double>(0, 0, U, ldu, m, shifts, 1, B, ldb, n, nullptr, scales, nullptr, nb));
}
int mstrsm_z(const mstrsm_dcomplex *U, int64_t ldu, int64_t m, const mstrsm_dcomplex *shifts, mstrsm_dcomplex *B,
             int64_t ldb, int64_t n, double *scales, int nb) {
    return short_pos(mstrsm_ex_impl<cplx>(0, 0, (const cplx *)U, ldu, m, (const cplx *)shifts, 1, (cplx *)B, ldb, n,
                                nullptr, scales, nullptr, nb));
}
int mstrsm_d_safe(const double *U, int64_t ldu, int64_t m, const double *shifts, double *B,
                  int64_t ldb, int64_t n, double *scales, int nb) {
    return sync_status(short_pos(mstrsm_ex_impl<double>(1, 0, U, ldu, m, shifts, 1, B, ldb, n, nullptr, scales, nullptr, nb)));
}
int mstrsm_z_safe(const mstrsm_dcomplex *U, int64_t ldu, int64_t m, const mstrsm_dcomplex *shifts, mstrsm_dcomplex *B,
                  int64_t ldb, int64_t n, double *scales, int nb) {
    return sync_status(short_pos(mstrsm_ex_impl<cplx>(1, 0, (const cplx *)U, ldu, m, (const cplx *)shifts, 1, (cplx *)B, ldb, n,
                                nullptr, scales, nullptr, nb)));
}
int mstrsm_d_ex(int safe, mstrsm_op op, const double *U, int64_t ldu, int64_t m, const double *shifts,
                int64_t shift_stride, double *B, int64_t ldb, int64_t n, const int64_t *row_end,
                double *scales, int32_t *scale_exp, int nb) {
    return sync_status(mstrsm_ex_impl<double>(safe, int(op), U, ldu, m, shifts, shift_stride, B, ldb, n, row_end,
                                  scales, scale_exp, nb));
}
int mstrsm_z_ex(int safe, mstrsm_op op, const mstrsm_dcomplex *U, int64_t ldu, int64_t m, const mstrsm_dcomplex *shifts,
                int64_t shift_stride, mstrsm_dcomplex *B, int64_t ldb, int64_t n, const int64_t *row_end,
                double *scales, int32_t *scale_exp, int nb) {
    return sync_status(mstrsm_ex_impl<cplx>(safe, int(op), (const cplx *)U, ldu, m, (const cplx *)shifts, shift_stride,
                                (cplx *)B, ldb, n, row_end, scales, scale_exp, nb));
}

size_t mstrsm_workspace_size(int64_t m, int64_t n, int nb, int is_complex, int safe) {
    if (m <= 0 || n <= 0) return 0;
    if (nb == 0) nb = 64;
    if (nb < 1 || nb > 128) return 0;
    Work w;
    size_t work = 0;
    if (is_complex) alloc_work<cplx>(w, m, n, nb, true, false, &work);
    else alloc_work<double>(w, m, n, nb, true, false, &work);
    size_t total = work + 256;
    if (safe) total += size_t(cdiv(m, kRowsumChunk)) * m * 8 + 256;              // norm pass partials
    if (is_complex && gemm_variant() == 0 && gemm_presum_enabled())            // 3M operand-sum planes
        total += size_t((m + 2) & ~int64_t(1)) * m * 8 + 4 * size_t((nb + 1) & ~1) * n * 8 + 768;
    return total;
}

int mstrsm_d_ex_ws(int safe, mstrsm_op op, const double *U, int64_t ldu, int64_t m, const double *shifts,
                   int64_t shift_stride, double *B, int64_t ldb, int64_t n, const int64_t *row_end,
                   double *scales, int32_t *scale_exp, int nb, void *workspace, size_t workspace_bytes) {
    return sync_status(ex_ws_impl<double>(safe, int(op), U, ldu, m, shifts, shift_stride, B, ldb, n, row_end, scales,
                              scale_exp, nb, workspace, workspace_bytes));
}
int mstrsm_z_ex_ws(int safe, mstrsm_op op, const mstrsm_dcomplex *U, int64_t ldu, int64_t m,
                   const mstrsm_dcomplex *shifts, int64_t shift_stride, mstrsm_dcomplex *B, int64_t ldb, int64_t n,
                   const int64_t *row_end, double *scales, int32_t *scale_exp, int nb, void *workspace,
                   size_t workspace_bytes) {
    return sync_status(ex_ws_impl<cplx>(safe, int(op), (const cplx *)U, ldu, m, (const cplx *)shifts, shift_stride, (cplx *)B,
                            ldb, n, row_end, scales, scale_exp, nb, workspace, workspace_bytes));
}

int trevc_d(const double *T, int64_t ldt, int64_t m, double *Z, int64_t ldz, double *scales,
            int32_t *scale_exp, int nb) {
    int rc = trevc_impl<double>(T, ldt, m, nullptr, m, Z, ldz, scales, scale_exp, nb);
    return rc < 0 ? (rc == -4 ? -1 : (rc <= -6 ? rc + 2 : rc)) : sync_status(rc);
}
int trevc_z(const mstrsm_dcomplex *T, int64_t ldt, int64_t m, mstrsm_dcomplex *Z, int64_t ldz, double *scales,
            int32_t *scale_exp, int nb) {
    int rc = trevc_impl<cplx>((const cplx *)T, ldt, m, nullptr, m, (cplx *)Z, ldz, scales, scale_exp, nb);
    return rc < 0 ? (rc == -4 ? -1 : (rc <= -6 ? rc + 2 : rc)) : sync_status(rc);
}
int trevc_d_cols(const double *T, int64_t ldt, int64_t m, const int64_t *cols_host, int64_t ncols,
                 double *Z, int64_t ldz, double *scales, int32_t *scale_exp, int nb) {
    return sync_status(trevc_impl<double>(T, ldt, m, cols_host, ncols, Z, ldz, scales, scale_exp, nb));
}
int trevc_z_cols(const mstrsm_dcomplex *T, int64_t ldt, int64_t m, const int64_t *cols_host, int64_t ncols,
                 mstrsm_dcomplex *Z, int64_t ldz, double *scales, int32_t *scale_exp, int nb) {
    return sync_status(trevc_impl<cplx>((const cplx *)T, ldt, m, cols_host, ncols, (cplx *)Z, ldz, scales, scale_exp, nb));
}

int spectral_cloud_z(const mstrsm_dcomplex *U, int64_t ldu, int64_t m, const mstrsm_dcomplex *z, int64_t npts,
                     int maxit, double tol, const mstrsm_dcomplex *v0, double *sigma, int32_t *flags, int32_t *its,
                     int nb) {
    return spectral_cloud_impl((const cplx *)U, ldu, m, (const cplx *)z, npts, maxit, tol, (const cplx *)v0, sigma,
                               flags, its, nb);
}
int spectral_window_z(const mstrsm_dcomplex *U, int64_t ldu, int64_t m, double x0, double x1, int64_t nx, double y0,
                      double y1, int64_t ny, int maxit, double tol, const mstrsm_dcomplex *v0, double *sigma,
                      int32_t *flags, int32_t *its, int nb) {
    return spectral_window_impl((const cplx *)U, ldu, m, x0, x1, nx, y0, y1, ny, maxit, tol, (const cplx *)v0, sigma,
                                flags, its, nb);
}
int spectral_portrait_z(const mstrsm_dcomplex *U, int64_t ldu, int64_t m, int64_t nx, int64_t ny, int maxit,
                        double tol, const mstrsm_dcomplex *v0, double *sigma, int32_t *flags, int32_t *its,
                        double *window_host, int nb) {
    if (m < 0) return -3;
    if (ldu < std::max<int64_t>(1, m)) return -2;
    if (nx < 0) return -4;
    if (ny < 0) return -5;
    if (m == 0 || nx == 0 || ny == 0) return 0;
    if (!U) return -1;
    if (int rc = ensure_init()) return rc;
    double win[4];
    if (int rc = portrait_window((const cplx *)U, ldu, m, win)) return rc;
    if (window_host) for (int i = 0; i < 4; i++) window_host[i] = win[i];
    int rc = spectral_window_impl((const cplx *)U, ldu, m, win[0], win[1], nx, win[2], win[3], ny, maxit, tol,
                                  (const cplx *)v0, sigma, flags, its, nb);
    if (rc < 0) {                                 // positions of spectral_portrait_z
        const int map[17] = {0, -1, -2, -3, 1, 1, -4, 1, 1, -5, -6, -7, -8, -9, -10, -11, -13};
        rc = -rc < 17 ? map[-rc] : rc;
    }
    return rc;
}

int mstrsm_d_side(int safe, mstrsm_side side, mstrsm_uplo uplo, const double *A, int64_t lda, int64_t m,
                  const double *shifts, int64_t shift_stride, double *B, int64_t ldb, int64_t n, double *scales,
                  int32_t *scale_exp, int nb) {
    return sync_status(side_impl<double>(safe, int(side), int(uplo), A, lda, m, shifts, shift_stride, B, ldb, n, scales,
                             scale_exp, nb));
}
int mstrsm_z_side(int safe, mstrsm_side side, mstrsm_uplo uplo, const mstrsm_dcomplex *A, int64_t lda, int64_t m,
                  const mstrsm_dcomplex *shifts, int64_t shift_stride, mstrsm_dcomplex *B, int64_t ldb, int64_t n,
                  double *scales, int32_t *scale_exp, int nb) {
    return sync_status(side_impl<cplx>(safe, int(side), int(uplo), (const cplx *)A, lda, m, (const cplx *)shifts, shift_stride,
                           (cplx *)B, ldb, n, scales, scale_exp, nb));
}

int eig_backtransform_d(const double *Q, int64_t ldq, int64_t m, const double *Z, int64_t ldz, int64_t n,
                        const int64_t *cols_host, double *X, int64_t ldx) {
    return backtransform_impl<double>(Q, ldq, m, Z, ldz, n, cols_host, X, ldx);
}
int eig_backtransform_z(const mstrsm_dcomplex *Q, int64_t ldq, int64_t m, const mstrsm_dcomplex *Z, int64_t ldz,
                        int64_t n, const int64_t *cols_host, mstrsm_dcomplex *X, int64_t ldx) {
    return backtransform_impl<cplx>((const cplx *)Q, ldq, m, (const cplx *)Z, ldz, n, cols_host, (cplx *)X, ldx);
}
int trevc_qz_d(const double *T, int64_t ldt, int64_t m, const double *Q, int64_t ldq, double *X, int64_t ldx,
               double *scales, int32_t *scale_exp, int nb) {
    return sync_status(trevc_qz_impl<double>(T, ldt, m, Q, ldq, X, ldx, scales, scale_exp, nb));
}
int trevc_qz_z(const mstrsm_dcomplex *T, int64_t ldt, int64_t m, const mstrsm_dcomplex *Q, int64_t ldq,
               mstrsm_dcomplex *X, int64_t ldx, double *scales, int32_t *scale_exp, int nb) {
    return sync_status(trevc_qz_impl<cplx>((const cplx *)T, ldt, m, (const cplx *)Q, ldq, (cplx *)X, ldx, scales, scale_exp, nb));
}

// Host <-> device copies of the triangles the TriangEig path reads and writes: only the upper
// triangle of T is read and only rows 0..k of eigenvector k are nonzero, so both
// directions move 128-column panels, rows 0 .. panel end (about m^2/2 elements instead of m^2).
static cudaError_t copy_upper_panels(cplx *dst, int64_t ldd, const cplx *src, int64_t lds, int64_t m,
                                     cudaMemcpyKind kind, cudaStream_t st) {
    for (int64_t c0 = 0; c0 < m; c0 += 128) {
        const int64_t c1 = std::min<int64_t>(m, c0 + 128);
        cudaError_t e = cudaMemcpy2DAsync(dst + c0 * ldd, ldd * sizeof(cplx), src + c0 * lds, lds * sizeof(cplx),
                                          size_t(c1) * sizeof(cplx), size_t(c1 - c0), kind, st);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

// Device buffers and events of the host entries; the destructor drains the copy streams (so no
// copy still reads or writes the caller's host buffers after an error return) and frees.
struct HostStage {
    cudaStream_t cs = nullptr, h2d = nullptr, d2h = nullptr;
    cplx *dT[2] = {nullptr, nullptr}, *dZ[2] = {nullptr, nullptr};
    double *ds[2] = {nullptr, nullptr};
    int *de[2] = {nullptr, nullptr};
    cudaEvent_t ev[7] = {};
    ~HostStage() {
        if (h2d) cudaStreamSynchronize(h2d);
        if (d2h) cudaStreamSynchronize(d2h);
        for (int s = 0; s < 2; s++) {
            if (dT[s]) cudaFreeAsync(dT[s], cs);
            if (dZ[s]) cudaFreeAsync(dZ[s], cs);
            if (ds[s]) cudaFreeAsync(ds[s], cs);
            if (de[s]) cudaFreeAsync(de[s], cs);
        }
        for (auto e : ev)
            if (e) cudaEventDestroy(e);
        if (cs) cudaStreamSynchronize(cs);
    }
    int alloc(int s, int64_t m) {
        const size_t bytes = size_t(m) * m * sizeof(cplx);
        CK(cudaMallocAsync(&dT[s], bytes, cs));
        CK(cudaMallocAsync(&dZ[s], bytes, cs));
        CK(cudaMallocAsync(&ds[s], m * 8, cs));
        CK(cudaMallocAsync(&de[s], m * 4, cs));
        return 0;
    }
};

int trevc_z_host(const mstrsm_dcomplex *T_host, int64_t ldt, int64_t m, mstrsm_dcomplex *Z_host, int64_t ldz,
                 double *scales_host, int32_t *scale_exp_host, int nb) {
    if (m < 0) return -3;
    if (ldt < std::max<int64_t>(1, m)) return -2;
    if (ldz < std::max<int64_t>(1, m)) return -5;
    if (m == 0) return 0;
    if (!T_host) return -1;
    if (!Z_host) return -4;
    if (int rc = ensure_init()) return rc;
    HostStage hs;
    hs.cs = g_stream;
    if (int rc = hs.alloc(0, m)) return rc;
    CK(copy_upper_panels(hs.dT[0], m, (const cplx *)T_host, ldt, m, cudaMemcpyHostToDevice, g_stream));
    int rc = trevc_impl<cplx>(hs.dT[0], m, m, nullptr, m, hs.dZ[0], m, hs.ds[0], hs.de[0], nb);
    if (rc == 0) {
        CK(copy_upper_panels((cplx *)Z_host, ldz, hs.dZ[0], m, m, cudaMemcpyDeviceToHost, g_stream));
        if (scales_host) CK(cudaMemcpyAsync(scales_host, hs.ds[0], m * 8, cudaMemcpyDeviceToHost, g_stream));
        if (scale_exp_host) CK(cudaMemcpyAsync(scale_exp_host, hs.de[0], m * 4, cudaMemcpyDeviceToHost, g_stream));
    }
    CK(cudaStreamSynchronize(g_stream));
    return rc;
}

// Batched host entry: problem k+1's H2D (copy stream 1) and problem k-1's D2H (copy stream 2)
// overlap problem k's solve (library stream), with two device buffer sets in flight.
int trevc_z_host_batch(const mstrsm_dcomplex *const *T_host, int64_t ldt, int64_t m, mstrsm_dcomplex *const *Z_host,
                       int64_t ldz, double *const *scales_host, int32_t *const *scale_exp_host, int64_t count,
                       int nb) {
    if (m < 0) return -3;
    if (ldt < std::max<int64_t>(1, m)) return -2;
    if (ldz < std::max<int64_t>(1, m)) return -5;
    if (count < 0) return -8;
    if (nb != 0 && (nb < 1 || nb > 128)) return -9;
    if (m == 0 || count == 0) return 0;
    if (!T_host) return -1;
    if (!Z_host) return -4;
    for (int64_t k = 0; k < count; k++) {
        if (!T_host[k]) return -1;
        if (!Z_host[k]) return -4;
    }
    if (int rc = ensure_init()) return rc;
    DevRes *res = dev_res();                   // this thread's copy streams on this device
    if (!res) return 1;
    HostStage hs;
    hs.cs = g_stream;
    const cudaStream_t cs = g_stream, s_h2d = res->h2d, s_d2h = res->d2h;
    for (auto &e : hs.ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    cudaEvent_t e_alloc = hs.ev[0], e_h2d[2] = {hs.ev[1], hs.ev[2]}, e_comp[2] = {hs.ev[3], hs.ev[4]},
                e_d2h[2] = {hs.ev[5], hs.ev[6]};
    for (int s = 0; s < 2 && s < count; s++)
        if (int rc = hs.alloc(s, m)) return rc;
    CK(cudaEventRecord(e_alloc, cs));
    hs.h2d = s_h2d;                            // from here on the destructor drains the copy streams
    hs.d2h = s_d2h;
    CK(cudaStreamWaitEvent(s_h2d, e_alloc, 0));
    CK(cudaStreamWaitEvent(s_d2h, e_alloc, 0));
    int rc = 0;
    for (int64_t k = 0; k < count && !rc; k++) {
        const int s = int(k & 1);
        if (k >= 2) CK(cudaStreamWaitEvent(s_h2d, e_comp[s], 0));   // dT[s] released by solve k-2
        CK(copy_upper_panels(hs.dT[s], m, (const cplx *)T_host[k], ldt, m, cudaMemcpyHostToDevice, s_h2d));
        CK(cudaEventRecord(e_h2d[s], s_h2d));
        CK(cudaStreamWaitEvent(cs, e_h2d[s], 0));
        if (k >= 2) CK(cudaStreamWaitEvent(cs, e_d2h[s], 0));         // dZ[s] read out by D2H k-2
        rc = trevc_impl<cplx>(hs.dT[s], m, m, nullptr, m, hs.dZ[s], m, hs.ds[s], hs.de[s], nb);
        if (rc < 0) rc = -9;
        if (rc) break;
        CK(cudaEventRecord(e_comp[s], cs));
        CK(cudaStreamWaitEvent(s_d2h, e_comp[s], 0));
        CK(copy_upper_panels((cplx *)Z_host[k], ldz, hs.dZ[s], m, m, cudaMemcpyDeviceToHost, s_d2h));
        if (scales_host && scales_host[k])
            CK(cudaMemcpyAsync(scales_host[k], hs.ds[s], m * 8, cudaMemcpyDeviceToHost, s_d2h));
        if (scale_exp_host && scale_exp_host[k])
            CK(cudaMemcpyAsync(scale_exp_host[k], hs.de[s], m * 4, cudaMemcpyDeviceToHost, s_d2h));
        CK(cudaEventRecord(e_d2h[s], s_d2h));
    }
    CK(cudaStreamSynchronize(s_h2d));
    CK(cudaStreamSynchronize(s_d2h));
    return rc;
}

int mstrsm_d_gen(int safe, const double *U, int64_t ldu, const double *V, int64_t ldv, int64_t m,
                 const double *shifts, int64_t shift_stride, double *B, int64_t ldb, int64_t n,
                 const int64_t *row_end, double *scales, int32_t *scale_exp, int nb) {
    return sync_status(mstrsm_gen_impl<double>(safe, U, ldu, V, ldv, m, shifts, shift_stride, B, ldb, n, row_end,
                                   scales, scale_exp, nb));
}
int mstrsm_z_gen(int safe, const mstrsm_dcomplex *U, int64_t ldu, const mstrsm_dcomplex *V, int64_t ldv,
                 int64_t m, const mstrsm_dcomplex *shifts, int64_t shift_stride, mstrsm_dcomplex *B,
                 int64_t ldb, int64_t n, const int64_t *row_end, double *scales, int32_t *scale_exp,
                 int nb) {
    return sync_status(mstrsm_gen_impl<cplx>(safe, (const cplx *)U, ldu, (const cplx *)V, ldv, m, (const cplx *)shifts,
                                 shift_stride, (cplx *)B, ldb, n, row_end, scales, scale_exp, nb));
}
int tgevc_d(const double *T, int64_t ldt, const double *S, int64_t lds, int64_t m, double *Z, int64_t ldz,
            double *lambda, double *scales, int32_t *scale_exp, int nb) {
    return sync_status(tgevc_impl<double>(T, ldt, S, lds, m, Z, ldz, lambda, scales, scale_exp, nb));
}
int tgevc_z(const mstrsm_dcomplex *T, int64_t ldt, const mstrsm_dcomplex *S, int64_t lds, int64_t m,
            mstrsm_dcomplex *Z, int64_t ldz, mstrsm_dcomplex *lambda, double *scales, int32_t *scale_exp,
            int nb) {
    return sync_status(tgevc_impl<cplx>((const cplx *)T, ldt, (const cplx *)S, lds, m, (cplx *)Z, ldz, (cplx *)lambda,
                            scales, scale_exp, nb));
}

int pseudospectra_z(const mstrsm_dcomplex *U, int64_t ldu, int64_t m, const mstrsm_dcomplex *z, int64_t npts, int iters,
                    const mstrsm_dcomplex *v0, double *sigma_min, int32_t *flags, int nb) {
    return pseudospectra_impl((const cplx *)U, ldu, m, (const cplx *)z, npts, iters, (const cplx *)v0,
                              sigma_min, flags, nb);
}

int mstrsm_set_stream(void *s) {
    g_stream = static_cast<cudaStream_t>(s);
    return 0;
}
void *mstrsm_get_stream(void) { return g_stream; }

const char *mstrsm_error_string(int code) {
    switch (code) {
        case 0: return "success";
        case 1: return g_errmsg;
        case 2: return "non-finite entry in U or the shifts";
        case 3: return "communication error";
        default: return code < 0 ? "invalid argument" : "unknown error";
    }
}

int mstrsm_status(void) {
    if (int rc = ensure_init()) return rc;
    CK(cudaStreamSynchronize(g_stream));
    int h = 0;
    CK(cudaMemcpy(&h, g_flag, sizeof(int), cudaMemcpyDeviceToHost));
    CK(cudaMemset(g_flag, 0, sizeof(int)));
    return h ? 2 : 0;
}

int mstrsm_set_sync_status(int on) {
    t_sync_status = on != 0;
    return 0;
}

int64_t mstrsm_launch_count(int reset) {
    return reset ? g_launches.exchange(0) : g_launches.load();
}

int mstrsm_gemm_real_products(void) { return mstrsm::rt::gemm_variant() == 0 ? 3 : 4; }

int mstrsm_profile(int enable) {
    for (auto &r : g_prof_recs) { g_ev_pool.push_back(r.e0); g_ev_pool.push_back(r.e1); }
    g_prof_recs.clear();
    g_prof = enable != 0;
    return 0;
}

int mstrsm_profile_read(int kind, double *total_ms, int64_t *launches, double *flops) {
    CK(cudaStreamSynchronize(g_stream));
    double t = 0.0, f = 0.0;
    int64_t c = 0;
    for (auto &r : g_prof_recs) {
        if (r.kind != kind) continue;
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, r.e0, r.e1));
        t += ms; f += r.flops; c++;
    }
    if (total_ms) *total_ms = t;
    if (launches) *launches = c;
    if (flops) *flops = f;
    return 0;
}

}  // extern "C"

// ---------------------------------------------------------------- FP64 roofline probe
__global__ void __launch_bounds__(256) dmma_peak_kernel(double *out, int iters, double seed) {
    double a = seed * (threadIdx.x + 1), b = 1.0 - seed * threadIdx.x;
    double c[8][2];
#pragma unroll
    for (int q = 0; q < 8; q++) c[q][0] = c[q][1] = 0.0;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int q = 0; q < 8; q++) dmma(c[q][0], c[q][1], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < 8; q++) s += c[q][0] + c[q][1];
    if (s == 1234.5) out[0] = s;
}

__global__ void __launch_bounds__(256) dfma_peak_kernel(double *out, int iters, double seed) {
    double a = 1.0 - seed, b = seed * threadIdx.x;
    double c[8];
#pragma unroll
    for (int q = 0; q < 8; q++) c[q] = q * seed;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int q = 0; q < 8; q++) c[q] = fma(c[q], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < 8; q++) s += c[q];
    if (s == 1234.5) out[0] = s;
}

extern "C" int mstrsm_fp64_peak(double ms, double *dmma_tflops, double *dfma_tflops) {
    if (int rc = ensure_init()) return rc;
    double *out = nullptr;
    CK(cudaMalloc(&out, 8));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const int blocks = g_num_sms * 8, threads = 256;
    for (int which = 0; which < 2; which++) {
        int iters = 1000;
        double tf = 0.0;
        for (int rep = 0; rep < 6; rep++) {
            CK(cudaEventRecord(e0, g_stream));
            if (which == 0) dmma_peak_kernel<<<blocks, threads, 0, g_stream>>>(out, iters, 1e-3);
            else dfma_peak_kernel<<<blocks, threads, 0, g_stream>>>(out, iters, 1e-3);
            CK_LAUNCH("fp64_peak_kernel");
            CK(cudaEventRecord(e1, g_stream));
            CK(cudaEventSynchronize(e1));
            float t = 0.f;
            CK(cudaEventElapsedTime(&t, e0, e1));
            double flops = which == 0 ? double(blocks) * (threads / 32) * iters * 8.0 * 512.0
                                      : double(blocks) * threads * iters * 8.0 * 2.0;
            if (rep >= 2) tf = std::max(tf, flops / (t * 1e-3) / 1e12);
            if (t > 0.f && t < ms) iters = int(std::min(1e9, iters * (ms / t)));
        }
        if (which == 0 && dmma_tflops) *dmma_tflops = tf;
        if (which == 1 && dfma_tflops) *dfma_tflops = tf;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    return 0;
}

// ---------------------------------------------------------------- triangular shard packing
// Eigenvector k is zero below row k, so a shard travels as its columns' rows 0 .. k only
// (≈ half the bytes of the m x ncols block): column q goes to out[offsets[q] .. + heights[q]).
template <typename T>
__global__ void pack_cols_kernel(const T *__restrict__ Z, int64_t ldz, int64_t n, const int64_t *__restrict__ src,
                                 const int64_t *__restrict__ heights, const int64_t *__restrict__ offsets,
                                 T *__restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t q = w; q < n; q += nw) {
        const T *z = Z + (src ? src[q] : q) * ldz;
        T *o = out + offsets[q];
        for (int64_t i = lane; i < heights[q]; i += 32) o[i] = z[i];
    }
}
template <typename T>
__global__ void unpack_cols_kernel(const T *__restrict__ in, int64_t n, const int64_t *__restrict__ heights,
                                   const int64_t *__restrict__ offsets, const int64_t *__restrict__ dst, int64_t m,
                                   T *__restrict__ Z, int64_t ldz) {
    const int lane = threadIdx.x & 31;
    const int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t q = w; q < n; q += nw) {
        const T *s = in + offsets[q];
        T *z = Z + dst[q] * ldz;
        const int64_t h = heights[q];
        for (int64_t i = lane; i < m; i += 32) z[i] = i < h ? s[i] : S<T>::zero();
    }
}
template <typename T>
int pack_cols_impl(const T *Z, int64_t ldz, int64_t n, const int64_t *src, const int64_t *heights,
                   const int64_t *offsets, T *out) {
    if (n < 0) return -3;
    if (n == 0) return 0;
    if (!Z) return -1;
    if (!heights) return -5;
    if (!offsets) return -6;
    if (!out) return -7;
    if (int rc = ensure_init()) return rc;
    const int blocks = int(std::min<int64_t>(cdiv(n, 8), int64_t(g_num_sms) * 16));
    pack_cols_kernel<T><<<blocks, 256, 0, g_stream>>>(Z, ldz, n, src, heights, offsets, out);
    CK_LAUNCH("pack_cols_kernel");
    return 0;
}
template <typename T>
int unpack_cols_impl(const T *in, int64_t n, const int64_t *heights, const int64_t *offsets, const int64_t *dst,
                     int64_t m, T *Z, int64_t ldz) {
    if (n < 0) return -2;
    if (m < 0) return -6;
    if (ldz < std::max<int64_t>(1, m)) return -8;
    if (n == 0 || m == 0) return 0;
    if (!in) return -1;
    if (!heights) return -3;
    if (!offsets) return -4;
    if (!dst) return -5;
    if (!Z) return -7;
    if (int rc = ensure_init()) return rc;
    const int blocks = int(std::min<int64_t>(cdiv(n, 8), int64_t(g_num_sms) * 16));
    unpack_cols_kernel<T><<<blocks, 256, 0, g_stream>>>(in, n, heights, offsets, dst, m, Z, ldz);
    CK_LAUNCH("unpack_cols_kernel");
    return 0;
}

extern "C" {
int mstrsm_d_pack_cols(const double *Z, int64_t ldz, int64_t n, const int64_t *src_cols, const int64_t *heights,
                       const int64_t *offsets, double *out) {
    return pack_cols_impl<double>(Z, ldz, n, src_cols, heights, offsets, out);
}
int mstrsm_z_pack_cols(const mstrsm_dcomplex *Z, int64_t ldz, int64_t n, const int64_t *src_cols,
                       const int64_t *heights, const int64_t *offsets, mstrsm_dcomplex *out) {
    return pack_cols_impl<cplx>((const cplx *)Z, ldz, n, src_cols, heights, offsets, (cplx *)out);
}
int mstrsm_d_unpack_cols(const double *in, int64_t n, const int64_t *heights, const int64_t *offsets,
                         const int64_t *dst_cols, int64_t m, double *Z, int64_t ldz) {
    return unpack_cols_impl<double>(in, n, heights, offsets, dst_cols, m, Z, ldz);
}
int mstrsm_z_unpack_cols(const mstrsm_dcomplex *in, int64_t n, const int64_t *heights, const int64_t *offsets,
                         const int64_t *dst_cols, int64_t m, mstrsm_dcomplex *Z, int64_t ldz) {
    return unpack_cols_impl<cplx>((const cplx *)in, n, heights, offsets, dst_cols, m, (cplx *)Z, ldz);
}
}  // extern "C"

// ================================================================ multi-GPU
// One process per GPU; an NCCL communicator bootstrapped by the caller (rank 0 draws the unique
// id, the caller distributes it, e.g. over its torch process group).  trevc_*_dist replicates the
// upper triangle of T from `root` (packed 128-column panels, one ncclBroadcast), solves this
// rank's serpentine block-cyclic column shard (groups of 16; trevc_*_cols), all-gathers the
// shards with their scales and exponents and unpacks them into natural order on every rank.
// Bit-identical to the single-GPU trevc_* (columns are independent).
#include <nccl.h>

namespace {
ncclComm_t g_comm = nullptr;
int g_comm_n = 0, g_comm_r = 0;
constexpr int kShardGroup = 16;

int64_t shard_of(int64_t m, int P, int r, int g, int64_t *cols) {
    int64_t n = 0;
    for (int64_t k = 0; k < m; k++) {
        const int64_t q = k / g;
        const int c = int(q % P);
        const int own = ((q / P) % 2 == 0) ? c : P - 1 - c;
        if (own == r) {
            if (cols) cols[n] = k;
            n++;
        }
    }
    return n;
}

template <typename T>
__global__ void gather_dist_kernel(const T *__restrict__ Za, int64_t m, const int64_t *__restrict__ perm,
                                   int64_t n, T *__restrict__ Z, int64_t ldz, const double *__restrict__ sa,
                                   const int *__restrict__ ea, double *__restrict__ scales, int *__restrict__ exps) {
    const int lane = threadIdx.x & 31;
    const int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t k = w; k < n; k += nw) {
        const int64_t p = perm[k];
        if (Za) {                              // (NULL: vectors unpacked elsewhere)
            const T *src = Za + p * m;
            T *dst = Z + k * ldz;
            for (int64_t i = lane; i < m; i += 32) dst[i] = src[i];
        }
        if (lane == 0) {
            if (scales) scales[k] = sa[p];
            if (exps) exps[k] = ea[p];
        }
    }
}

#define NCK(call)                                                                             \
    do {                                                                                      \
        ncclResult_t r_ = (call);                                                             \
        if (r_ != ncclSuccess) {                                                              \
            snprintf(g_errmsg, sizeof(g_errmsg), "NCCL error in %s: %s", #call, ncclGetErrorString(r_)); \
            return 3;                                                                         \
        }                                                                                     \
    } while (0)

// The upper triangle of root's T on every rank: packed by 128-column panels (rows 0 .. panel
// end), one ncclBroadcast, unpacked into a workspace copy on the other ranks.  *pack / *Tw are
// stream-ordered allocations the caller frees.
template <typename T>
int replicate_upper(const T *Tm, int64_t ldt, int64_t m, int root, T **pack_out, T **Tw_out, const T **Tuse,
                    int64_t *lduse) {
    const size_t es = sizeof(T), ndbl = es / 8;
    const int r = g_comm_r;
    size_t packed = 0;
    for (int64_t c0 = 0; c0 < m; c0 += 128) {
        const int64_t c1 = std::min<int64_t>(m, c0 + 128);
        packed += size_t(c1) * size_t(c1 - c0);
    }
    T *pack = nullptr, *Tw = nullptr;
    CK(cudaMallocAsync(&pack, packed * es, g_stream));
    *pack_out = pack;
    if (r == root) {
        size_t off = 0;
        for (int64_t c0 = 0; c0 < m; c0 += 128) {
            const int64_t c1 = std::min<int64_t>(m, c0 + 128);
            CK(cudaMemcpy2DAsync(pack + off, c1 * es, Tm + c0 * ldt, ldt * es, c1 * es, c1 - c0,
                                 cudaMemcpyDeviceToDevice, g_stream));
            off += size_t(c1) * size_t(c1 - c0);
        }
    }
    NCK(ncclBroadcast(pack, pack, packed * ndbl, ncclDouble, root, g_comm, g_stream));
    *Tuse = Tm;
    *lduse = ldt;
    if (r != root) {
        CK(cudaMallocAsync(&Tw, size_t(m) * m * es, g_stream));
        *Tw_out = Tw;
        size_t off = 0;
        for (int64_t c0 = 0; c0 < m; c0 += 128) {
            const int64_t c1 = std::min<int64_t>(m, c0 + 128);
            CK(cudaMemcpy2DAsync(Tw + c0 * m, m * es, pack + off, c1 * es, c1 * es, c1 - c0,
                                 cudaMemcpyDeviceToDevice, g_stream));
            off += size_t(c1) * size_t(c1 - c0);
        }
        *Tuse = Tw;
        *lduse = m;
    }
    return 0;
}

// Wait for the work enqueued on st, polling NCCL's asynchronous error state: a failed or hung
// peer aborts the communicator and returns 3 instead of blocking forever.
// MSTRSM_NCCL_TIMEOUT_S (default 600) bounds the wait.
int nccl_wait(cudaStream_t st, const char *what) {
    static const double timeout_s = [] {
        const char *e = getenv("MSTRSM_NCCL_TIMEOUT_S");
        const double v = e ? atof(e) : 600.0;
        return v > 0 ? v : 600.0;
    }();
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
        const cudaError_t e = cudaStreamQuery(st);
        if (e == cudaSuccess) return 0;
        if (e != cudaErrorNotReady) return set_cuda_error(e, what);
        ncclResult_t ar = ncclSuccess;
        if (g_comm) ncclCommGetAsyncError(g_comm, &ar);
        const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if ((ar != ncclSuccess && ar != ncclInProgress) || el > timeout_s) {
            snprintf(g_errmsg, sizeof(g_errmsg), "%s: %s; communicator aborted", what,
                     ar != ncclSuccess && ar != ncclInProgress ? ncclGetErrorString(ar) : "timeout");
            if (g_comm) ncclCommAbort(g_comm);
            g_comm = nullptr;
            return 3;
        }
        std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
}

// T's upper triangle from root, streamed in the order the blocks consume it: op N block b needs
// columns [lo_b, hi_b) (rows 0 .. hi_b) -- its diagonal block and the update panel U(I0, I1), and
// the per-panel prepass (P:503-508 shortcut: nothing below the diagonal travels).  On the comm
// stream cs: delta of root's T (R4: ||T||_inf needs all of T, so root computes it and sends it
// first), then, through the returned feed, one ncclBroadcast per panel, right to left (non-root:
// followed by the unpack into the workspace copy of T).  trevc_impl queues each panel's prepass
// behind it and gates block b on it, so block b computes while panels b+1.. are in flight
// (SURVEY §8e item 1).
template <typename T>
int stream_upper(const T *Tm, int64_t ldt, int64_t m, int nb, int root, cudaStream_t cs, T **pack_out,
                 double *dbuf, PanelFeed &feed) {
    const size_t es = sizeof(T), ndbl = es / 8;
    const int r = g_comm_r;
    const int64_t nblk = cdiv(m, nb);
    // One region per pair of blocks (2q, 2q+1) as blocked_solve pairs them: columns [lo_{2q+1},
    // hi_{2q}), rows 0 .. hi_{2q} (ld = hi_{2q}), so that the pair's merged update sees both panels
    // through one leading dimension; an unpaired last block has its own (ld = hi_b).  Panel b is
    // columns [lo_b, hi_b) of its region: contiguous, sent as whole columns of ld rows (rows
    // hi_b .. ld of the pair's upper panel lie below T's diagonal: never written, never read).
    const int64_t nreg = (nblk + 1) / 2;
    std::vector<size_t> roff(static_cast<size_t>(nreg) + 1, 0);
    std::vector<int64_t> rld(static_cast<size_t>(nreg), 0), rc0(static_cast<size_t>(nreg), 0);
    for (int64_t q = 0; q < nreg; q++) {
        const Blk lo_blk = block_rows(0, m, nb, 2 * q);
        const Blk hi_blk = block_rows(0, m, nb, 2 * q + 1 < nblk ? 2 * q + 1 : 2 * q);
        rld[q] = lo_blk.hi;
        rc0[q] = hi_blk.lo;
        roff[q + 1] = roff[q] + size_t(rld[q]) * size_t(lo_blk.hi - hi_blk.lo);
    }
    T *pack = nullptr;
    CK(cudaMallocAsync(&pack, roff[nreg] * es, g_stream));
    *pack_out = pack;
    // MSTRSM_DIST_TEST_UNPACK=1 (testing on one GPU): root also solves from the broadcast buffer, so
    // the non-root path runs at nranks = 1
    static const bool test_unpack = [] { const char *e = getenv("MSTRSM_DIST_TEST_UNPACK"); return e && e[0] == '1'; }();
    const bool from_pack = r != root || test_unpack;
    if (r == root) {
        double *rs = nullptr;
        CK(ws_malloc((void **)&rs, size_t(m) * 8));
        if (int rc = compute_delta_n<T>(Tm, ldt, m, rs, dbuf)) return rc;
        ws_free(rs, g_stream);
    }
    cudaEvent_t e0;
    CK(cudaEventCreateWithFlags(&e0, cudaEventDisableTiming));
    CK(cudaEventRecord(e0, g_stream));
    CK(cudaStreamWaitEvent(cs, e0, 0));
    cudaEventDestroy(e0);
    NCK(ncclBroadcast(dbuf, dbuf, 2, ncclDouble, root, g_comm, cs));
    feed.cs = cs;
    feed.delta = dbuf;
    feed.enqueue = [=](int64_t b) -> int {
        const Blk bl = block_rows(0, m, nb, b);
        const int64_t q = b / 2, ld = rld[q], w = bl.hi - bl.lo;
        T *dst = pack + roff[q] + (bl.lo - rc0[q]) * ld;
        if (r == root)
            CK(cudaMemcpy2DAsync(dst, ld * es, Tm + bl.lo * ldt, ldt * es, bl.hi * es, w, cudaMemcpyDeviceToDevice,
                                 cs));
        NCK(ncclBroadcast(dst, dst, size_t(ld) * w * ndbl, ncclDouble, root, g_comm, cs));
        return 0;
    };
    // a non-root rank solves straight from the broadcast buffer: block b sees its pair's region as
    // a column-major matrix with leading dimension ld whose column rc0 is its first (no unpack, no
    // second copy of T); a block reads only its own panel, a pair's merged update both of its panels
    if (from_pack)
        feed.view = [=](int64_t b, const void **ptr, int64_t *ld) {
            const int64_t q = b / 2;
            *ptr = static_cast<const void *>(pack + roff[q] - rc0[q] * rld[q]);
            *ld = rld[q];
        };
    return 0;
}

// Dense right-hand sides (SURVEY §8b mstrsm_z_safe_dist): U from root, every rank solves its own
// columns of B (its shard of shifts); no gather.
template <typename T>
int ex_dist_impl(int safe, int op, const T *U, int64_t ldu, int64_t m, const T *shifts, int64_t sstride, T *B,
                 int64_t ldb, int64_t n, double *scales, int32_t *scale_exp, int nb, int root) {
    if (!g_comm) {
        snprintf(g_errmsg, sizeof(g_errmsg), "mstrsm_*_dist: no communicator (mstrsm_comm_init)");
        return 3;
    }
    if (root < 0 || root >= g_comm_n) return -15;
    if (m < 0) return -5;
    if (g_comm_r == root && ldu < std::max<int64_t>(1, m)) return -4;
    if (m == 0) return 0;
    if (g_comm_r == root && !U) return -3;
    if (int rc = ensure_init()) return rc;
    T *pack = nullptr, *Tw = nullptr;
    const T *Uuse = U;
    int64_t lduse = ldu;
    int rc = replicate_upper<T>(U, ldu, m, root, &pack, &Tw, &Uuse, &lduse);
    if (!rc)      // the collective is done on every rank; an empty local shard just returns
        rc = mstrsm_ex_impl<T>(safe, op, Uuse, lduse, m, shifts, sstride, B, ldb, n, nullptr, scales, scale_exp, nb);
    if (pack) cudaFreeAsync(pack, g_stream);
    if (Tw) cudaFreeAsync(Tw, g_stream);
    if (int wrc = nccl_wait(g_stream, "mstrsm_*_dist")) return wrc;
    return rc;
}

// Receiver side of the row-block gather (a.6 applied here, as finalize_kernel does on one GPU):
// Z(l, k) = ldexp(slab value, e_k - E_b(k)) for l < k (block b of row l), Z(k, k) = c_k = 2^e_k,
// Z(l, k) = 0 for l > k; scales / exponents in natural order.  One warp per eigenvector k.
template <typename T>
__global__ void unpack_slabs_kernel(T *__restrict__ Z, int64_t ldz, int64_t m, int nb, int64_t nblk, int P,
                                    const T *__restrict__ recv, const int64_t *__restrict__ slab_off,
                                    const int64_t *__restrict__ slab_cols, const int64_t *__restrict__ c0,
                                    const int *__restrict__ owner, const int *__restrict__ qidx, int64_t mc,
                                    const int *__restrict__ Eall, const int *__restrict__ eall,
                                    double *__restrict__ scales, int *__restrict__ scale_exp) {
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t k = w; k < m; k += nw) {
        const int r = owner[k];
        const int64_t q = qidx[k];
        const int ek = eall[int64_t(r) * mc + q];
        T *z = Z + k * ldz;
        for (int64_t l = lane; l < m; l += 32) {
            T v = S<T>::zero();
            if (l < k) {
                const int64_t b = (m - 1 - l) / nb;
                const Blk bl = block_rows(0, m, nb, b);
                const int64_t nbr = bl.hi - bl.lo;
                const int64_t col = q - c0[b * P + r];
                v = recv[slab_off[b] + (int64_t(r) * slab_cols[b] + col) * nbr + (l - bl.lo)];
                const int d = ek - Eall[(int64_t(r) * nblk + b) * mc + q];
                if (d != 0) v = S<T>::ldx(v, d);
            } else if (l == k) {
                v = S<T>::real(ldexp(1.0, ek));
            }
            z[l] = v;
        }
        if (lane == 0) {
            if (scales) scales[k] = ldexp(1.0, ek);
            if (scale_exp) scale_exp[k] = ek;
        }
    }
}

template <typename T>
int trevc_dist_impl(const T *Tm, int64_t ldt, int64_t m, T *Z, int64_t ldz, double *scales, int32_t *scale_exp,
                    int nb, int root) {
    if (m < 0) return -3;
    if (ldz < std::max<int64_t>(1, m)) return -5;
    if (nb != 0 && (nb < 1 || nb > 128)) return -8;
    if (!g_comm) {
        snprintf(g_errmsg, sizeof(g_errmsg), "trevc_*_dist: no communicator (mstrsm_comm_init)");
        return 3;
    }
    // MSTRSM_DIST_EMULATE_P=P (experiments, nranks = 1 only): rank 0's step of a P-rank job on this
    // GPU -- rank 0's shard, the P-rank gather layout with the other ranks' slabs as device-to-device
    // copies of the same volume, the unpack of all m columns (tools/exp_dist_emul.py)
    static const int emul_p = [] { const char *e = getenv("MSTRSM_DIST_EMULATE_P"); return e ? atoi(e) : 0; }();
    const bool emul = g_comm_n == 1 && emul_p > 1;
    const int P = emul ? emul_p : g_comm_n, r = emul ? 0 : g_comm_r;
    if (root < 0 || root >= g_comm_n) return -9;
    if (r == root && ldt < std::max<int64_t>(1, m)) return -2;
    if (m == 0) return 0;
    if (r == root && !Tm) return -1;
    if (!Z) return -4;
    if (int rc = ensure_init()) return rc;
    const size_t es = sizeof(T), ndbl = es / 8;
    if (nb == 0) nb = 64;
    DevRes *res = dev_res();                        // this thread's comm stream on this device
    if (!res) return 1;
    const cudaStream_t cs = res->comm;              // every collective of the call runs on cs, in call order
    const int64_t nblk = cdiv(m, nb);

    // shard maps of every rank; per block b: the first active local column c0[b][q] (eigenvectors
    // k > lo_b are active), the slab width (most active columns over the ranks) and offsets
    std::vector<std::vector<int64_t>> rc_cols(P);
    int64_t mc = 1;
    for (int q = 0; q < P; q++) {
        rc_cols[q].resize(size_t(std::max<int64_t>(shard_of(m, P, q, kShardGroup, nullptr), 1)));
        rc_cols[q].resize(size_t(shard_of(m, P, q, kShardGroup, rc_cols[q].data())));
        mc = std::max<int64_t>(mc, int64_t(rc_cols[q].size()));
    }
    const std::vector<int64_t> &cols = rc_cols[r];
    const int64_t ncols = int64_t(cols.size());
    std::vector<int64_t> c0(size_t(nblk) * P), slab_cols(nblk), slab_off(nblk + 1, 0), send_off(nblk + 1, 0);
    for (int64_t b = 0; b < nblk; b++) {
        const Blk bl = block_rows(0, m, nb, b);
        int64_t wmax = 0;
        for (int q = 0; q < P; q++) {
            const auto &cq = rc_cols[q];
            const int64_t f = std::upper_bound(cq.begin(), cq.end(), bl.lo) - cq.begin();
            c0[b * P + q] = f;
            wmax = std::max<int64_t>(wmax, int64_t(cq.size()) - f);
        }
        slab_cols[b] = wmax;
        const int64_t S = wmax * (bl.hi - bl.lo);
        send_off[b + 1] = send_off[b] + S;
        slab_off[b + 1] = slab_off[b] + S * P;
    }
    std::vector<int> owner(m), qidx(m);
    for (int q = 0; q < P; q++)
        for (size_t i = 0; i < rc_cols[q].size(); i++) {
            owner[rc_cols[q][i]] = q;
            qidx[rc_cols[q][i]] = int(i);
        }

    T *pack = nullptr, *Zs = nullptr, *sendb = nullptr, *recvb = nullptr;
    double *dbuf = nullptr, *ss = nullptr;
    int *es_ = nullptr, *ea = nullptr, *Eloc = nullptr, *Eall = nullptr, *owner_d = nullptr, *qidx_d = nullptr;
    int64_t *meta = nullptr;                        // [slab_off | slab_cols | c0]
    CK(cudaMallocAsync(&dbuf, 2 * sizeof(double), g_stream));
    CK(cudaMallocAsync(&Zs, size_t(m) * std::max<int64_t>(ncols, 1) * es, g_stream));
    CK(cudaMallocAsync(&ss, size_t(mc) * 8, g_stream));
    CK(cudaMallocAsync(&es_, size_t(mc) * 4, g_stream));
    CK(cudaMallocAsync(&ea, size_t(mc) * P * 4, g_stream));
    CK(cudaMallocAsync(&Eloc, size_t(nblk) * mc * 4, g_stream));
    CK(cudaMallocAsync(&Eall, size_t(nblk) * mc * P * 4, g_stream));
    CK(cudaMallocAsync(&sendb, size_t(std::max<int64_t>(send_off[nblk], 1)) * es, g_stream));
    CK(cudaMallocAsync(&recvb, size_t(std::max<int64_t>(slab_off[nblk], 1)) * es, g_stream));
    CK(cudaMallocAsync(&owner_d, size_t(m) * 4, g_stream));
    CK(cudaMallocAsync(&qidx_d, size_t(m) * 4, g_stream));
    CK(cudaMallocAsync(&meta, size_t(2 * nblk + nblk * P) * 8, g_stream));
    CK(cudaMemsetAsync(es_, 0, size_t(mc) * 4, g_stream));
    CK(cudaMemsetAsync(Eloc, 0, size_t(nblk) * mc * 4, g_stream));
    {
        std::vector<int64_t> mh(size_t(2 * nblk + nblk * P));
        std::copy(slab_off.begin(), slab_off.begin() + nblk, mh.begin());
        std::copy(slab_cols.begin(), slab_cols.end(), mh.begin() + nblk);
        std::copy(c0.begin(), c0.end(), mh.begin() + 2 * nblk);
        CK(cudaMemcpyAsync(meta, mh.data(), mh.size() * 8, cudaMemcpyHostToDevice, g_stream));
        CK(cudaMemcpyAsync(owner_d, owner.data(), size_t(m) * 4, cudaMemcpyHostToDevice, g_stream));
        CK(cudaMemcpyAsync(qidx_d, qidx.data(), size_t(m) * 4, cudaMemcpyHostToDevice, g_stream));
        CK(cudaStreamSynchronize(g_stream));        // host arrays go out of scope
    }
    std::vector<cudaEvent_t> evs;
    struct EvGuard {
        std::vector<cudaEvent_t> &v;
        ~EvGuard() { for (auto e : v) cudaEventDestroy(e); }
    } evg{evs};
    auto new_event = [&](cudaEvent_t *e) -> int {
        CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        evs.push_back(*e);
        return 0;
    };
    auto free_all = [&]() {
        for (void *p : {(void *)pack, (void *)Zs, (void *)sendb, (void *)recvb, (void *)dbuf, (void *)ss, (void *)es_,
                        (void *)ea, (void *)Eloc, (void *)Eall, (void *)owner_d, (void *)qidx_d, (void *)meta})
            if (p) cudaFreeAsync(p, g_stream);
    };

    // 1. T streamed from root panel by panel (comm stream), overlapping the solve below
    PanelFeed feed;
    if (int rc = stream_upper<T>(Tm, ldt, m, nb, root, cs, &pack, dbuf, feed)) {
        nccl_wait(cs, "trevc_*_dist (broadcast)");
        free_all();
        return rc;
    }
    // (non-root: T is never read outside the panels; the solve's U argument is only a placeholder)
    const T *Tuse = Tm ? Tm : pack;
    const int64_t lduse = Tm ? ldt : m;
    // 2. row blocks gathered behind the compute front: once block b's diagonal
    //    step is done, rows I1_b of this rank's active columns are final up to the lazy exponent
    //    fix-up; the slab is packed and all-gathered on cs while the solve goes on
    feed.after_diag = [&](int64_t b) -> int {
        const Blk bl = block_rows(0, m, nb, b);
        const int64_t nbr = bl.hi - bl.lo, act = ncols - c0[b * P + r];
        cudaEvent_t e;
        if (int rc = new_event(&e)) return rc;
        CK(cudaEventRecord(e, g_stream));
        CK(cudaStreamWaitEvent(cs, e, 0));
        if (act > 0)
            CK(cudaMemcpy2DAsync(sendb + send_off[b], size_t(nbr) * es, Zs + bl.lo + c0[b * P + r] * m, size_t(m) * es,
                                 size_t(nbr) * es, size_t(act), cudaMemcpyDeviceToDevice, cs));
        const int64_t S = send_off[b + 1] - send_off[b];
        if (S > 0) {
            NCK(ncclAllGather(sendb + send_off[b], recvb + slab_off[b], size_t(S) * ndbl, ncclDouble, g_comm, cs));
            if (emul)   // stand-in for the other ranks' slabs (same byte volume)
                CK(cudaMemcpyAsync(recvb + slab_off[b] + S, pack, size_t(S) * (P - 1) * es,
                                   cudaMemcpyDeviceToDevice, cs));
        }
        return 0;
    };
    feed.etab_out = Eloc;
    feed.ld_etab = mc;
    // MSTRSM_DIST_EMULATE_FULL=1 (testing, with MSTRSM_DIST_EMULATE_P): every rank's shard is solved
    // here in turn and its slabs, E table and exponents land where the P-rank gathers would put
    // them, so the unpack must reproduce trevc_* bit for bit -- the P-rank layout tested on one GPU
    static const bool emul_full = [] { const char *e = getenv("MSTRSM_DIST_EMULATE_FULL"); return e && e[0] == '1'; }();
    if (emul && emul_full) {
        int rc = 0;
        std::vector<T *> zq(P, nullptr);
        for (int q = 0; q < P && !rc; q++) {
            const auto &cq = rc_cols[q];
            const int64_t nq = int64_t(cq.size());
            CK(cudaMallocAsync(&zq[q], size_t(m) * std::max<int64_t>(nq, 1) * es, g_stream));
            PanelFeed fq = feed;
            T *Zq = zq[q];
            fq.after_diag = [&, q, Zq, nq](int64_t b) -> int {
                const Blk bl = block_rows(0, m, nb, b);
                const int64_t nbr = bl.hi - bl.lo, act = nq - c0[b * P + q], S = send_off[b + 1] - send_off[b];
                cudaEvent_t e;
                if (int erc = new_event(&e)) return erc;
                CK(cudaEventRecord(e, g_stream));
                CK(cudaStreamWaitEvent(cs, e, 0));
                if (act > 0)
                    CK(cudaMemcpy2DAsync(recvb + slab_off[b] + q * S, size_t(nbr) * es, Zq + bl.lo + c0[b * P + q] * m,
                                         size_t(m) * es, size_t(nbr) * es, size_t(act), cudaMemcpyDeviceToDevice, cs));
                return 0;
            };
            fq.etab_out = Eall + int64_t(q) * nblk * mc;
            if (nq > 0) rc = trevc_impl<T>(Tuse, lduse, m, cq.data(), nq, Zq, m, ss, ea + int64_t(q) * mc, nb, &fq);
        }
        cudaEvent_t e;
        if (int erc = new_event(&e)) return erc;
        CK(cudaEventRecord(e, cs));
        CK(cudaStreamWaitEvent(g_stream, e, 0));
        if (!rc) {
            const int blocks = int(std::min<int64_t>(cdiv(m, 8), int64_t(g_num_sms) * 16));
            CK(launch_k_lvl(2, unpack_slabs_kernel<T>, dim3(blocks), dim3(256), 0, g_stream, Z, ldz, m, nb, nblk, P,
                            (const T *)recvb, (const int64_t *)meta, (const int64_t *)(meta + nblk),
                            (const int64_t *)(meta + 2 * nblk), (const int *)owner_d, (const int *)qidx_d, mc,
                            (const int *)Eall, (const int *)ea, scales, reinterpret_cast<int *>(scale_exp)));
            CK_LAUNCH("unpack_slabs_kernel");
        }
        CK(cudaStreamSynchronize(g_stream));
        for (T *z : zq)
            if (z) cudaFreeAsync(z, g_stream);
        free_all();
        return rc < 0 ? 1 : rc;
    }
    int rc = 0;
    if (ncols > 0) {
        // With P > 1 the solve's diagonal and update kernels leave k SMs (MSTRSM_DIST_RESERVE_SMS,
        // default 8) to the comm stream's work -- panel prepass, slab packing, the collectives'
        // kernels -- which cannot share an SM with the update GEMM (it holds the whole register
        // file).  One-GPU emulation of rank 0's step: P = 8 32.6 -> 30.1 ms, P = 2
        // 86.8 -> 84.9 ms.  The arithmetic does not depend on the grid size.
        static const int reserve = [] { const char *e = getenv("MSTRSM_DIST_RESERVE_SMS"); return e ? atoi(e) : 8; }();
        if (P > 1 && reserve > 0 && reserve < g_num_sms) g_cta_cap = g_num_sms - reserve;
        rc = trevc_impl<T>(Tuse, lduse, m, cols.data(), ncols, Zs, m, ss, es_, nb, &feed);
        g_cta_cap = 0;
    } else {                                        // no columns here: the collectives still run
        for (int64_t b = 0; b < nblk && !rc; b++) {
            rc = feed.enqueue(b);
            if (!rc) rc = feed.after_diag(b);
        }
    }
    if (rc < 0) rc = 1;
    // 3. status agreement (a rank that failed must not leave its peers in the final gathers), then
    //    the exponents (final e_j, the E table) -- all on cs, after the solve
    {
        cudaEvent_t e;
        if (int erc = new_event(&e)) return erc;
        CK(cudaEventRecord(e, g_stream));
        CK(cudaStreamWaitEvent(cs, e, 0));
        int *st = nullptr;
        CK(cudaMallocAsync(&st, sizeof(int), cs));
        const int rc_local = rc;
        CK(cudaMemcpyAsync(st, &rc_local, sizeof(int), cudaMemcpyHostToDevice, cs));
        NCK(ncclAllReduce(st, st, 1, ncclInt32, ncclMax, g_comm, cs));
        int rc_all = 0;
        CK(cudaMemcpyAsync(&rc_all, st, sizeof(int), cudaMemcpyDeviceToHost, cs));
        cudaFreeAsync(st, cs);
        if (int wrc = nccl_wait(cs, "trevc_*_dist (solve)")) return wrc;
        if (rc_all && !rc) {
            snprintf(g_errmsg, sizeof(g_errmsg), "trevc_*_dist: another rank failed");
            rc = 3;
        }
    }
    if (!rc) {
        NCK(ncclGroupStart());
        NCK(ncclAllGather(es_, ea, size_t(mc), ncclInt32, g_comm, cs));
        NCK(ncclAllGather(Eloc, Eall, size_t(nblk) * mc, ncclInt32, g_comm, cs));
        NCK(ncclGroupEnd());
        cudaEvent_t e;
        if (int erc = new_event(&e)) return erc;
        CK(cudaEventRecord(e, cs));
        CK(cudaStreamWaitEvent(g_stream, e, 0));
        // 4. natural order, lazy fix-up applied, zeros below the diagonal, c_k on it
        const int blocks = int(std::min<int64_t>(cdiv(m, 8), int64_t(g_num_sms) * 16));
        CK(launch_k_lvl(2, unpack_slabs_kernel<T>, dim3(blocks), dim3(256), 0, g_stream, Z, ldz, m, nb, nblk, P,
                        (const T *)recvb, (const int64_t *)meta, (const int64_t *)(meta + nblk),
                        (const int64_t *)(meta + 2 * nblk), (const int *)owner_d, (const int *)qidx_d, mc,
                        (const int *)Eall, (const int *)ea, scales, reinterpret_cast<int *>(scale_exp)));
        CK_LAUNCH("unpack_slabs_kernel");
        if (int wrc = nccl_wait(g_stream, "trevc_*_dist (gather)")) return wrc;
    }
    free_all();
    return rc;
}
}  // namespace

extern "C" {

int mstrsm_comm_unique_id(void *id_out) {
    if (!id_out) return -1;
    ncclUniqueId id;
    NCK(ncclGetUniqueId(&id));
    memcpy(id_out, &id, sizeof(id));
    return 0;
}

int mstrsm_comm_init(int nranks, int rank, const void *unique_id) {
    if (nranks < 1) return -1;
    if (rank < 0 || rank >= nranks) return -2;
    if (!unique_id) return -3;
    if (int rc = ensure_init()) return rc;
    if (g_comm) {
        ncclCommDestroy(g_comm);
        g_comm = nullptr;
    }
    ncclUniqueId id;
    memcpy(&id, unique_id, sizeof(id));
    NCK(ncclCommInitRank(&g_comm, nranks, id, rank));
    g_comm_n = nranks;
    g_comm_r = rank;
    return 0;
}

int mstrsm_comm_destroy(void) {
    if (g_comm) {
        NCK(ncclCommDestroy(g_comm));
        g_comm = nullptr;
    }
    g_comm_n = g_comm_r = 0;
    return 0;
}

int64_t mstrsm_dist_shard(int64_t m, int nranks, int rank, int64_t *cols_out) {
    if (m < 0 || nranks < 1 || rank < 0 || rank >= nranks) return -1;
    return shard_of(m, nranks, rank, kShardGroup, cols_out);
}

int mstrsm_d_dist(int safe, mstrsm_op op, const double *U, int64_t ldu, int64_t m, const double *shifts,
                  int64_t shift_stride, double *B, int64_t ldb, int64_t n, double *scales, int32_t *scale_exp,
                  int nb, int root) {
    return ex_dist_impl<double>(safe, int(op), U, ldu, m, shifts, shift_stride, B, ldb, n, scales, scale_exp, nb,
                                root);
}
int mstrsm_z_dist(int safe, mstrsm_op op, const mstrsm_dcomplex *U, int64_t ldu, int64_t m,
                  const mstrsm_dcomplex *shifts, int64_t shift_stride, mstrsm_dcomplex *B, int64_t ldb, int64_t n,
                  double *scales, int32_t *scale_exp, int nb, int root) {
    return ex_dist_impl<cplx>(safe, int(op), (const cplx *)U, ldu, m, (const cplx *)shifts, shift_stride,
                              (cplx *)B, ldb, n, scales, scale_exp, nb, root);
}

int trevc_d_dist(const double *T, int64_t ldt, int64_t m, double *Z, int64_t ldz, double *scales,
                 int32_t *scale_exp, int nb, int root) {
    return trevc_dist_impl<double>(T, ldt, m, Z, ldz, scales, scale_exp, nb, root);
}
int trevc_z_dist(const mstrsm_dcomplex *T, int64_t ldt, int64_t m, mstrsm_dcomplex *Z, int64_t ldz,
                 double *scales, int32_t *scale_exp, int nb, int root) {
    return trevc_dist_impl<cplx>((const cplx *)T, ldt, m, (cplx *)Z, ldz, scales, scale_exp, nb, root);
}

}  // extern "C"
