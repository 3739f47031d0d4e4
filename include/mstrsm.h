/*
 * mstrsm.h -- C ABI of libmstrsm.so: the B200-native (sm_100a) blocked, optionally
 * overflow-safe, multi-shift triangular solve of Moon & Poulson, arXiv 1607.01477
 * ("Accelerating eigenvector and pseudospectra computation using blocked multi-shift
 * triangular solves"), plus the two drivers the paper builds on it.
 *
 * Citations: P:n = line n of the paper text.  R# = reading in DESIGN.md §3.
 *
 * Conventions for every call
 *   - Column-major (LAPACK) storage with leading dimensions; element (i,j) of a matrix A
 *     with leading dimension lda is A[i + j*lda] (0-based).
 *   - Complex numbers are interleaved (re, im) doubles: mstrsm_dcomplex has the layout of C99
 *     double _Complex, std::complex<double>, cuDoubleComplex and torch.complex128.
 *   - Unless stated otherwise, every array argument is a DEVICE pointer, owned by the
 *     caller, and must stay valid until the work enqueued by the call has completed.
 *     B / Z are overwritten in place.  U, T, shifts are read-only.
 *   - The strictly lower triangle of U / T is never read.
 *   - Calls are ASYNCHRONOUS on the library's current stream (mstrsm_set_stream; default
 *     the legacy default stream): they enqueue kernels and return.  Device workspace is
 *     allocated stream-ordered (cudaMallocAsync) and released stream-ordered.
 *   - Thread and device safety: the current stream (mstrsm_set_stream), the status flag
 *     (mstrsm_status), the error string and the library's helper streams and events are kept
 *     per calling thread and per device (the device current at the call).  Several host
 *     threads may call the library concurrently, each on its own stream, and one thread may
 *     drive several GPUs.  The NCCL communicator of the multi-GPU entries is process-wide
 *     (one process per GPU).
 *   - nb is the block size n_b of Alg. 2/3/5.  nb = 0 selects the default
 *     (64).  1 <= nb <= 128.  nb is part of the semantics of the safe variants (it sets
 *     the granularity of the growth-bound updates, R10).
 *
 * Return codes (LAPACK INFO style)
 *     0   success (possibly with rescaling, reported through scales / scale_exp)
 *    -i   argument i is invalid (1-based position in the C prototype)
 *     1   CUDA launch / runtime error (message: mstrsm_error_string(1))
 *     2   non-finite entry in U or the shifts (safe variants; reported by
 *         mstrsm_status(), which synchronises -- the solve itself stays asynchronous; after
 *         mstrsm_set_sync_status(1) the call itself synchronises and returns it)
 *     3   communication error (multi-GPU helpers)
 *   m == 0 or n == 0 returns 0 immediately.  A zero right-hand-side column yields x = 0,
 *   c = 1 (R13).  The unsafe variants do not replace zero pivots: Inf/NaN propagate.
 */
#ifndef MSTRSM_H
#define MSTRSM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct { double re, im; } mstrsm_dcomplex;

typedef enum {
    MSTRSM_OP_N = 0,   /* (U - s_j I)   x_j = c_j b_j : back substitution, blocks bottom-up   */
    MSTRSM_OP_C = 1    /* (U - s_j I)^H x_j = c_j b_j : forward substitution, blocks top-down
                          (P:58-62 footnote: the lower-triangular case)                      */
} mstrsm_op;

/* ------------------------------------------------------------------------------------
 * Multi-shift triangular solve, Alg. 3: for j = 0..n-1 solve
 *     (U - shifts[j] I) x_j = b_j          (B(:,j) = b_j on entry, x_j on exit)
 * U: m x m upper triangular (ldu >= max(1,m)); shifts: n scalars; B: m x n (ldb >= max(1,m)).
 * scales (nullable, n doubles) is set to 1.0 (the plain solve never rescales).
 * Work: per block one diagonal-block solve per column + one shift-free update GEMM
 * B(I0,:) -= U(I0,I1) X(I1,:) shared by every shift.
 */
int mstrsm_d(const double *U, int64_t ldu, int64_t m, const double *shifts,
             double *B, int64_t ldb, int64_t n, double *scales, int nb);
int mstrsm_z(const mstrsm_dcomplex *U, int64_t ldu, int64_t m, const mstrsm_dcomplex *shifts,
             mstrsm_dcomplex *B, int64_t ldb, int64_t n, double *scales, int nb);

/* ------------------------------------------------------------------------------------
 * Safe multi-shift triangular solve, Alg. 5 with Alg. 4 on the
 * diagonal blocks: find x_j and c_j in [0,1] with (U - s_j I) x_j = c_j b_j
 * such that no intermediate reaches Omega = 2^970 (R1).  c_j = 2^{e_j} exactly (R2);
 * scales (required, n doubles) receives c_j, which may underflow to 0 (R12).
 * Zero pivots U(i,i) - s_j == 0 are replaced by delta = 2^-52 ||U||_inf (R4).
 */
int mstrsm_d_safe(const double *U, int64_t ldu, int64_t m, const double *shifts,
                  double *B, int64_t ldb, int64_t n, double *scales, int nb);
int mstrsm_z_safe(const mstrsm_dcomplex *U, int64_t ldu, int64_t m, const mstrsm_dcomplex *shifts,
                  mstrsm_dcomplex *B, int64_t ldb, int64_t n, double *scales, int nb);

/* ------------------------------------------------------------------------------------
 * Extended form of both solves.
 *   safe          0: Alg. 3, 1: Alg. 5
 *   op            MSTRSM_OP_N or MSTRSM_OP_C (C: (U - s I)^H, i.e. L = U^H - conj(s) I)
 *   shift_stride  stride between consecutive shifts (ldu + 1 reads diag(U) in place)
 *   row_end       nullable, op N only: n values r_j (clamped to [0, m]); column j is
 *                 solved on rows [0, r_j) and rows [r_j, m) are set to 0 (R26; the eigen
 *                 shortcut of P:503-508 is r_k = k).  Device memory or host
 *                 memory, told apart with cudaPointerGetAttributes.  If the values are
 *                 non-decreasing the library skips inactive columns per block; to know that it
 *                 reads them on the host, so a DEVICE row_end costs one synchronisation of the
 *                 caller's stream (the work already enqueued on it completes first).  Read
 *                 before return; the caller may free or reuse it afterwards.
 *   scales        nullable for safe = 0; required for safe = 1
 *   scale_exp     nullable: n int32 receiving e_j (c_j = 2^{e_j}); 0 for safe = 0
 */
int mstrsm_d_ex(int safe, mstrsm_op op, const double *U, int64_t ldu, int64_t m,
                const double *shifts, int64_t shift_stride, double *B, int64_t ldb, int64_t n,
                const int64_t *row_end, double *scales, int32_t *scale_exp, int nb);
int mstrsm_z_ex(int safe, mstrsm_op op, const mstrsm_dcomplex *U, int64_t ldu, int64_t m,
                const mstrsm_dcomplex *shifts, int64_t shift_stride, mstrsm_dcomplex *B, int64_t ldb,
                int64_t n, const int64_t *row_end, double *scales, int32_t *scale_exp,
                int nb);

/* Caller-managed workspace: as mstrsm_*_ex, with every device allocation of the
 * solve carved from `workspace` (device, 256-byte aligned, caller-owned, not touched after the
 * work enqueued by the call completes) instead of the stream-ordered pool.  workspace = NULL
 * behaves as mstrsm_*_ex.  mstrsm_workspace_size returns a sufficient size (bytes) for the
 * given problem (0 for an empty problem or an invalid nb).  Errors as mstrsm_*_ex, plus -15
 * (misaligned workspace) and -16 (workspace_bytes too small).                               */
size_t mstrsm_workspace_size(int64_t m, int64_t n, int nb, int is_complex, int safe);
int mstrsm_d_ex_ws(int safe, mstrsm_op op, const double *U, int64_t ldu, int64_t m,
                   const double *shifts, int64_t shift_stride, double *B, int64_t ldb, int64_t n,
                   const int64_t *row_end, double *scales, int32_t *scale_exp, int nb,
                   void *workspace, size_t workspace_bytes);
int mstrsm_z_ex_ws(int safe, mstrsm_op op, const mstrsm_dcomplex *U, int64_t ldu, int64_t m,
                   const mstrsm_dcomplex *shifts, int64_t shift_stride, mstrsm_dcomplex *B,
                   int64_t ldb, int64_t n, const int64_t *row_end, double *scales,
                   int32_t *scale_exp, int nb, void *workspace, size_t workspace_bytes);

/* ------------------------------------------------------------------------------------
 * The footnote family of P:58-62: left/right, upper/lower.
 *   side = LEFT : (A - s_j I) x_j = c_j b_j          B is m x n (ldb >= max(1,m)), column j = b_j
 *   side = RIGHT: x_j^T (A - s_j I) = c_j b_j^T      B is n x m (ldb >= max(1,n)), row j = b_j^T
 *   uplo = UPPER: A upper triangular (strictly lower part never read);
 *   uplo = LOWER: A lower triangular (strictly upper part never read); lower = forward substitution.
 * No conjugation on either side (X op(A) with op = identity).  Left-upper is mstrsm_*_ex op N;
 * the others run the op N / op C kernels on a transformed copy of the triangle (A^H, A^T or
 * conj A, library workspace) and, for RIGHT, on B^T.  Other arguments as
 * mstrsm_*_ex (no row_end).  Errors: -i for argument i, 1 CUDA error.                     */
typedef enum { MSTRSM_LEFT = 0, MSTRSM_RIGHT = 1 } mstrsm_side;
typedef enum { MSTRSM_UPPER = 0, MSTRSM_LOWER = 1 } mstrsm_uplo;
int mstrsm_d_side(int safe, mstrsm_side side, mstrsm_uplo uplo, const double *A, int64_t lda, int64_t m,
                  const double *shifts, int64_t shift_stride, double *B, int64_t ldb, int64_t n,
                  double *scales, int32_t *scale_exp, int nb);
int mstrsm_z_side(int safe, mstrsm_side side, mstrsm_uplo uplo, const mstrsm_dcomplex *A, int64_t lda,
                  int64_t m, const mstrsm_dcomplex *shifts, int64_t shift_stride, mstrsm_dcomplex *B,
                  int64_t ldb, int64_t n, double *scales, int32_t *scale_exp, int nb);

/* ------------------------------------------------------------------------------------
 * Triangular eigenvectors, Alg. 6 TriangEig: lambda = diag(T); Z := -T with
 * diag(Z) := 0; safe multi-shift solve with shifts lambda, shortcut to the strictly upper
 * RHS (R11); diag(Z) := s.  T Z = Z diag(lambda) backward-stably.
 *   T      m x m upper triangular (ldt >= max(1,m)), read-only
 *   Z      m x m output (ldz >= max(1,m)); Z(k,k) = c_k = 2^{e_k}, rows > k are 0
 *   scales nullable (m doubles, = diag Z); scale_exp nullable (m int32)
 */
int trevc_d(const double *T, int64_t ldt, int64_t m, double *Z, int64_t ldz,
            double *scales, int32_t *scale_exp, int nb);
int trevc_z(const mstrsm_dcomplex *T, int64_t ldt, int64_t m, mstrsm_dcomplex *Z, int64_t ldz,
            double *scales, int32_t *scale_exp, int nb);

/* Column subset (the shard of one GPU when shifts are partitioned across GPUs):
 *   cols_host  HOST pointer, ncols strictly increasing eigenvector indices in [0, m)
 *   Z          m x ncols output: Z(:,q) is eigenvector cols_host[q]; scales/scale_exp
 *              have ncols entries.  Results are bit-identical to the corresponding columns
 *              of trevc_* (columns are independent).                         */
int trevc_d_cols(const double *T, int64_t ldt, int64_t m, const int64_t *cols_host,
                 int64_t ncols, double *Z, int64_t ldz, double *scales, int32_t *scale_exp,
                 int nb);
int trevc_z_cols(const mstrsm_dcomplex *T, int64_t ldt, int64_t m, const int64_t *cols_host,
                 int64_t ncols, mstrsm_dcomplex *Z, int64_t ldz, double *scales,
                 int32_t *scale_exp, int nb);

/* End-to-end entry with HOST buffers: copies T (pinned or pageable host memory) to the
 * device, runs trevc_z, copies Z, scales and scale_exp back, and synchronises.
 * All pointers are HOST pointers (scales / scale_exp nullable).  Blocking.
 * Only the triangles travel (eigenvector k is zero below row k): T's upper triangle
 * up, Z's upper triangle down, in 128-column panels.  Entries of Z_host below the diagonal are
 * either left as the caller provided them or set to zero (those inside a panel's diagonal
 * 128 x 128 tile); pass a zeroed Z_host to receive the full matrix Z.                    */
int trevc_z_host(const mstrsm_dcomplex *T_host, int64_t ldt, int64_t m, mstrsm_dcomplex *Z_host,
                 int64_t ldz, double *scales_host, int32_t *scale_exp_host, int nb);

/* Batched host entry: count independent TriangEig problems, HOST pointer arrays (each entry a
 * HOST buffer, pinned for the copies to overlap).  Problem k+1's upload of T (upper triangle) and
 * problem k-1's download of Z / scales / scale_exp run on two copy streams while problem k is
 * solved, with two device buffer sets in flight.  scales_host / scale_exp_host: nullable arrays
 * (or nullable entries).  Blocking.  Z_host[k] below the diagonal: as trevc_z_host.  Copy
 * streams are per calling thread and device.  Errors: -i for argument i (-9 also for a failed
 * solve's argument check), 1 CUDA error (the copy streams are drained before returning, so no
 * copy touches the caller's buffers afterwards).                                        */
int trevc_z_host_batch(const mstrsm_dcomplex *const *T_host, int64_t ldt, int64_t m,
                       mstrsm_dcomplex *const *Z_host, int64_t ldz, double *const *scales_host,
                       int32_t *const *scale_exp_host, int64_t count, int nb);

/* ------------------------------------------------------------------------------------
 * Pseudospectra, Van Loan / Lui with multi-shift batching: for
 * every point z_p, sigma_min(U - z_p I) = 1/sqrt(lambda_max((U - zI)^{-H}(U - zI)^{-1}))
 * (P:600-604), lambda_max by `iters` Lanczos steps (R14) from the
 * shared unit-2-norm start vector v0 (m complex, device).  Each step is one op-N and one
 * op-C safe multi-shift solve over all points at once.
 *   z          npts complex shifts (device)
 *   sigma_min  npts doubles (device, output)
 *   flags      nullable npts int32: bit0 = a solve rescaled (near-singular point); sigma
 *              is then the upper bound c_1/||y||_2 of that step (R25)
 */
int pseudospectra_z(const mstrsm_dcomplex *U, int64_t ldu, int64_t m, const mstrsm_dcomplex *z,
                    int64_t npts, int iters, const mstrsm_dcomplex *v0, double *sigma_min,
                    int32_t *flags, int nb);

/* SpectralCloud: pseudospectra_z with per-point deflation.
 * With tol > 0 a point leaves the batch after the first Lanczos step k >= 2 whose Ritz value
 * theta_k = lambda_max(T_k) satisfies |theta_k - theta_{k-1}| <= tol theta_k (R33); the remaining
 * columns are compacted so later solves run on fewer shifts (one host synchronisation per step).
 * tol = 0: exactly pseudospectra_z with maxit steps.
 *   sigma  npts doubles (device): sigma_min(U - z_p I) estimates
 *   flags  nullable npts int32 (device): bit0 = rescaled solve (R25), bit1 = not settled within
 *          maxit steps (tol > 0)
 *   its    nullable npts int32 (device): Lanczos steps taken
 * Errors: -i for argument i (tol must be >= 0), 1 CUDA error.                              */
int spectral_cloud_z(const mstrsm_dcomplex *U, int64_t ldu, int64_t m, const mstrsm_dcomplex *z,
                     int64_t npts, int maxit, double tol, const mstrsm_dcomplex *v0, double *sigma,
                     int32_t *flags, int32_t *its, int nb);

/* SpectralWindow: SpectralCloud over the nx x ny grid x_i = linspace(x0, x1, nx),
 * y_j = linspace(y0, y1, ny) (endpoint-inclusive, numpy.linspace arithmetic), point index
 * i + nx j (R15).  sigma / flags / its have nx*ny entries.                                 */
int spectral_window_z(const mstrsm_dcomplex *U, int64_t ldu, int64_t m, double x0, double x1,
                      int64_t nx, double y0, double y1, int64_t ny, int maxit, double tol,
                      const mstrsm_dcomplex *v0, double *sigma, int32_t *flags, int32_t *its, int nb);

/* SpectralPortrait: SpectralWindow over the automatic window (R34): the bounding box
 * of diag(U) padded on each side by 0.25 max(box width, box height, 1e-2 ||U||_inf).
 * window_host: nullable HOST pointer, receives (x0, x1, y0, y1).  Synchronises the stream.  */
int spectral_portrait_z(const mstrsm_dcomplex *U, int64_t ldu, int64_t m, int64_t nx, int64_t ny,
                        int maxit, double tol, const mstrsm_dcomplex *v0, double *sigma,
                        int32_t *flags, int32_t *its, double *window_host, int nb);

/* ------------------------------------------------------------------------------------
 * Generalized multi-shift triangular solve, appendix Alg. 7 (safe = 0) and Alg. 8
 * (safe = 1): for j = 0..n-1 find x_j and c_j = 2^{e_j} in [0,1] with
 *     (U - shifts[j] V) x_j = c_j b_j          (op N only; B(:,j) = b_j on entry, x_j on exit)
 * U, V: m x m upper triangular, device, read-only (strictly lower triangles never read).
 * The diagonal blocks U' = U(I1,I1) - lambda V(I1,I1) are formed on the fly; the update
 * is B(I0) -= U(I0,I1) X(I1) and B(I0) += V(I0,I1) C, C = lambda X(I1).  Bounds: R30;
 * zero pivots of U' are replaced by delta_j = 2^-52 (||U|| + |lambda_j| ||V||) (R31); C is formed
 * after the column rescale (R32).  1 <= nb <= 64 (nb = 0: 64).  Other arguments as mstrsm_*_ex
 * (row_end nullable, device or host memory, as there).  Errors: -i for argument i, 1 CUDA
 * error.                                                                                   */
int mstrsm_d_gen(int safe, const double *U, int64_t ldu, const double *V, int64_t ldv, int64_t m,
                 const double *shifts, int64_t shift_stride, double *B, int64_t ldb, int64_t n,
                 const int64_t *row_end, double *scales, int32_t *scale_exp, int nb);
int mstrsm_z_gen(int safe, const mstrsm_dcomplex *U, int64_t ldu, const mstrsm_dcomplex *V, int64_t ldv,
                 int64_t m, const mstrsm_dcomplex *shifts, int64_t shift_stride, mstrsm_dcomplex *B,
                 int64_t ldb, int64_t n, const int64_t *row_end, double *scales, int32_t *scale_exp,
                 int nb);

/* GeneralizedTriangEig, appendix Alg. 9 first function: lambda_k = T(k,k)/S(k,k)
 * (finite eigenvalues: S(k,k) != 0 required), Z(:,k) := -T(:,k) + lambda_k S(:,k) on rows < k,
 * safe generalized solve with the P:503-508 shortcut, Z(k,k) := c_k = 2^{e_k}; rows > k are 0.
 * T Z = S Z diag(lambda) backward-stably.  T, S (device, read-only), Z (device, m x m output),
 * lambda (device, nullable, m), scales / scale_exp (device, nullable, m).  1 <= nb <= 64.   */
int tgevc_d(const double *T, int64_t ldt, const double *S, int64_t lds, int64_t m, double *Z, int64_t ldz,
            double *lambda, double *scales, int32_t *scale_exp, int nb);
int tgevc_z(const mstrsm_dcomplex *T, int64_t ldt, const mstrsm_dcomplex *S, int64_t lds, int64_t m,
            mstrsm_dcomplex *Z, int64_t ldz, mstrsm_dcomplex *lambda, double *scales, int32_t *scale_exp,
            int nb);

/* ------------------------------------------------------------------------------------
 * Back-transformation of Eig: X := Q Z, the xGEMM step after
 * TriangEig, here a TRMM-shaped DMMA contraction exploiting that column q of Z is zero below
 * row cols[q] (Z from trevc_*: upper triangular).  Column scales are unchanged: X(:,q) is the
 * eigenvector of A = Q T Q^H times the same c_q as Z(:,q).
 *   Q      m x m (ldq >= max(1,m)), device, read-only (any matrix; unitary for Eig)
 *   Z      m x n (ldz >= max(1,m)), device, read-only
 *   cols_host  HOST pointer, nullable: n strictly increasing row bounds, Z(r,q) = 0 for
 *          r > cols_host[q] (trevc_*_cols order); NULL = cols[q] = q (n <= m)
 *   X      m x n output (ldx >= max(1,m)), device; must not overlap Q or Z
 * Errors: -i for argument i, 1 CUDA error.  Asynchronous on the library stream.            */
int eig_backtransform_d(const double *Q, int64_t ldq, int64_t m, const double *Z, int64_t ldz, int64_t n,
                        const int64_t *cols_host, double *X, int64_t ldx);
int eig_backtransform_z(const mstrsm_dcomplex *Q, int64_t ldq, int64_t m, const mstrsm_dcomplex *Z,
                        int64_t ldz, int64_t n, const int64_t *cols_host, mstrsm_dcomplex *X, int64_t ldx);

/* Eig's last two steps fused: Z := TriangEig(T) in a library-owned workspace
 * (trevc_*, same nb rules), then X := Q Z.  X (m x m, device) holds the eigenvectors of
 * A = Q T Q^H, column k scaled by c_k = scales[k] = 2^{scale_exp[k]} (nullable outputs).   */
int trevc_qz_d(const double *T, int64_t ldt, int64_t m, const double *Q, int64_t ldq, double *X,
               int64_t ldx, double *scales, int32_t *scale_exp, int nb);
int trevc_qz_z(const mstrsm_dcomplex *T, int64_t ldt, int64_t m, const mstrsm_dcomplex *Q, int64_t ldq,
               mstrsm_dcomplex *X, int64_t ldx, double *scales, int32_t *scale_exp, int nb);

/* ------------------------------------------------------------------------------------
 * Multi-GPU: one process per GPU, an NCCL communicator over the ranks.
 *   mstrsm_comm_unique_id  rank 0 draws the 128-byte NCCL id (host buffer); the caller hands it
 *                          to every rank (e.g. over its torch process group)
 *   mstrsm_comm_init       every rank, on its current device; replaces a previous communicator
 *   mstrsm_dist_shard      host only: the eigenvector indices rank `rank` of `nranks` owns
 *                          (groups of 16 columns dealt serpentine block-cyclically, balancing the
 *                          ~(k-1)^2 cost); returns the count, fills cols_out (nullable) ascending
 *   trevc_*_dist           TriangEig over all ranks: T (device) is read on `root` only (other
 *                          ranks may pass NULL / any ldt).  Root computes delta (R4, ||T||_inf)
 *                          and broadcasts it, then T's upper triangle in 128-column panels right
 *                          to left (the order the blocks consume it) on a separate
 *                          stream; each rank's block b waits only for panel b, so the solve of its
 *                          shard overlaps the rest of the broadcast.  Each block's finished rows
 *                          are all-gathered behind the compute front; the ranks then agree on a
 *                          status (one all-reduce), gather the exponents, and every rank receives
 *                          the full Z (m x m, ldz), scales and scale_exp (nullable, m entries) in
 *                          natural order -- bit-identical to trevc_*.  Collective and blocking: every rank must call it; the call
 *                          returns when its work is done.  NCCL's asynchronous errors are polled
 *                          while waiting; an error or a wait longer than MSTRSM_NCCL_TIMEOUT_S
 *                          (default 600 s) aborts the communicator and returns 3.  Errors: -i for
 *                          argument i, 1 CUDA error, 3 communication error, timeout, a failure
 *                          on another rank, or no communicator.                            */
/* Triangular shard packing for the all-gather (eigenvector k is zero below row k):
 *   pack:   out[offsets[q] .. + heights[q]) = Z(0 : heights[q], src_cols[q])   (src_cols
 *           nullable: q), q < n
 *   unpack: Z(0 : heights[q], dst_cols[q]) = in[offsets[q] ..], rows heights[q] .. m-1 of that
 *           column set to 0, q < n
 * All pointers DEVICE; heights / offsets / cols int64.  Errors: -i for argument i.           */
int mstrsm_d_pack_cols(const double *Z, int64_t ldz, int64_t n, const int64_t *src_cols,
                       const int64_t *heights, const int64_t *offsets, double *out);
int mstrsm_z_pack_cols(const mstrsm_dcomplex *Z, int64_t ldz, int64_t n, const int64_t *src_cols,
                       const int64_t *heights, const int64_t *offsets, mstrsm_dcomplex *out);
int mstrsm_d_unpack_cols(const double *in, int64_t n, const int64_t *heights, const int64_t *offsets,
                         const int64_t *dst_cols, int64_t m, double *Z, int64_t ldz);
int mstrsm_z_unpack_cols(const mstrsm_dcomplex *in, int64_t n, const int64_t *heights,
                         const int64_t *offsets, const int64_t *dst_cols, int64_t m,
                         mstrsm_dcomplex *Z, int64_t ldz);
int     mstrsm_comm_unique_id(void *id_out);
int     mstrsm_comm_init(int nranks, int rank, const void *unique_id);
int     mstrsm_comm_destroy(void);
int64_t mstrsm_dist_shard(int64_t m, int nranks, int rank, int64_t *cols_out);
int trevc_d_dist(const double *T, int64_t ldt, int64_t m, double *Z, int64_t ldz, double *scales,
                 int32_t *scale_exp, int nb, int root);
/* Dense right-hand sides sharded by column (shifts / B / scales / scale_exp hold this rank's n
 * columns): U (device) is read on `root` only and its upper triangle broadcast; every rank then
 * runs mstrsm_*_ex on its own columns (no gather).  Collective and blocking (NCCL errors and
 * timeouts as trevc_*_dist: return 3).  Arguments as mstrsm_*_ex (no row_end), root last.   */
int mstrsm_d_dist(int safe, mstrsm_op op, const double *U, int64_t ldu, int64_t m, const double *shifts,
                  int64_t shift_stride, double *B, int64_t ldb, int64_t n, double *scales,
                  int32_t *scale_exp, int nb, int root);
int mstrsm_z_dist(int safe, mstrsm_op op, const mstrsm_dcomplex *U, int64_t ldu, int64_t m,
                  const mstrsm_dcomplex *shifts, int64_t shift_stride, mstrsm_dcomplex *B, int64_t ldb,
                  int64_t n, double *scales, int32_t *scale_exp, int nb, int root);
int trevc_z_dist(const mstrsm_dcomplex *T, int64_t ldt, int64_t m, mstrsm_dcomplex *Z, int64_t ldz,
                 double *scales, int32_t *scale_exp, int nb, int root);

/* ------------------------------------------------------------------------------------
 * Runtime helpers */
int         mstrsm_set_stream(void *cuda_stream);  /* cudaStream_t; NULL = legacy stream */
void       *mstrsm_get_stream(void);
const char *mstrsm_error_string(int code);
/* Synchronises the current stream; returns 0, 1 (sticky CUDA error) or 2 (a safe call
 * since the last mstrsm_status saw a non-finite U entry or shift); clears the flag.   */
int         mstrsm_status(void);
/* on = 1: every safe solve / eigenvector entry (mstrsm_*_safe, _ex, _ex_ws, _side, _gen,
 * trevc_*, trevc_*_cols, trevc_qz_*, tgevc_*) synchronises the current stream before it
 * returns and returns 2 itself when the input held a non-finite value (clearing the flag as
 * mstrsm_status does).  on = 0 (default): asynchronous, code 2 through mstrsm_status only.
 * Per calling thread.  Returns 0.                                                         */
int         mstrsm_set_sync_status(int on);
/* Number of kernels libmstrsm.so has launched since the last reset (for bench/gpu_launches). */
int64_t     mstrsm_launch_count(int reset);

/* Live kernel timing for the bench: mstrsm_profile(1) clears and starts bracketing every
 * library launch with CUDA events on the launching stream; mstrsm_profile(0) stops.
 * mstrsm_profile_read synchronises and returns, for one kernel kind (0 = update GEMM,
 * 1 = diagonal-block kernel, 2 = other), the summed device time, the launch count and the
 * algorithmic flops of those launches (GEMM: 2 M N K real / 8 M N K complex).            */
int         mstrsm_profile(int enable);
/* Real DMMA products per complex multiply-add in the update GEMM: 3 (default: P1 = Ar Xr,
 * P2 = Ai Xi, P3 = (Ar + Ai)(Xr + Xi), Re = P1 - P2, Im = P3 - P1 - P2) or 4 (Re = Ar Xr - Ai Xi,
 * Im = Ar Xi + Ai Xr; environment MSTRSM_GEMM=4m or classic).  The profile's flops stay the
 * algorithmic complex count (8 M N K); executed real flops = that x (products / 4).            */
int         mstrsm_gemm_real_products(void);
int         mstrsm_profile_read(int kind, double *total_ms, int64_t *launches, double *flops);

/* FP64 roofline probe: a register-resident DMMA (mma.sync.m8n8k4.f64) loop and a DFMA loop
 * on every SM for about `ms` milliseconds each; returns achieved TFLOP/s (2 flops/FMA).
 * Synchronous.                                                                          */
int mstrsm_fp64_peak(double ms, double *dmma_tflops, double *dfma_tflops);

#ifdef __cplusplus
}
#endif
#endif /* MSTRSM_H */
