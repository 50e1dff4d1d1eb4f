/*
 * choldiff.h -- C ABI of libcholdiff.so: B200 (sm_100a) kernels that propagate
 * derivatives through the Cholesky decomposition Sigma = L L^T
 * (arXiv 1602.07527, "the paper"; PAPER.md line numbers below).
 *
 *   reverse mode  cd_chol_rev*:  (L, Lbar)      -> Sigma_bar
 *   forward mode  cd_chol_fwd*:  (L, Sigma_dot) -> L_dot
 *
 * ---------------------------------------------------------------------------
 * Layout (all entry points)
 *   - Matrices are n x n, COLUMN-MAJOR (LAPACK): element (i, j), 0-based, of a
 *     matrix at pointer P with leading dimension ld is P[i + j*ld]; ld >= max(1,n).
 *   - Only the LOWER triangle (i >= j) of L, Lbar and Sigma_dot is ever read
 *     (PAPER.md:448-451, 612-613).  The upper triangle of L may hold anything
 *     (e.g. Sigma); it is never read.
 *   - Element type per cd_dtype: CD_F64 = IEEE double, CD_F32 = IEEE float.
 *   - Batched variants: either base + stride (matrix b at P + b*stride elements,
 *     stride >= ld*n, e.g. a contiguous batch has ld = n, stride = n*n), or a
 *     DEVICE array of DEVICE pointers (cuBLAS "...Batched" style).
 *
 * In-place semantics
 *   - Reverse: on entry tril(Abar) = Lbar; on exit tril(Abar) = tril(Sigma_bar),
 *     the paper's Eq. 10 convention: Sigma_bar_kl = df/dSigma_kl
 *     with Sigma_kl = Sigma_lk counted as ONE variable.  out_mode selects what is
 *     written (cd_out_mode below).
 *   - Forward: on entry tril(Adot) = tril(Sigma_dot) (Sigma_dot symmetric, only
 *     its lower triangle is read); on exit tril(Adot) = L_dot.
 *   - The upper triangle of Abar / Adot is never read, and is not written in
 *     CD_OUT_TRIL mode (the default).
 *   - L must not overlap Abar / Adot.
 *
 * Ownership
 *   - The caller owns every buffer.  All pointers are DEVICE pointers unless the
 *     function name ends in _host.  The library never allocates device memory,
 *     never frees, and retains no pointer past the call's enqueue.
 *   - `ws` is a device workspace of at least cd_workspace_size(...) bytes,
 *     256-byte aligned; it may be NULL only when that size is 0.
 *
 * Streams and errors
 *   - All work is enqueued on `stream` (a cudaStream_t; NULL = legacy default
 *     stream); the host call returns after enqueue (asynchronous).
 *   - Return value: CD_SUCCESS (0) when the work was enqueued; -i when argument
 *     i (1-based position in the C signature) is invalid (LAPACK INFO style:
 *     n < 0, ld < max(1,n), stride too small, bad enum, NULL pointer with work
 *     to do, workspace too small); CD_ERR_CUDA when a launch failed
 *     (cd_status_string / cd_last_cuda_error give the text); CD_ERR_UNSUPPORTED
 *     for a valid but unimplemented combination.
 *   - Numerical status is asynchronous: if `d_info` (device int[batch], may be
 *     NULL) is given, d_info[b] = 0 when matrix b was processed normally, or
 *     j > 0 (1-based) when L[j-1, j-1] is zero or non-finite (the first such j);
 *     outputs of that matrix are then unspecified.  Other non-finite inputs are
 *     not checked (finiteness is a precondition).
 *   - n = 0 or batch = 0 is a no-op returning CD_SUCCESS.
 *   - Reentrant from any number of host threads.  Library state: per-device caches
 *     (kernel attributes, occupancies, SM counts; initialised once, thread-safe);
 *     per-host-thread, per-device CUDA streams and events that some calls create on
 *     first use (the lookahead and host-copy streams, chol_rev_fwd's side stream),
 *     released when the thread exits; per-thread measurement state (launch counter,
 *     profiling records, last CUDA error text).  Measurement switches are read from
 *     the environment once per process.  L may be shared read-only by concurrent
 *     calls; calls that share an output or a workspace must be ordered by the caller.
 */
#ifndef CHOLDIFF_H
#define CHOLDIFF_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CD_VERSION 100 /* 1.0.0 */

typedef struct CUstream_st* cd_stream_t; /* == cudaStream_t */

typedef enum { CD_F64 = 0, CD_F32 = 1 } cd_dtype;
typedef enum { CD_OP_REV = 0, CD_OP_FWD = 1, CD_OP_CHOL_FWD = 2 } cd_op;

/* Route (the symbolic result may be preferable for small
 * matrices).  AUTO = ALGORITHMIC (measured faster on B200 at every size); ALGORITHMIC =
 * the paper's unblocked/blocked sweeps; SYMBOLIC = Eq. 10
 * (reverse) / Eq. 8 (forward) on the whole matrix:
 * one CTA per matrix for n <= 64, blocked triangular solves on the GEMM kernels above
 * (about 6x the sweep's flops; for measurement). */
typedef enum { CD_ROUTE_AUTO = 0, CD_ROUTE_ALGORITHMIC = 1, CD_ROUTE_SYMBOLIC = 2 } cd_route;

/* Reverse-mode output convention (reading c1):
 *   TRIL: tril(Sigma_bar) of Eq. 10, lower triangle only (default);
 *   SYM : the full symmetric Sigma_bar = S + S^T - diag(S) of Eq. 9:
 *         lower as TRIL, upper triangle written as its exact mirror;
 *   GRAD: G = (S + S^T)/2, the symmetric-gradient convention of autograd
 *         frameworks: off-diagonal entries of Eq. 9 halved, both triangles written.
 * Forward mode accepts TRIL only. */
typedef enum { CD_OUT_TRIL = 0, CD_OUT_SYM = 1, CD_OUT_GRAD = 2 } cd_out_mode;

typedef struct cd_opts {
  int32_t nb;       /* block size N_b of the blocked sweeps; 0 = auto */
  int32_t route;    /* cd_route   */
  int32_t out_mode; /* cd_out_mode */
  int32_t flags;    /* reserved, must be 0 */
} cd_opts;          /* NULL opts = {0, CD_ROUTE_AUTO, CD_OUT_TRIL, 0} */

enum {
  CD_SUCCESS = 0,
  CD_ERR_CUDA = 1,        /* a CUDA launch / copy failed */
  CD_ERR_UNSUPPORTED = 2  /* valid arguments, combination not implemented */
};

/* Single matrix, reverse mode: tril(Abar) = Lbar -> tril(Sigma_bar) (in place).
 * Blocked sweep of PAPER.md:689-701 for n > the on-chip limit, unblocked on-chip
 * sweep otherwise. */
int cd_chol_rev(cd_dtype dt, int64_t n, const void* L, int64_t ldl, void* Abar, int64_t ldabar,
                const cd_opts* opts, void* ws, size_t ws_bytes, int* d_info, cd_stream_t stream);

/* Single matrix, forward mode: tril(Adot) = tril(Sigma_dot) -> L_dot (in place).
 * PAPER.md:655-666 (blocked) / 489-498 (unblocked). */
int cd_chol_fwd(cd_dtype dt, int64_t n, const void* L, int64_t ldl, void* Adot, int64_t ldadot,
                const cd_opts* opts, void* ws, size_t ws_bytes, int* d_info, cd_stream_t stream);

/* Batched, base + stride (strides in ELEMENTS). */
int cd_chol_rev_strided_batched(cd_dtype dt, int64_t n, const void* L, int64_t ldl, int64_t strideL,
                                void* Abar, int64_t ldabar, int64_t strideAbar, int64_t batch,
                                const cd_opts* opts, void* ws, size_t ws_bytes, int* d_info,
                                cd_stream_t stream);
int cd_chol_fwd_strided_batched(cd_dtype dt, int64_t n, const void* L, int64_t ldl, int64_t strideL,
                                void* Adot, int64_t ldadot, int64_t strideAdot, int64_t batch,
                                const cd_opts* opts, void* ws, size_t ws_bytes, int* d_info,
                                cd_stream_t stream);

/* Batched, device arrays of device pointers (L_array[b], Abar_array[b]). */
int cd_chol_rev_batched(cd_dtype dt, int64_t n, const void* const* L_array, int64_t ldl,
                        void* const* Abar_array, int64_t ldabar, int64_t batch, const cd_opts* opts,
                        void* ws, size_t ws_bytes, int* d_info, cd_stream_t stream);
int cd_chol_fwd_batched(cd_dtype dt, int64_t n, const void* const* L_array, int64_t ldl,
                        void* const* Adot_array, int64_t ldadot, int64_t batch, const cd_opts* opts,
                        void* ws, size_t ws_bytes, int* d_info, cd_stream_t stream);

/* Both sensitivities of the same factors in one call (configs[3]'s workload): Abar (tril(Lbar) ->
 * tril(Sigma_bar), per opts->out_mode) and Adot (tril(Sigma_dot) -> L_dot), i.e. cd_chol_rev and
 * cd_chol_fwd on the same L.  The two sweeps are independent; the forward one runs on a
 * library-owned stream (per device and host thread) that starts after the work already queued on
 * `stream` and that `stream` waits for, so the call is ordered on `stream` like any other.
 * d_info (optional) receives the reverse sweep's status.  Argument checks as for the strided
 * batched calls (1-based positions); ws >= cd_workspace_size_rev_fwd(...) bytes (-14 otherwise). */
size_t cd_workspace_size_rev_fwd(cd_dtype dt, int64_t n, int64_t batch, const cd_opts* opts);
int cd_chol_rev_fwd_strided_batched(cd_dtype dt, int64_t n, const void* L, int64_t ldl, int64_t strideL,
                                    void* Abar, int64_t ldabar, int64_t strideAbar, void* Adot, int64_t ldadot,
                                    int64_t strideAdot, int64_t batch, const cd_opts* opts, void* ws,
                                    size_t ws_bytes, int* d_info, cd_stream_t stream);

/* Device workspace (bytes) that a call with these arguments needs; 0 if none.
 * `batch` = 1 for the single-matrix calls.  For the pointer-array batched calls
 * pass the batch size as well. */
size_t cd_workspace_size(cd_op op, cd_dtype dt, int64_t n, int64_t batch, const cd_opts* opts);

/* Host-buffer convenience for one matrix (end-to-end measurement path): copies
 * the dense n x n column-major host arrays L and A (ld = n) to the device
 * workspace, runs cd_chol_rev / cd_chol_fwd there, and copies A back.
 * `ws` must hold cd_workspace_size_host(...) bytes.  Host buffers should be
 * pinned for the copies to be asynchronous; the call is asynchronous on `stream`
 * (synchronize before reading A). */
size_t cd_workspace_size_host(cd_op op, cd_dtype dt, int64_t n, const cd_opts* opts);
int cd_chol_host(cd_op op, cd_dtype dt, int64_t n, const void* L_host, void* A_host,
                 const cd_opts* opts, void* ws, size_t ws_bytes, cd_stream_t stream);
/* Fused factorisation + forward mode: chol_blocked and
 * chol_blocked_fwd accumulated in one sweep, as PAPER.md:501-503 and
 * 649-651 suggest ("these updates could be accumulated at the same time as computing the
 * original Cholesky decomposition").
 *   in:  tril(A) = tril(Sigma) (Sigma symmetric positive definite), tril(Adot) = tril(Sigma_dot)
 *   out: tril(A) = L with Sigma = L L^T, tril(Adot) = Ldot
 * Both in place, column-major, only lower triangles read or written.  fp64 only (fp32 returns
 * CD_ERR_UNSUPPORTED); n <= 128 runs on chip, larger n needs the fused nb = 128 schedule:
 * 16-byte aligned arrays with even ld (otherwise CD_ERR_UNSUPPORTED).  d_info[b] = j > 0 if
 * the j-th (1-based) pivot of the factorisation was not positive (Sigma not positive
 * definite); outputs are then unspecified.  Workspace: cd_workspace_size(CD_OP_CHOL_FWD, ...). */
int cd_chol_fwd_fused(cd_dtype dt, int64_t n, void* A, int64_t lda, void* Adot, int64_t ldadot,
                      const cd_opts* opts, void* ws, size_t ws_bytes, int* d_info, cd_stream_t stream);
int cd_chol_fwd_fused_strided_batched(cd_dtype dt, int64_t n, void* A, int64_t lda, int64_t strideA,
                                      void* Adot, int64_t ldadot, int64_t strideAdot, int64_t batch,
                                      const cd_opts* opts, void* ws, size_t ws_bytes, int* d_info,
                                      cd_stream_t stream);

/* ---- Distributed single-matrix sweeps -------------------------------------
 * The blocked reverse sweep with the columns distributed 1-D block-cyclically
 * over P ranks: block K = [j, k) of the reverse partition (the short block at the top left,
 * PAPER.md:704-707) lives on rank K mod P, which stores its column blocks -- ALL n rows of L and
 * Abar -- side by side in a local n x c_loc column-major array.  Per block, right to left:
 *   owner:      cd_dist_rev_panel   Cbar <- Cbar D^{-1}; Dbar <- Dbar - tril(Cbar^T C);
 *                                   Dbar <- chol_unblocked_rev(D, Dbar)
 *                                   and packs X = [S; Cbar] ((n-j) x w), S = Dbar + Dbar^T
 *   broadcast X from the owner to every rank (the caller's collective: NCCL / torch.distributed)
 *   every rank: cd_dist_rev_update  for its column blocks left of the panel (the first q local
 *                                   columns): Bbar <- Bbar - Cbar R; Rbar <- Rbar - [S; Cbar]^T [R; B]
 *
 * The data exchanged per block is X alone; every update is local to the column owner.
 *
 * cd_dist_rev_panel: Lk, Ak = the owner's local column block (n rows, w columns, ld ldl / lda >= n),
 *   global rows; j = the block's first row/column (0-based), 1 <= w <= 128, j + w <= n.
 *   Ak is updated in place (rows j..n-1); X (device, ld ldx >= n - j) receives [S; Cbar].
 * cd_dist_rev_update: X from the panel of block [j, j+w); Lq, Aq = the rank's first q local columns
 *   (all global columns < j); Aq rows j..n-1 are updated in place.  q = 0 is a no-op.
 * Both: device pointers, asynchronous on `stream`, fp64 / fp32, batch 1, no d_info (check the
 * diagonal with cd_chol_rev on the owner if needed); ws >= cd_dist_workspace_size(dt, w) bytes.
 * Returns 0, -i for an invalid i-th argument, or CD_ERR_CUDA. */
size_t cd_dist_workspace_size(cd_dtype dt, int64_t w);
int cd_dist_rev_panel(cd_dtype dt, int64_t n, int64_t j, int64_t w, const void* Lk, int64_t ldl, void* Ak,
                      int64_t lda, void* X, int64_t ldx, void* ws, size_t ws_bytes, cd_stream_t stream);
int cd_dist_rev_update(cd_dtype dt, int64_t n, int64_t j, int64_t w, const void* X, int64_t ldx, int64_t q,
                       const void* Lq, int64_t ldl, void* Aq, int64_t lda, void* ws, size_t ws_bytes,
                       cd_stream_t stream);

/* Distributed forward sweep, same distribution and block partition as above
 * (any partition is exact), blocks left to right.  Per block [j, k):
 *   every rank: cd_dist_fwd_partial  Z_r = [Adot L][j:n, its first q local columns] .
 *                                         [L Adot][j:k, same columns]^T     ((n-j) x w, ldz = n - j;
 *                                         zero when q = 0) -- its share of [Rdot R^T + R Rdot^T ;
 *                                         Bdot R^T + B Rdot^T]
 *   sum-reduce Z_r onto the owner (the caller's collective)
 *   owner:      cd_dist_fwd_panel    Ddot <- Ddot - tril(Z_top); Cdot <- Cdot - Z_bottom;
 *                                    Ddot <- chol_unblocked_fwd(D, Ddot); Cdot <- (Cdot - C Ddot^T) D^{-T}
 *
 * Adot holds tril(Sigma_dot) in and L_dot out (the owner's block rows j..n-1).  Arguments and
 * errors as for the reverse steps. */
int cd_dist_fwd_partial(cd_dtype dt, int64_t n, int64_t j, int64_t w, int64_t q, const void* Lq, int64_t ldl,
                        const void* Aq, int64_t lda, void* Z, int64_t ldz, void* ws, size_t ws_bytes,
                        cd_stream_t stream);
int cd_dist_fwd_panel(cd_dtype dt, int64_t n, int64_t j, int64_t w, const void* Lk, int64_t ldl, void* Ak,
                      int64_t lda, const void* Z, int64_t ldz, void* ws, size_t ws_bytes, cd_stream_t stream);

/* Bytes the last cd_chol_host call on this thread moved host -> device and device -> host.
 * fp64 with the fused nb = 128 schedules and TRIL output (the default) pipelines the copies:
 * the lower part of each 128-column block streams in on a library copy stream just before
 * the sweep needs it and streams out as soon as it is final, so only the lower triangles
 * (plus the diagonal blocks once more) cross the bus; other cases copy the dense arrays. */
void cd_host_bytes(int64_t* h2d, int64_t* d2h);

/* Diagnostic entry point (kernel validation): C = alpha * op(A) op(B) + beta * C with the
 * library's Level-3 kernel family (op = transpose when ta / tb = 1), column-major, device
 * pointers, one matrix; `ws` >= 304*128*128*sizeof(element) bytes (split-K partials). */
int cd_debug_gemm(cd_dtype dt, int64_t M, int64_t N, int64_t K, int ta, int tb, const void* A, int64_t lda,
                  const void* B, int64_t ldb, void* C, int64_t ldc, double alpha, double beta, void* ws,
                  size_t ws_bytes, cd_stream_t stream);

const char* cd_status_string(int status);
const char* cd_last_cuda_error(void); /* text of the last CUDA error seen by this thread */
int cd_version(void);

/* Number of kernel launches the library enqueued on this thread since the last
 * reset (evidence for bench.py's "gpu_launches"). */
int64_t cd_launch_count(void);
void cd_reset_launch_count(void);

/* Measurement only: enable (1) / disable (0) clock64 stamps at the phase boundaries of CTA 0 of the
 * on-chip reverse sweep for n = 57..64 (while enabled the library launches a separately compiled
 * instance with the stamps; production launches carry none) and copy the last stamps (up to `max`,
 * at most 40) to host memory `out` (may be NULL).  Synchronous (cudaMemcpyFromSymbol). */
int cd_debug_phase_clocks(int enable, long long* out, int max);

/* Kernel-class timing (measurement evidence for bench.py's roofline).  While
 * enabled, the library brackets every launch it enqueues on this thread with a
 * pair of CUDA events on the launch stream and records the launch's ALGORITHMIC
 * flop count (the paper's operation count for that update, e.g. 2*M*N*K for
 * Bbar -= Cbar R, p*w*(w+1) for the panel solve Cbar D^{-1}).  cd_profile_read
 * synchronizes the recorded events and returns, for kernel class `cls`
 * (CD_PROF_GEMM, CD_PROF_REDUCE, CD_PROF_SWEEP, CD_PROF_TRINV, CD_PROF_OTHER,
 * CD_PROF_SYMM = the left-looking trailing update k_symm_ll, CD_PROF_PANEL = the fused
 * panel solve + diagonal correction k_panel_rev), the summed device time (ms), flops and
 * launch count.  Returns 0 or CD_ERR_CUDA. */
enum {
  CD_PROF_GEMM = 0,
  CD_PROF_REDUCE = 1,
  CD_PROF_SWEEP = 2,
  CD_PROF_TRINV = 3,
  CD_PROF_OTHER = 4,
  CD_PROF_SYMM = 5,
  CD_PROF_PANEL = 6,
  CD_PROF_NCLS = 7
};
void cd_profile_enable(int on);
void cd_profile_reset(void);
int cd_profile_read(int cls, double* ms, double* flops, int64_t* launches);

#ifdef __cplusplus
}
#endif
#endif /* CHOLDIFF_H */
