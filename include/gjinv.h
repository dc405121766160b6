/*
 * gjinv.h — C-ABI of the B200-native Gauss–Jordan inversion library (libgjinv.so).
 *
 * The operation (arxiv 1401.7962, /root/reference/PAPER.md):
 *   Gauss–Jordan diagonalisation of the augmented system [A | I] -> [I | A^-1]
 *   (§2, Eqs. (1)-(2) L24-L28, row-operation form Eqs. (14)-(15) L61-L72, result
 *   Eq. (12)), with the pivot chosen as the max-|a_ik| candidate of column k
 *   (Obs. 3, L60; listing L151-L154), the swaps undone at the end ("depivotarea",
 *   Obs. 3 L60, listing L179-L198, §4), a pivot below a stated zero threshold
 *   flagging the matrix singular (Obs. 2, L59), and det A as the signed product of
 *   the pivots (Eq. (13); §4).
 *
 * Readings of the paper that fix the contract (DESIGN.md §3 lists all of them):
 *   - pivot candidates: rows not yet pivoted; ties -> smallest row index (G3);
 *   - zero threshold: RELATIVE — item is singular at the first step k whose largest
 *     candidate |a_rk| <= tol * max_ij |a_ij| (G1); tol = 0 flags exact zeros only;
 *     tol < 0 selects GJ_TOL_DEFAULT = n * eps(dtype);
 *   - det = (-1)^(#swaps) * prod(pivots) (G4 — Eq. (13) omits the swap sign);
 *   - ipiv: LAPACK-style 1-based swap sequence: at step k (1-based) the pivot row is
 *     the row then at position ipiv[k] of the physically-swapped matrix (the listing's
 *     p[k] = j, L154; reading G13).  Equal to LAPACK getrf's ipiv.
 *
 * Conventions for every entry point
 *   Ownership: the caller owns every buffer; the library never frees or keeps
 *     pointers.  Device entry points take DEVICE pointers and enqueue all work on
 *     `stream` (a cudaStream_t passed as void*, NULL = legacy default stream); they
 *     return as soon as the work is enqueued; outputs are valid once the caller
 *     synchronises that stream.  Host entry points (suffix _host) take HOST pointers
 *     and are synchronous.
 *   Layout: matrices are dense row-major, item b of a batch at offset b*n*n
 *     elements (contiguous batch), base addresses 16-byte aligned for the fastest
 *     path (any element-aligned address is accepted).
 *   Errors: the returned gj_status reports argument / launch / CUDA errors known at
 *     enqueue time.  Numerical singularity is per-item DATA in `info` and never
 *     aborts a batch: info[b] = 0 if item b is regular, else the first failing step
 *     k (1-based); for such items det = 0, sign = 0, logabsdet = -inf, and the
 *     inverse and ipiv contents are unspecified.
 *   Inputs containing NaN/Inf give unspecified results (not validated).
 *   Optional outputs: any output pointer documented "or NULL" may be NULL and is
 *     then not computed / written.
 *   Scratch memory: the fp32 n = 32 batched paths (gj_invert_batched, gj_solve_batched,
 *     gj_det) called with ipiv == NULL run two passes (K1f): a pass without
 *     the tie-break, then the exact kernel over the matrices in which it met an exact
 *     tie; the list of those (4 bytes per two matrices) is a stream-ordered allocation
 *     from a memory pool the library owns, freed on the same stream.  Outputs are
 *     bitwise those of the single exact pass.  Under stream capture, or if the pool
 *     allocation fails, the call runs the single exact pass instead.  A batch in which
 *     exact ties are common (e.g. small-integer matrices) runs up to ~1.3x slower this
 *     way; passing an ipiv buffer selects the single exact pass.
 */
#ifndef GJINV_H
#define GJINV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum { GJ_F32 = 0, GJ_F64 = 1 } gj_dtype;

typedef enum {
    GJ_OK = 0,
    GJ_ERR_ARG = 1,          /* invalid argument (NULL required pointer, n < 1, batch < 0, ...)  */
    GJ_ERR_UNSUPPORTED = 2,  /* (dtype, n) combination not supported by this entry point        */
    GJ_ERR_WORKSPACE = 3,    /* workspace too small                                             */
    GJ_ERR_CUDA = 4,         /* a CUDA runtime call or kernel launch failed                      */
    GJ_ERR_NCCL = 5          /* an NCCL call failed (distributed entry points)                   */
} gj_status;

#define GJ_TOL_DEFAULT (-1.0)  /* => tol = n * eps(dtype), relative to max|a_ij| of each matrix */

/* Largest n accepted by the batched (one matrix per warp / CTA) entry points. */
#define GJ_BATCHED_MAX_N 64

/*
 * gj_invert_batched — invert `batch` independent n x n matrices (1 <= n <= 64).
 *   dt         GJ_F32 or GJ_F64: element type of A, Ainv and det; the arithmetic is
 *              done in this type (logabsdet is accumulated in fp64 for both).
 *   n, batch   matrix order and item count (batch = 0 is a no-op).
 *   A          [batch][n][n] input, read only.
 *   Ainv       [batch][n][n] output A^-1 (Eq. (12)), may equal A (in place), or NULL
 *              (determinant-only run).
 *   ipiv       [batch][n] int32 1-based swap sequence, or NULL.
 *   logabsdet  [batch] fp64 log|det A| = sum_k log|p_k|, or NULL.
 *   sign       [batch] int8 in {-1, 0, +1}, or NULL.
 *   det        [batch] det A in dtype `dt` (may overflow to +-inf), or NULL.
 *   info       [batch] int32 singular flag (see above), or NULL.
 *   tol        relative zero threshold; < 0 selects GJ_TOL_DEFAULT.
 *   stream     cudaStream_t.
 * Returns GJ_OK, GJ_ERR_ARG, GJ_ERR_UNSUPPORTED (n > 64) or GJ_ERR_CUDA.
 */
gj_status gj_invert_batched(gj_dtype dt, int n, int64_t batch, const void* A, void* Ainv,
                            int32_t* ipiv, double* logabsdet, int8_t* sign, void* det,
                            int32_t* info, double tol, void* stream);

/*
 * gj_invert_batched_full — as gj_invert_batched with FULL pivoting:
 * Obs. 2-3 — the pivot of step k is the element of maximum |a_ij|
 * over all rows AND columns not yet pivoted (ties: the first in the row-major scan of the
 * physically swapped array, i.e. smallest row position, then smallest column position —
 * reading G23 of DESIGN.md), rows k <-> i and columns k <-> j are swapped, and the swaps
 * are undone at the end.  n <= GJ_FULLPIV_MAX_N (32); any batch.
 *   ipiv, jpiv  [batch][n] int32, 1-based row / column swap sequences (LAPACK getc2
 *               convention: at step k rows k and ipiv[k], columns k and jpiv[k]); may be NULL.
 *   sign        includes the parity of both swap sequences (det A = det(A Q) det Q).
 * Other arguments, layouts, ownership and errors exactly as gj_invert_batched
 * (Ainv NULL: determinants only).
 */
#define GJ_FULLPIV_MAX_N 32
gj_status gj_invert_batched_full(gj_dtype dt, int n, int64_t batch, const void* A, void* Ainv,
                                 int32_t* ipiv, int32_t* jpiv, double* logabsdet, int8_t* sign, void* det,
                                 int32_t* info, double tol, void* stream);

/*
 * gj_invert_batched_pivoting — the K6 kernel under a chosen pivoting strategy, for the
 * strategy / rounding-error comparison of the paper's §4 claim (Obs. 3
 * L60 "to reduce rounding errors"):
 *   GJ_PIVOT_NONE    (0)  pivot a_kk as in Eqs. (3)-(10) (L32-L46); info = first step with
 *                         |a_kk| <= tau (a zero pivot, Obs. 2 — not necessarily singular)
 *   GJ_PIVOT_PARTIAL (1)  the listing's row search in column k (L151-L162)
 *   GJ_PIVOT_FULL    (2)  as gj_invert_batched_full
 * Same arguments and outputs as gj_invert_batched_full (jpiv = 1..n for none/partial,
 * ipiv = 1..n for none).  n <= GJ_FULLPIV_MAX_N.  GJ_ERR_ARG for another strategy.
 * The production partial-pivoting path is gj_invert_batched (K1/K1b/K2); this entry exists
 * so that the three strategies run with identical arithmetic.
 */
#define GJ_PIVOT_NONE 0
#define GJ_PIVOT_PARTIAL 1
#define GJ_PIVOT_FULL 2
gj_status gj_invert_batched_pivoting(gj_dtype dt, int n, int64_t batch, const void* A, void* Ainv,
                                     int32_t* ipiv, int32_t* jpiv, double* logabsdet, int8_t* sign, void* det,
                                     int32_t* info, double tol, int strategy, void* stream);

/*
 * gj_solve_batched — X = A^-1 B for a batch of systems with nrhs right-hand sides by
 * Gauss–Jordan on the augmented [A | B] (Eq. (12) with B in place of the identity, the
 * elimination of Eqs. (14)-(15); the listing's partial pivoting, ties to
 * the smallest physical position, G3) — SURVEY.md §8f f4.  n <= GJ_SOLVE_MAX_N (32),
 * nrhs <= GJ_SOLVE_MAX_NRHS (32).
 *   A     [batch][n][n] row-major dt, read only.
 *   B     [batch][n][nrhs] row-major dt, read only (unless X aliases it).
 *   X     [batch][n][nrhs] row-major dt, written; may equal B (in place).
 *   ipiv, logabsdet, sign, info, tol, stream as gj_invert_batched (each output may be NULL);
 *   X of an item with info != 0 is unspecified.
 * Returns GJ_OK, GJ_ERR_ARG (null A/B/X, n < 1, nrhs < 1), GJ_ERR_UNSUPPORTED, GJ_ERR_CUDA.
 */
#define GJ_SOLVE_MAX_N 32
#define GJ_SOLVE_MAX_NRHS 32
gj_status gj_solve_batched(gj_dtype dt, int n, int nrhs, int64_t batch, const void* A, const void* B, void* X,
                           int32_t* ipiv, double* logabsdet, int8_t* sign, int32_t* info, double tol,
                           void* stream);

/*
 * gj_solve — X = A^-1 B for ONE system of any order n >= 1 with nrhs right-hand sides, by
 * Gauss–Jordan on [A | B] (Eq. (12) with B for I; Eqs. (14)-(15)) — SURVEY.md §8f f4.
 * n <= 32 and nrhs <= 32 with dense rows (lda == n, ldb == ldx == nrhs): the batched K7
 * kernel (batch 1).  Otherwise the blocked large-n path on the working array [A | B] —
 * gj_invert's panels and pivots (FP64 DMMA updates for GJ_F64, tcgen05 3xTF32 for GJ_F32),
 * with each panel's trailing update restricted to the columns right of the next panel (the
 * rest of A and all of B): ~2/3 n^3 + 2 n^2 nrhs.
 *   A, lda   input (row stride lda >= n), read only.
 *   B, ldb   right-hand sides, n x nrhs (row stride ldb >= nrhs), read only.
 *   X, ldx   solution, n x nrhs (row stride ldx >= nrhs); must not overlap A or B on the
 *            large path (may equal B on the batched path).
 *   ipiv, logabsdet, sign, info, tol  as gj_invert (each output may be NULL).
 *   workspace  device buffer of gj_solve_workspace_size(dt, n, nrhs) bytes (0: may be NULL).
 * Returns GJ_OK, GJ_ERR_ARG, GJ_ERR_UNSUPPORTED (a strided system within the batched
 * limits), GJ_ERR_WORKSPACE or GJ_ERR_CUDA.
 */
gj_status gj_solve(gj_dtype dt, int n, int nrhs, const void* A, int64_t lda, const void* B, int64_t ldb, void* X,
                   int64_t ldx, int32_t* ipiv, double* logabsdet, int8_t* sign, int32_t* info, double tol,
                   void* workspace, size_t workspace_bytes, void* stream);
/* Workspace bytes for gj_solve (0 when the batched kernel serves the call). */
size_t gj_solve_workspace_size(gj_dtype dt, int n, int nrhs);

/*
 * gj_det — determinants only (Eq. (13); §4 "without laborious extra computation"):
 * the same elimination as gj_invert_batched without storing A^-1.
 * Arguments as gj_invert_batched; `workspace`/`workspace_bytes` are used for n > 64
 * (batch must then be 1; size from gj_workspace_size(dt, n, 1, 2)), else may be NULL/0.
 */
gj_status gj_det(gj_dtype dt, int n, int64_t batch, const void* A, double* logabsdet,
                 int8_t* sign, void* det, int32_t* ipiv, int32_t* info, double tol,
                 void* workspace, size_t workspace_bytes, void* stream);

/*
 * gj_invert — one n x n matrix, 1 <= n <= GJ_LARGE_MAX_N (n <= 64 uses the batched kernels; larger n
 * the blocked Gauss–Jordan: panel factorisation + tensor-core trailing updates, the
 * aggregated form of Eqs. (14)-(15): FP64 DMMA for GJ_F64; for GJ_F32 tcgen05.mma
 * kind::tf32 with the accumulator in TMEM and a 3xTF32 split for fp32 accuracy).
 *   A, lda       input (row stride lda >= n elements), read only.
 *   Ainv, ldainv output (row stride ldainv >= n); may equal A when lda == ldainv.
 *   ipiv, logabsdet, sign, info  as gj_invert_batched with batch = 1 (each may be NULL).
 *   workspace    device buffer of at least gj_workspace_size(dt, n, 1, 1) bytes (may be
 *                NULL when that size is 0).
 */
#define GJ_LARGE_MAX_N 65536   /* rows of one thread-block cluster's panel kernel (16 CTAs x 512 threads x 8) */
gj_status gj_invert(gj_dtype dt, int n, const void* A, int64_t lda, void* Ainv, int64_t ldainv,
                    int32_t* ipiv, double* logabsdet, int8_t* sign, int32_t* info, double tol,
                    void* workspace, size_t workspace_bytes, void* stream);

/* Workspace bytes for entry 0 = gj_invert_batched (always 0), 1 = gj_invert, 2 = gj_det. */
size_t gj_workspace_size(gj_dtype dt, int n, int64_t batch, int entry);

/*
 * gj_invert_batched_host — gj_invert_batched on HOST buffers (synchronous).  The library
 * stages `chunk` items at a time (chunk <= 0: automatic, 128 MiB) through four device
 * buffers and pipelines host->device copy, inversion and device->host copy of consecutive
 * chunks on its own streams.  Pinned (page-locked) host buffers give overlapped copies;
 * pageable buffers work but copy synchronously.  Ainv must not alias A.  The streams and
 * staging buffers are kept per device between calls (grown when a call needs more) and
 * freed by gj_host_release(); concurrent calls on one device are serialised.
 * Returns as gj_invert_batched.
 */
gj_status gj_invert_batched_host(gj_dtype dt, int n, int64_t batch, const void* A_host,
                                 void* Ainv_host, int32_t* ipiv_host, double* logabsdet_host,
                                 int8_t* sign_host, void* det_host, int32_t* info_host,
                                 double tol, int64_t chunk);
/* Frees the device staging buffers and streams gj_invert_batched_host keeps (all devices). */
gj_status gj_host_release(void);

/*
 * ---------------------------------------------------------------------------------------
 * Distributed large-n inversion (fp64, n > 64) over P ranks, one GPU each: the building
 * blocks of the column-block-cyclic Gauss–Jordan.  The global matrix is
 * padded with an identity block to npad = ceil(n / GJ_DIST_BLOCK) * GJ_DIST_BLOCK;
 * global column block j (GJ_DIST_BLOCK columns) lives on rank j % P.  Rows are complete
 * on every rank, so the pivot search of a panel (the max-|a_ik| rule, Obs. 3 L60) is
 * local to the panel's owner.  The collectives are the caller's (NCCL via
 * torch.distributed in paper_1401_7962_b200/dist.py): per panel k the owner calls
 * gj_dist_step_factor, broadcasts W, pos, pivstep and the record of steps [k*B, (k+1)*B),
 * then every rank calls gj_dist_step_update; the un-permutation (listing L179-L198) is one
 * all-to-all of columns planned by gj_dist_step_unpermute_plan.  Same pivots, det and
 * inverse as gj_invert (the aggregation of Eqs. (14)-(15), L61-L72, is identical).
 * All pointers are DEVICE pointers owned by the caller; work is enqueued on `stream`.
 * Replicated arrays (length npad, int32 unless stated): pos (physical position of each
 * row in the listing's swapped array), pivstep (step at which a row was pivot, -1 if
 * not yet), rec_p (fp64 pivot per step), rec_q (pivot position per step), rec_row
 * (pivot row per step).  X_local is npad x ncols_local row-major (this rank's padded
 * columns in increasing global order), W is npad x GJ_DIST_BLOCK, R GJ_DIST_BLOCK x
 * ncols_local.  Errors: GJ_ERR_ARG for bad sizes / ranks / NULL, GJ_ERR_CUDA on launch
 * failure.
 * ---------------------------------------------------------------------------------------
 */
#define GJ_DIST_BLOCK 128
#define GJ_DIST_MAX_RANKS 8

/* npad, this rank's padded column count and how many of them are real (< n). */
gj_status gj_dist_sizes(int n, int nranks, int rank, int* npad, int* ncols_local, int* ncols_local_real);

/* X_local = this rank's columns of blockdiag(A, I); A_local holds the rank's ncols_local_real
 * real columns (n rows, row stride lda >= ncols_local_real).  pos/pivstep initialised;
 * *smax_bits = bit pattern of max |a_ij| over the local columns (reduce MAX over ranks
 * before gj_dist_step_finalize: the zero threshold of Obs. 2, L59, is relative to it, G1). */
gj_status gj_dist_step_init(int n, int nranks, int rank, const double* A_local, int64_t lda, double* X_local,
                       int32_t* pos, int32_t* pivstep, uint64_t* smax_bits, void* stream);

/* Owner of panel k (k % nranks == rank) only: GJ_DIST_BLOCK pivot steps (a2-a6) on the
 * panel's local columns, in place, updating pos / pivstep / rec_* and copying the
 * factored panel to W. */
gj_status gj_dist_step_factor(int n, int nranks, int rank, int k, double* X_local, int32_t* pos, int32_t* pivstep,
                         double* rec_p, int32_t* rec_q, int32_t* rec_row, double* W, void* stream);

/* Every rank, after the broadcast of panel k: X_local[:, c] += (W - S) R for the local
 * columns c outside panel k (R = the panel's pivot rows of X_local, staged in R).
 *   part 0: all of them (gathers R first);
 *   part 1: only the local columns of panel k+1 (gathers R first; the rank must own k+1);
 *   part 2: the rest, after part 1 and gj_dist_step_factor(k+1) on the same stream: launched as
 *           a programmatic dependent of that factorisation so the two overlap (look-ahead).
 * Parts 1 and 2 need (k+1) % nranks == rank. */
gj_status gj_dist_step_update(int n, int nranks, int rank, int k, int part, double* X_local, const double* W,
                         const int32_t* pivstep, const int32_t* rec_row, double* R, void* stream);

/* log|det|, sign, info and ipiv from the replicated record (Eq. (13) + G4); tol as
 * gj_invert (< 0: n * eps). Any rank; outputs may be NULL. */
gj_status gj_dist_step_finalize(int n, const double* rec_p, const int32_t* rec_q, double tol, const uint64_t* smax_bits,
                           int32_t* ipiv, double* logabsdet, int8_t* sign, int32_t* info, void* stream);

/* Un-permutation plan: send_cols (<= ncols_local) = local compact columns ordered by
 * (destination rank, output column); recv_cols = local output columns ordered by
 * (source rank, output column); counts[0..P) columns sent to / counts[P..2P) received
 * from each rank. nranks <= GJ_DIST_MAX_RANKS. */
gj_status gj_dist_step_unpermute_plan(int n, int nranks, int rank, const int32_t* pivstep, int32_t* send_cols,
                                 int32_t* recv_cols, int32_t* counts, void* stream);

/* sendbuf[t][i] = X_local[rec_row[i]][send_cols[t]], t < m, i < n (m columns of n). */
gj_status gj_dist_step_unpermute_pack(int n, int nranks, int rank, const double* X_local, const int32_t* rec_row,
                                 const int32_t* send_cols, int m, double* sendbuf, void* stream);

/* Ainv_local[i][recv_cols[t]] = recvbuf[t][i]: Ainv_local is n x (this rank's real output
 * columns, in increasing global order) with row stride ld. */
gj_status gj_dist_step_unpermute_unpack(int n, const double* recvbuf, const int32_t* recv_cols, int m, double* Ainv_local,
                                   int64_t ld, void* stream);

/*
 * ---------------------------------------------------------------------------------------
 * Distributed large-n inversion, library-driven: the same column-block-cyclic method as the
 * step functions above (Eqs. (14)-(15) aggregated over 128-column panels, PAPER.md L61-L72;
 * the max-|a_ik| pivot search of Obs. 3, L60, local to each panel's owner; the
 * un-permutation of the listing, L179-L198, as one all-to-all of columns), with the library
 * owning the NCCL communicator and driving the per-panel exchange itself:
 *   per panel k: the owner factors it; W (npad x 128 fp64) and the replicated state
 *   (pos | pivstep | rec_q | rec_row | rec_p, 6 npad int32) are broadcast from the owner with
 *   ncclBroadcast on an internal side stream, double-buffered by panel parity, while panel
 *   k-1's update still runs (look-ahead: the owner of k+1 updates and factors k+1 first);
 *   every rank applies the update to its local columns (K4b DMMA GEMM);
 *   then ncclAllReduce (max) of max|a_ij| for the threshold, and grouped ncclSend/ncclRecv
 *   for the un-permutation.
 * NCCL is loaded at run time (dlopen "libnccl.so.2"; the copy torch loaded is reused), so
 * the library has no link-time NCCL dependency; without it these return GJ_ERR_NCCL.
 * ---------------------------------------------------------------------------------------
 */
typedef struct gj_dist_ctx* gj_dist_handle;
#define GJ_DIST_UNIQUE_ID_BYTES 128

/* A new NCCL unique id (rank 0 calls it and shares the 128 bytes with every rank out of
 * band).  Returns GJ_OK or GJ_ERR_NCCL. */
gj_status gj_dist_get_unique_id(unsigned char unique_id[GJ_DIST_UNIQUE_ID_BYTES]);

/* Collective over the nranks processes (one GPU each, `device` = this rank's CUDA device):
 * creates the communicator (ncclCommInitRank) and the internal stream / events.  *handle is
 * owned by the caller until gj_dist_finalize.  Returns GJ_OK, GJ_ERR_ARG (nranks outside
 * 1..GJ_DIST_MAX_RANKS, rank outside 0..nranks-1, NULL), GJ_ERR_CUDA or GJ_ERR_NCCL. */
gj_status gj_dist_init(int nranks, int rank, const unsigned char unique_id[GJ_DIST_UNIQUE_ID_BYTES], int device,
                       gj_dist_handle* handle);

/* Collective: every rank calls it with the same n (> 64) and tol.  A_local: this rank's real
 * columns of A (gj_dist_sizes' ncols_local_real of them, the global columns c with
 * (c / GJ_DIST_BLOCK) % nranks == rank, increasing), n rows, row stride lda; Ainv_local: the
 * same columns of A^-1, row stride ldainv (may not alias A_local).  ipiv [n], logabsdet,
 * sign, info: replicated outputs on every rank (any may be NULL).  All DEVICE pointers on
 * the handle's device; the work is enqueued on `stream`, and the call returns after one host
 * synchronisation of it (the all-to-all sizes depend on the pivots) with the un-permutation
 * enqueued.  The device workspace (~(npad x local columns + 3 npad x 128) doubles) is kept in the
 * handle between calls and freed by gj_dist_finalize.
 * Returns GJ_OK, GJ_ERR_ARG, GJ_ERR_CUDA or GJ_ERR_NCCL; a singular matrix is data (info). */
gj_status gj_invert_dist(gj_dist_handle handle, int n, const double* A_local, int64_t lda, double* Ainv_local,
                         int64_t ldainv, int32_t* ipiv, double* logabsdet, int8_t* sign, int32_t* info, double tol,
                         void* stream);

/* Destroys the communicator and the handle (collective).  NULL is a no-op. */
gj_status gj_dist_finalize(gj_dist_handle handle);

/* Static description of a status code. */
const char* gj_status_string(gj_status s);

/* Library version, e.g. "gjinv 0.1.0 sm_100a". */
const char* gj_version(void);

#ifdef __cplusplus
}
#endif

#endif /* GJINV_H */
