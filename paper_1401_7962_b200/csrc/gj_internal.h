// Internal declarations shared by the libgjinv translation units (not part of the C-ABI).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/gjinv.h"

namespace gj {

struct BatchedArgs {
  int n;
  int64_t batch;
  const void* A;
  void* Ainv;          // may be null (determinant-only)
  int32_t* ipiv;       // may be null
  double* logabsdet;   // may be null
  int8_t* sign;        // may be null
  void* det;           // may be null
  int32_t* info;       // may be null
  double tol;          // >= 0 (default already resolved)
};

// K1 launcher, n <= 32 (gj_batched.cu); K2 launcher, 32 < n <= 64 (gj_batched64.cu).
// Return cudaSuccess or the launch error.
cudaError_t launch_batched(gj_dtype dt, const BatchedArgs& a, cudaStream_t s);
cudaError_t launch_batched64(gj_dtype dt, const BatchedArgs& a, cudaStream_t s);
// K2e, fp64 n = 64 (gj_batched64e.cu: one warp per matrix, shared-memory resident, DMMA
// blocked update); cudaErrorNotSupported for a batch that is not 16-byte aligned.
cudaError_t launch_batched64e(const BatchedArgs& a, cudaStream_t s);
// K7, multi-RHS solve X = A^-1 B, n <= 32, m <= 32 (gj_solve.cu).
struct SolveArgs {
  int n, m;             // order, right-hand sides
  int64_t batch;
  const void* A;        // [batch][n][n]
  const void* B;        // [batch][n][m]
  void* X;              // [batch][n][m], may alias B
  int32_t* ipiv;        // may be null
  double* logabsdet;    // may be null
  int8_t* sign;         // may be null
  int32_t* info;        // may be null
  double tol;
};
cudaError_t launch_solve_batched(gj_dtype dt, const SolveArgs& a, cudaStream_t s);
// K1s (gj_batched.cu): fp32 n = 32, 1 <= m <= 8 on the blocked K1b elimination without the
// D half; cudaErrorNotSupported when it does not apply (then K7 runs)
cudaError_t launch_blk32_solve(const SolveArgs& a, cudaStream_t s);
// Large-n solve, fp64, one matrix (gj_large.cu): [A | B] with the det-only trailing update.
size_t large_solve_workspace_size(int n, int m);
size_t large_solve_workspace_size_f32(int n, int m);
cudaError_t solve_large_f32(int n, int m, const float* A, int64_t lda, const float* B, int64_t ldb, float* Xs,
                            int64_t ldx, int32_t* ipiv, double* logabsdet, int8_t* sign, int32_t* info, double tol,
                            void* ws, cudaStream_t s);
cudaError_t solve_large_f64(int n, int m, const double* A, int64_t lda, const double* B, int64_t ldb, double* Xs,
                            int64_t ldx, int32_t* ipiv, double* logabsdet, int8_t* sign, int32_t* info, double tol,
                            void* ws, cudaStream_t s);
// K6, n <= 32 (gj_fullpiv.cu): strategy 2 = full pivoting, 1 = partial, 0 = none; jpiv may be null.
cudaError_t launch_batched_strategy(gj_dtype dt, const BatchedArgs& a, int32_t* jpiv, int strategy, cudaStream_t s);

// K4b (gj_dgemm.cu): the K = 128 trailing update on the FP64 tensor pipe, TMA-fed and
// warp-specialised.  C[i][c] = (replace(i) ? 0 : C[i][c]) + sum_s X[i][a_col0 + s] RT[c][s]
// for i < M and the N compact columns c (c_base + nc, shifted past [skip_lo, skip_hi)).
struct DgemmArgs {
  const double* X;      // A = X[:, a_col0 .. a_col0 + K), row stride ldx; X is x_rows x x_cols
  int64_t ldx;
  int x_rows, x_cols, a_col0;
  const double* RT;     // B^T: RT[c][s], row stride K (= 128), rt_rows rows
  int rt_rows;
  double* C;            // row stride ldc, real column index
  int64_t ldc;
  int M, N, K;
  int c_base, skip_lo, skip_hi;
  const int* pivstep;   // replace(i) = pivstep[i] in [rep_lo, rep_hi)
  int rep_lo, rep_hi;
  // Tile-range weights: CTAs [0, late_from) take weight 1024 each, CTAs from late_from on
  // take late_w each (late_from >= the grid: uniform ranges).  The late CTAs are the ones
  // that only become resident when the panel kernel beside this launch frees its SMs.
  int late_from = 1 << 30, late_w = 1024;
};
bool dgemm_tma_supported(const DgemmArgs& g);
// cudaErrorNotSupported if the arguments do not suit it (the caller falls back to K4).
// grid_sms: CTAs (one per SM; 0: every SM); each takes a contiguous range of the tiles.
cudaError_t launch_dgemm_tma(const DgemmArgs& g, int grid_sms, bool pdl, cudaStream_t s);
#ifdef GJ_TIMELINE
// diagnostic builds only (%globaltimer ns): gj_large.cu keeps per panel k [0] leaf start,
// [1] leaf end; gj_dgemm.cu [0] trailing-update first CTA start, [1] its end, [2] its last CTA start
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#endif
#ifndef GJ_DGEMM_CW16_MAX_M
#define GJ_DGEMM_CW16_MAX_M 12288   // K4b: 16 consumer warps up to this many rows, 8 above
#endif

// Large-n blocked path (gj_large.cu), fp64, one matrix; Ainv may be null (det only).
size_t large_workspace_size(int n);
cudaError_t invert_large_f64(int n, const double* A, int64_t lda, double* Ainv, int64_t ldainv, int32_t* ipiv,
                             double* logabsdet, int8_t* sign, double* det, int32_t* info, double tol, void* ws,
                             cudaStream_t s);

// Large-n fp32 path (gj_large.cu) and its tcgen05 TF32 trailing update (gj_tcgemm.cu).
cudaError_t invert_large_f32(int n, const float* A, int64_t lda, float* Ainv, int64_t ldainv, int32_t* ipiv,
                             double* logabsdet, int8_t* sign, float* det, int32_t* info, double tol, void* ws,
                             cudaStream_t s);
size_t large_workspace_size_f32(int n);
struct TcUpdateArgs {
  const float* Ah;   // M x 128, K-major: the panel W split, high TF32 part
  const float* Al;   //                   low part
  const float* Bh;   // Nrows x 128, K-major: R transposed (B[c][s] = R[s][c]), high part
  const float* Bl;   //                   low part
  float* C;          // C[i][c], row stride ldc (absolute column index c)
  int64_t ldc;
  int M, N, Nrows;   // N: columns updated (the skipped range excluded); Nrows: rows of Bh / Bl
  const int* pivstep;
  int rep_lo, rep_hi;   // rows with pivstep in [rep_lo, rep_hi) are replaced, not added to
  int skip_lo, skip_hi; // columns [skip_lo, skip_hi) are not updated
};
cudaError_t launch_tc_update(const TcUpdateArgs& g, int grid_sms, bool pdl, cudaStream_t s);

// Distributed large-n steps (gj_large.cu; column-block-cyclic, block 128).
void dist_sizes(int n, int P, int rank, int* npad, int* nl, int* nl_real);
cudaError_t dist_init(int n, int P, int rank, const double* A_local, int64_t lda, double* Xl, int* pos, int* pivstep,
                      unsigned long long* smax, cudaStream_t s);
cudaError_t dist_factor(int n, int P, int rank, int k, double* Xl, int* pos, int* pivstep, double* rec_p, int* rec_q,
                        int* rec_row, double* W, cudaStream_t s);
cudaError_t dist_update(int n, int P, int rank, int k, int part, double* Xl, const double* W, const int* pivstep,
                        const int* rec_row, double* R, cudaStream_t s);
cudaError_t dist_finalize(int n, const double* rec_p, const int* rec_q, double tol, const unsigned long long* smax,
                          int32_t* ipiv, double* logabsdet, int8_t* sign, int32_t* info, cudaStream_t s);
cudaError_t dist_unpermute_plan(int n, int P, int rank, const int* pivstep, int* send_cols, int* recv_cols, int* counts,
                                cudaStream_t s);
cudaError_t dist_unpermute_pack(int n, int P, int rank, const double* Xl, const int* rec_row, const int* send_cols,
                                int m, double* sendbuf, cudaStream_t s);
cudaError_t dist_unpermute_unpack(int n, const double* recvbuf, const int* recv_cols, int m, double* Ainv_local,
                                  int64_t ld, cudaStream_t s);

// Number of SMs of the current device (cached per device).
int device_sm_count();
// Stream-ordered scratch allocation from a library-owned memory pool of the current device
// (free with cudaFreeAsync on the same stream); nullptr if unavailable.
void* pool_alloc_async(size_t bytes, cudaStream_t s);
// Bit of the current device: launch-time function attributes (dynamic shared memory,
// cluster size) are per device context, so "configured once" caches are per device.
inline unsigned long long device_bit() {
  int d = 0;
  cudaGetDevice(&d);
  return 1ull << (d & 63);
}

}  // namespace gj

#include <cuda.h>

namespace gj {
// Encode a 2-D tiled TMA descriptor (driver entry point fetched at run time, so the
// library does not link libcuda).  swizzle_bytes in {0, 32, 64, 128}.  Returns false
// if the driver entry point is unavailable or the encode fails.
bool make_tma_map_2d(CUtensorMap* m, bool f64, const void* base, uint64_t cols, uint64_t rows,
                     uint64_t row_stride_bytes, uint32_t box_cols, uint32_t box_rows, int swizzle_bytes);
}  // namespace gj
