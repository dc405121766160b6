// libgjinv C-ABI (include/gjinv.h): argument validation, dispatch on (dtype, n),
// stream handling and the host-buffer pipeline.  No compute happens here: every step
// of the method runs in the kernels of gj_batched.cu / gj_large.cu.
#include <cuda_runtime.h>
#include <mutex>
#include <cstdio>
#include <cstring>
#include <vector>

#include "gj_internal.h"

namespace gj {

int device_sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (dev < 0 || dev >= 64) return 148;
  if (cached[dev] == 0) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    cached[dev] = v;
  }
  return cached[dev];
}

void* pool_alloc_async(size_t bytes, cudaStream_t s) {
  // one library-owned pool per device, keeping its memory between calls (release threshold
  // = max), so that a per-call scratch buffer costs no device allocation after the first.
  // Not under stream capture: an allocation from a user pool there may fail and invalidate
  // the caller's capture, so a captured call takes the single-pass path instead.
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    return nullptr;
  }
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  cudaMemPool_t pool;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (pools[dev] == nullptr) {
      cudaMemPoolProps props = {};
      props.allocType = cudaMemAllocationTypePinned;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = dev;
      cudaMemPool_t p = nullptr;
      if (cudaMemPoolCreate(&p, &props) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
      }
      uint64_t keep = ~0ull;
      cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &keep);
      pools[dev] = p;
    }
    pool = pools[dev];
  }
  void* ptr = nullptr;
  if (cudaMallocFromPoolAsync(&ptr, bytes, pool, s) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return ptr;
}

static double resolve_tol(gj_dtype dt, int n, double tol) {
  if (tol >= 0.0) return tol;
  const double eps = dt == GJ_F32 ? 1.1920928955078125e-07 : 2.220446049250313e-16;
  return n * eps;
}

static size_t esize(gj_dtype dt) { return dt == GJ_F32 ? 4 : 8; }

}  // namespace gj

using namespace gj;

namespace {
// Per-device state of gj_invert_batched_host (kept between calls; gj_host_release frees it).
struct HostCtx {
  static constexpr int NB = 4;
  struct Buf {
    void* p[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};   // X, ipiv, lg, sign, det, info
    size_t cap[6] = {0, 0, 0, 0, 0, 0};
    cudaEvent_t h = nullptr, k = nullptr, d = nullptr;
  } b[NB];
  cudaStream_t sH = nullptr, sK = nullptr, sD = nullptr;
  bool ready = false;
  std::mutex mu;
};
constexpr int kMaxDev = 64;
HostCtx g_host[kMaxDev];
HostCtx& host_ctx() {
  int d = 0;
  cudaGetDevice(&d);
  return g_host[(d >= 0 && d < kMaxDev) ? d : 0];
}
}  // namespace

extern "C" {

const char* gj_status_string(gj_status s) {
  switch (s) {
    case GJ_OK: return "GJ_OK";
    case GJ_ERR_ARG: return "GJ_ERR_ARG: invalid argument";
    case GJ_ERR_UNSUPPORTED: return "GJ_ERR_UNSUPPORTED: (dtype, n) not supported by this entry point";
    case GJ_ERR_WORKSPACE: return "GJ_ERR_WORKSPACE: workspace too small";
    case GJ_ERR_CUDA: return "GJ_ERR_CUDA: CUDA runtime / launch failure";
    case GJ_ERR_NCCL: return "GJ_ERR_NCCL: NCCL failure";
  }
  return "unknown gj_status";
}

const char* gj_version(void) { return "gjinv 0.1.0 sm_100a"; }

gj_status gj_invert_batched(gj_dtype dt, int n, int64_t batch, const void* A, void* Ainv,
                            int32_t* ipiv, double* logabsdet, int8_t* sign, void* det,
                            int32_t* info, double tol, void* stream) {
  if (dt != GJ_F32 && dt != GJ_F64) return GJ_ERR_ARG;
  if (n < 1 || batch < 0) return GJ_ERR_ARG;
  if (batch == 0) return GJ_OK;
  if (A == nullptr) return GJ_ERR_ARG;
  if (n > GJ_BATCHED_MAX_N) return GJ_ERR_UNSUPPORTED;
  BatchedArgs a{n, batch, A, Ainv, ipiv, logabsdet, sign, det, info, resolve_tol(dt, n, tol)};
  cudaError_t e = n <= 32 ? launch_batched(dt, a, static_cast<cudaStream_t>(stream))
                          : launch_batched64(dt, a, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? GJ_OK : GJ_ERR_CUDA;
}

gj_status gj_invert_batched_pivoting(gj_dtype dt, int n, int64_t batch, const void* A, void* Ainv,
                                     int32_t* ipiv, int32_t* jpiv, double* logabsdet, int8_t* sign, void* det,
                                     int32_t* info, double tol, int strategy, void* stream) {
  if (dt != GJ_F32 && dt != GJ_F64) return GJ_ERR_ARG;
  if (n < 1 || batch < 0) return GJ_ERR_ARG;
  if (strategy != GJ_PIVOT_NONE && strategy != GJ_PIVOT_PARTIAL && strategy != GJ_PIVOT_FULL) return GJ_ERR_ARG;
  if (batch == 0) return GJ_OK;
  if (A == nullptr) return GJ_ERR_ARG;
  if (n > GJ_FULLPIV_MAX_N) return GJ_ERR_UNSUPPORTED;
  BatchedArgs a{n, batch, A, Ainv, ipiv, logabsdet, sign, det, info, resolve_tol(dt, n, tol)};
  cudaError_t e = launch_batched_strategy(dt, a, jpiv, strategy, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? GJ_OK : GJ_ERR_CUDA;
}

gj_status gj_solve_batched(gj_dtype dt, int n, int nrhs, int64_t batch, const void* A, const void* B, void* X,
                           int32_t* ipiv, double* logabsdet, int8_t* sign, int32_t* info, double tol,
                           void* stream) {
  if (dt != GJ_F32 && dt != GJ_F64) return GJ_ERR_ARG;
  if (n < 1 || nrhs < 1 || batch < 0) return GJ_ERR_ARG;
  if (batch == 0) return GJ_OK;
  if (A == nullptr || B == nullptr || X == nullptr) return GJ_ERR_ARG;
  if (n > GJ_SOLVE_MAX_N || nrhs > GJ_SOLVE_MAX_NRHS) return GJ_ERR_UNSUPPORTED;
  SolveArgs a{n, nrhs, batch, A, B, X, ipiv, logabsdet, sign, info, resolve_tol(dt, n, tol)};
  cudaError_t e = launch_solve_batched(dt, a, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? GJ_OK : GJ_ERR_CUDA;
}

size_t gj_solve_workspace_size(gj_dtype dt, int n, int nrhs) {
  if (n < 1 || nrhs < 1) return 0;
  if (n <= GJ_SOLVE_MAX_N && nrhs <= GJ_SOLVE_MAX_NRHS) return 0;
  return dt == GJ_F64 ? large_solve_workspace_size(n, nrhs) : large_solve_workspace_size_f32(n, nrhs);
}

gj_status gj_solve(gj_dtype dt, int n, int nrhs, const void* A, int64_t lda, const void* B, int64_t ldb, void* X,
                   int64_t ldx, int32_t* ipiv, double* logabsdet, int8_t* sign, int32_t* info, double tol,
                   void* workspace, size_t workspace_bytes, void* stream) {
  if (dt != GJ_F32 && dt != GJ_F64) return GJ_ERR_ARG;
  if (n < 1 || nrhs < 1 || A == nullptr || B == nullptr || X == nullptr) return GJ_ERR_ARG;
  if (lda < n || ldb < nrhs || ldx < nrhs) return GJ_ERR_ARG;
  if (n <= GJ_SOLVE_MAX_N && nrhs <= GJ_SOLVE_MAX_NRHS) {
    if (lda != n || ldb != nrhs || ldx != nrhs) return GJ_ERR_UNSUPPORTED;   // the batched kernel is dense
    return gj_solve_batched(dt, n, nrhs, 1, A, B, X, ipiv, logabsdet, sign, info, tol, stream);
  }
  if (n > GJ_LARGE_MAX_N) return GJ_ERR_UNSUPPORTED;
  if (workspace == nullptr || workspace_bytes < gj_solve_workspace_size(dt, n, nrhs)) return GJ_ERR_WORKSPACE;
  cudaError_t e = dt == GJ_F64
      ? solve_large_f64(n, nrhs, static_cast<const double*>(A), lda, static_cast<const double*>(B), ldb,
                        static_cast<double*>(X), ldx, ipiv, logabsdet, sign, info, resolve_tol(dt, n, tol), workspace,
                        static_cast<cudaStream_t>(stream))
      : solve_large_f32(n, nrhs, static_cast<const float*>(A), lda, static_cast<const float*>(B), ldb,
                        static_cast<float*>(X), ldx, ipiv, logabsdet, sign, info, resolve_tol(dt, n, tol), workspace,
                        static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? GJ_OK : GJ_ERR_CUDA;
}

gj_status gj_invert_batched_full(gj_dtype dt, int n, int64_t batch, const void* A, void* Ainv,
                                 int32_t* ipiv, int32_t* jpiv, double* logabsdet, int8_t* sign, void* det,
                                 int32_t* info, double tol, void* stream) {
  return gj_invert_batched_pivoting(dt, n, batch, A, Ainv, ipiv, jpiv, logabsdet, sign, det, info, tol,
                                    GJ_PIVOT_FULL, stream);
}

size_t gj_workspace_size(gj_dtype dt, int n, int64_t batch, int entry) {
  (void)batch;
  if (n < 1) return 0;
  if (n > GJ_BATCHED_MAX_N && (entry == 1 || entry == 2))
    return dt == GJ_F64 ? large_workspace_size(n) : large_workspace_size_f32(n);
  if (entry == 1) return (size_t)n * n * esize(dt);  // lda != n repack
  return 0;
}

gj_status gj_det(gj_dtype dt, int n, int64_t batch, const void* A, double* logabsdet,
                 int8_t* sign, void* det, int32_t* ipiv, int32_t* info, double tol,
                 void* workspace, size_t workspace_bytes, void* stream) {
  if (n > GJ_BATCHED_MAX_N) {
    if ((dt != GJ_F64 && dt != GJ_F32) || batch != 1 || A == nullptr) return batch == 0 ? GJ_OK : GJ_ERR_UNSUPPORTED;
    if (n > GJ_LARGE_MAX_N) return GJ_ERR_UNSUPPORTED;
    if (workspace == nullptr || workspace_bytes < gj_workspace_size(dt, n, 1, 2)) return GJ_ERR_WORKSPACE;
    cudaError_t e = dt == GJ_F64
        ? invert_large_f64(n, static_cast<const double*>(A), n, nullptr, 0, ipiv, logabsdet, sign,
                           static_cast<double*>(det), info, resolve_tol(dt, n, tol), workspace,
                           static_cast<cudaStream_t>(stream))
        : invert_large_f32(n, static_cast<const float*>(A), n, nullptr, 0, ipiv, logabsdet, sign,
                           static_cast<float*>(det), info, resolve_tol(dt, n, tol), workspace,
                           static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? GJ_OK : GJ_ERR_CUDA;
  }
  return gj_invert_batched(dt, n, batch, A, nullptr, ipiv, logabsdet, sign, det, info, tol, stream);
}

gj_status gj_invert(gj_dtype dt, int n, const void* A, int64_t lda, void* Ainv, int64_t ldainv,
                    int32_t* ipiv, double* logabsdet, int8_t* sign, int32_t* info, double tol,
                    void* workspace, size_t workspace_bytes, void* stream) {
  if (dt != GJ_F32 && dt != GJ_F64) return GJ_ERR_ARG;
  if (n < 1 || A == nullptr || Ainv == nullptr || lda < n || ldainv < n) return GJ_ERR_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t es = esize(dt);
  if (n > GJ_BATCHED_MAX_N) {
    if (n > GJ_LARGE_MAX_N) return GJ_ERR_UNSUPPORTED;
    if (workspace == nullptr || workspace_bytes < gj_workspace_size(dt, n, 1, 1)) return GJ_ERR_WORKSPACE;
    cudaError_t e = dt == GJ_F64
        ? invert_large_f64(n, static_cast<const double*>(A), lda, static_cast<double*>(Ainv), ldainv, ipiv,
                           logabsdet, sign, nullptr, info, resolve_tol(dt, n, tol), workspace, s)
        // fp32: the tcgen05 TF32 (3xTF32) trailing update
        : invert_large_f32(n, static_cast<const float*>(A), lda, static_cast<float*>(Ainv), ldainv, ipiv,
                           logabsdet, sign, nullptr, info, resolve_tol(dt, n, tol), workspace, s);
    return e == cudaSuccess ? GJ_OK : GJ_ERR_CUDA;
  }
  if (lda == n && ldainv == n)
    return gj_invert_batched(dt, n, 1, A, Ainv, ipiv, logabsdet, sign, nullptr, info, tol, stream);
  // strided: repack into the workspace, invert in place, unpack
  if (workspace == nullptr || workspace_bytes < (size_t)n * n * es) return GJ_ERR_WORKSPACE;
  if (cudaMemcpy2DAsync(workspace, n * es, A, lda * es, n * es, n, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
    return GJ_ERR_CUDA;
  gj_status st = gj_invert_batched(dt, n, 1, workspace, workspace, ipiv, logabsdet, sign, nullptr, info, tol, stream);
  if (st != GJ_OK) return st;
  if (cudaMemcpy2DAsync(Ainv, ldainv * es, workspace, n * es, n * es, n, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
    return GJ_ERR_CUDA;
  return GJ_OK;
}

gj_status gj_invert_batched_host(gj_dtype dt, int n, int64_t batch, const void* A_host,
                                 void* Ainv_host, int32_t* ipiv_host, double* logabsdet_host,
                                 int8_t* sign_host, void* det_host, int32_t* info_host,
                                 double tol, int64_t chunk) {
  if (dt != GJ_F32 && dt != GJ_F64) return GJ_ERR_ARG;
  if (n < 1 || batch < 0 || A_host == nullptr) return GJ_ERR_ARG;
  if (n > GJ_BATCHED_MAX_N) return GJ_ERR_UNSUPPORTED;
  if (batch == 0) return GJ_OK;
  if (Ainv_host == A_host) return GJ_ERR_ARG;
  const size_t es = esize(dt);
  const size_t mat = (size_t)n * n * es;
  if (chunk <= 0) {
    chunk = (int64_t)((128u << 20) / mat);   // 128 MiB per chunk (measured best on C2)
    if (chunk < 1) chunk = 1;
  }
  if (chunk > batch) chunk = batch;
  // NB device buffers cycling through three streams — host->device copies, kernels,
  // device->host copies — ordered by events, so both copy directions and the kernels run
  // back to back on their own engines (PCIe is full duplex).  Streams, events and buffers
  // are kept per device between calls (cudaMalloc / cudaFree per call cost tens of ms and
  // made the end-to-end time erratic); gj_host_release() frees them.
  HostCtx& C = host_ctx();
  std::lock_guard<std::mutex> lock(C.mu);
  gj_status st = GJ_OK;
  auto ck = [&](cudaError_t e) { if (e != cudaSuccess && st == GJ_OK) st = GJ_ERR_CUDA; return e == cudaSuccess; };
  if (!C.ready) {
    ck(cudaStreamCreateWithFlags(&C.sH, cudaStreamNonBlocking));
    ck(cudaStreamCreateWithFlags(&C.sK, cudaStreamNonBlocking));
    ck(cudaStreamCreateWithFlags(&C.sD, cudaStreamNonBlocking));
    for (int i = 0; i < HostCtx::NB; ++i) {
      ck(cudaEventCreateWithFlags(&C.b[i].h, cudaEventDisableTiming));
      ck(cudaEventCreateWithFlags(&C.b[i].k, cudaEventDisableTiming));
      ck(cudaEventCreateWithFlags(&C.b[i].d, cudaEventDisableTiming));
    }
    if (st != GJ_OK) return st;
    C.ready = true;
  }
  const size_t need[6] = {mat * chunk, ipiv_host ? sizeof(int32_t) * n * chunk : 0, logabsdet_host ? sizeof(double) * chunk : 0,
                          sign_host ? (size_t)chunk : 0, det_host ? es * chunk : 0, info_host ? sizeof(int32_t) * chunk : 0};
  for (int i = 0; i < HostCtx::NB && st == GJ_OK; ++i)
    for (int f = 0; f < 6; ++f)
      if (need[f] > C.b[i].cap[f]) {
        if (C.b[i].p[f]) ck(cudaFree(C.b[i].p[f]));
        C.b[i].p[f] = nullptr;
        C.b[i].cap[f] = 0;
        if (ck(cudaMalloc(&C.b[i].p[f], need[f]))) C.b[i].cap[f] = need[f];
      }
  if (st != GJ_OK) return st;
  const char* Ah = static_cast<const char*>(A_host);
  char* Xh = static_cast<char*>(Ainv_host);
  for (int64_t c0 = 0, ci = 0; c0 < batch && st == GJ_OK; c0 += chunk, ++ci) {
    HostCtx::Buf& B = C.b[ci % HostCtx::NB];
    void* X = B.p[0];
    int32_t* ipiv = ipiv_host ? static_cast<int32_t*>(B.p[1]) : nullptr;
    double* lg = logabsdet_host ? static_cast<double*>(B.p[2]) : nullptr;
    int8_t* sg = sign_host ? static_cast<int8_t*>(B.p[3]) : nullptr;
    void* det = det_host ? B.p[4] : nullptr;
    int32_t* info = info_host ? static_cast<int32_t*>(B.p[5]) : nullptr;
    const int64_t m = (batch - c0) < chunk ? (batch - c0) : chunk;
    if (ci >= HostCtx::NB) ck(cudaStreamWaitEvent(C.sH, B.d, 0));   // the buffer's previous results are out
    ck(cudaMemcpyAsync(X, Ah + c0 * mat, m * mat, cudaMemcpyHostToDevice, C.sH));
    ck(cudaEventRecord(B.h, C.sH));
    ck(cudaStreamWaitEvent(C.sK, B.h, 0));
    gj_status k = gj_invert_batched(dt, n, m, X, Xh ? X : nullptr, ipiv, lg, sg, det, info, tol, C.sK);
    if (k != GJ_OK && st == GJ_OK) st = k;
    ck(cudaEventRecord(B.k, C.sK));
    ck(cudaStreamWaitEvent(C.sD, B.k, 0));
    if (Xh) ck(cudaMemcpyAsync(Xh + c0 * mat, X, m * mat, cudaMemcpyDeviceToHost, C.sD));
    if (ipiv) ck(cudaMemcpyAsync(ipiv_host + c0 * n, ipiv, sizeof(int32_t) * n * m, cudaMemcpyDeviceToHost, C.sD));
    if (lg) ck(cudaMemcpyAsync(logabsdet_host + c0, lg, sizeof(double) * m, cudaMemcpyDeviceToHost, C.sD));
    if (sg) ck(cudaMemcpyAsync(sign_host + c0, sg, m, cudaMemcpyDeviceToHost, C.sD));
    if (det) ck(cudaMemcpyAsync(static_cast<char*>(det_host) + c0 * es, det, es * m, cudaMemcpyDeviceToHost, C.sD));
    if (info) ck(cudaMemcpyAsync(info_host + c0, info, sizeof(int32_t) * m, cudaMemcpyDeviceToHost, C.sD));
    ck(cudaEventRecord(B.d, C.sD));
  }
  for (cudaStream_t x : {C.sH, C.sK, C.sD}) ck(cudaStreamSynchronize(x));
  return st;
}

gj_status gj_host_release(void) {
  gj_status st = GJ_OK;
  for (int d = 0; d < kMaxDev; ++d) {
    HostCtx& C = g_host[d];
    std::lock_guard<std::mutex> lock(C.mu);
    if (!C.ready) continue;
    int cur = 0;
    cudaGetDevice(&cur);
    if (cudaSetDevice(d) != cudaSuccess) { st = GJ_ERR_CUDA; continue; }
    for (cudaStream_t x : {C.sH, C.sK, C.sD}) cudaStreamSynchronize(x);
    for (int i = 0; i < HostCtx::NB; ++i) {
      for (int f = 0; f < 6; ++f) {
        if (C.b[i].p[f]) cudaFree(C.b[i].p[f]);
        C.b[i].p[f] = nullptr;
        C.b[i].cap[f] = 0;
      }
      cudaEventDestroy(C.b[i].h);
      cudaEventDestroy(C.b[i].k);
      cudaEventDestroy(C.b[i].d);
    }
    for (cudaStream_t x : {C.sH, C.sK, C.sD}) cudaStreamDestroy(x);
    C.ready = false;
    cudaSetDevice(cur);
  }
  return st;
}

// ---------------------------------------------------------------- distributed large n
static bool dist_args_ok(int n, int P, int rank) { return n > GJ_BATCHED_MAX_N && P >= 1 && P <= GJ_DIST_MAX_RANKS && rank >= 0 && rank < P; }

gj_status gj_dist_sizes(int n, int nranks, int rank, int* npad, int* ncols_local, int* ncols_local_real) {
  if (!dist_args_ok(n, nranks, rank) || !npad || !ncols_local || !ncols_local_real) return GJ_ERR_ARG;
  dist_sizes(n, nranks, rank, npad, ncols_local, ncols_local_real);
  return GJ_OK;
}

gj_status gj_dist_step_init(int n, int nranks, int rank, const double* A_local, int64_t lda, double* X_local,
                       int32_t* pos, int32_t* pivstep, uint64_t* smax_bits, void* stream) {
  if (!dist_args_ok(n, nranks, rank) || !X_local || !pos || !pivstep || !smax_bits) return GJ_ERR_ARG;
  int npad, nl, nr;
  dist_sizes(n, nranks, rank, &npad, &nl, &nr);
  if (nr > 0 && (!A_local || lda < nr)) return GJ_ERR_ARG;
  return dist_init(n, nranks, rank, A_local, lda, X_local, pos, pivstep, reinterpret_cast<unsigned long long*>(smax_bits),
                   static_cast<cudaStream_t>(stream)) == cudaSuccess ? GJ_OK : GJ_ERR_CUDA;
}

gj_status gj_dist_step_factor(int n, int nranks, int rank, int k, double* X_local, int32_t* pos, int32_t* pivstep,
                         double* rec_p, int32_t* rec_q, int32_t* rec_row, double* W, void* stream) {
  if (!dist_args_ok(n, nranks, rank) || !X_local || !pos || !pivstep || !rec_p || !rec_q || !rec_row || !W) return GJ_ERR_ARG;
  int npad, nl, nr;
  dist_sizes(n, nranks, rank, &npad, &nl, &nr);
  if (k < 0 || k >= npad / GJ_DIST_BLOCK || k % nranks != rank) return GJ_ERR_ARG;
  return dist_factor(n, nranks, rank, k, X_local, pos, pivstep, rec_p, rec_q, rec_row, W,
                     static_cast<cudaStream_t>(stream)) == cudaSuccess ? GJ_OK : GJ_ERR_CUDA;
}

gj_status gj_dist_step_update(int n, int nranks, int rank, int k, int part, double* X_local, const double* W,
                         const int32_t* pivstep, const int32_t* rec_row, double* R, void* stream) {
  if (!dist_args_ok(n, nranks, rank) || !W || !pivstep || !rec_row || part < 0 || part > 2) return GJ_ERR_ARG;
  int npad, nl, nr;
  dist_sizes(n, nranks, rank, &npad, &nl, &nr);
  const int nb = npad / GJ_DIST_BLOCK;
  if (k < 0 || k >= nb) return GJ_ERR_ARG;
  if (part > 0 && (k + 1 >= nb || (k + 1) % nranks != rank)) return GJ_ERR_ARG;
  if (part == 2 && k % nranks == rank && nranks != 1) return GJ_ERR_ARG;
  if (nl > 0 && (!X_local || !R)) return GJ_ERR_ARG;
  return dist_update(n, nranks, rank, k, part, X_local, W, pivstep, rec_row, R, static_cast<cudaStream_t>(stream)) ==
                 cudaSuccess ? GJ_OK : GJ_ERR_CUDA;
}

gj_status gj_dist_step_finalize(int n, const double* rec_p, const int32_t* rec_q, double tol, const uint64_t* smax_bits,
                           int32_t* ipiv, double* logabsdet, int8_t* sign, int32_t* info, void* stream) {
  if (n < 1 || !rec_p || !rec_q || !smax_bits) return GJ_ERR_ARG;
  return dist_finalize(n, rec_p, rec_q, resolve_tol(GJ_F64, n, tol), reinterpret_cast<const unsigned long long*>(smax_bits),
                       ipiv, logabsdet, sign, info, static_cast<cudaStream_t>(stream)) == cudaSuccess ? GJ_OK : GJ_ERR_CUDA;
}

gj_status gj_dist_step_unpermute_plan(int n, int nranks, int rank, const int32_t* pivstep, int32_t* send_cols,
                                 int32_t* recv_cols, int32_t* counts, void* stream) {
  if (!dist_args_ok(n, nranks, rank) || !pivstep || !send_cols || !recv_cols || !counts) return GJ_ERR_ARG;
  return dist_unpermute_plan(n, nranks, rank, pivstep, send_cols, recv_cols, counts, static_cast<cudaStream_t>(stream)) ==
                 cudaSuccess ? GJ_OK : GJ_ERR_CUDA;
}

gj_status gj_dist_step_unpermute_pack(int n, int nranks, int rank, const double* X_local, const int32_t* rec_row,
                                 const int32_t* send_cols, int m, double* sendbuf, void* stream) {
  if (!dist_args_ok(n, nranks, rank) || m < 0 || (m > 0 && (!X_local || !rec_row || !send_cols || !sendbuf))) return GJ_ERR_ARG;
  return dist_unpermute_pack(n, nranks, rank, X_local, rec_row, send_cols, m, sendbuf, static_cast<cudaStream_t>(stream)) ==
                 cudaSuccess ? GJ_OK : GJ_ERR_CUDA;
}

gj_status gj_dist_step_unpermute_unpack(int n, const double* recvbuf, const int32_t* recv_cols, int m, double* Ainv_local,
                                   int64_t ld, void* stream) {
  if (n < 1 || m < 0 || (m > 0 && (!recvbuf || !recv_cols || !Ainv_local))) return GJ_ERR_ARG;
  return dist_unpermute_unpack(n, recvbuf, recv_cols, m, Ainv_local, ld, static_cast<cudaStream_t>(stream)) == cudaSuccess
             ? GJ_OK : GJ_ERR_CUDA;
}

}  // extern "C"
