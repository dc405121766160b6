// Distributed large-n Gauss–Jordan, library-driven (gj_dist_init / gj_invert_dist /
// gj_dist_finalize, include/gjinv.h): the column-block-cyclic method of SURVEY.md §8e with
// the NCCL exchange inside the library.  The per-rank compute steps are the ones
// gj_dist_step_* expose (gj_large.cu: panel factorisation K3, trailing update K4b, the
// un-permutation kernels); this file is the host driver around them — the same schedule as
// paper_1401_7962_b200/dist.py, which runs it over torch.distributed (gloo or NCCL) for tests:
//   * panel 0 is factored by rank 0 and broadcast before the loop;
//   * per panel k every rank updates its local columns with panel k; the owner of panel
//     k+1 first updates only k+1's columns, copies the replicated state into the buffers of
//     parity k+1, factors k+1, then runs the rest of k's update beside that factorisation;
//   * panel k+1 (W and the state) is broadcast from its owner on a side stream into the
//     buffers of parity k+1 — after k+1's factorisation (owner) and after panel k-1's update
//     (every rank: the last reader of those buffers), not after panel k's update;
//   * the threshold's max|a_ij| is an all-reduce (max of the bit patterns of non-negative
//     doubles orders like the values), and the un-permutation (listing L179-L198) one
//     all-to-all of columns (grouped send / receive), planned on the device.
// NCCL is opened at run time (dlopen), so the library links no NCCL.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdint>
#include <cstring>
#include <vector>

#include "gj_internal.h"
#include "gjinv.h"

namespace {

// The NCCL C ABI (stable since 2.x): the few types and entry points used here.
typedef struct ncclComm* ncclComm_t;
struct ncclUniqueId {
  char internal[128];
};
typedef int ncclResult_t;   // ncclSuccess = 0
enum { nccl_uint8 = 1, nccl_int32 = 2, nccl_uint64 = 5, nccl_float64 = 8 };
enum { nccl_max = 2 };

struct Nccl {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
};

const Nccl& nccl() {
  static Nccl N;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
    if (h) {
      auto sym = [&](const char* a) { return dlsym(h, a); };
      N.GetUniqueId = reinterpret_cast<decltype(N.GetUniqueId)>(sym("ncclGetUniqueId"));
      N.CommInitRank = reinterpret_cast<decltype(N.CommInitRank)>(sym("ncclCommInitRank"));
      N.CommDestroy = reinterpret_cast<decltype(N.CommDestroy)>(sym("ncclCommDestroy"));
      N.Broadcast = reinterpret_cast<decltype(N.Broadcast)>(sym("ncclBroadcast"));
      N.AllReduce = reinterpret_cast<decltype(N.AllReduce)>(sym("ncclAllReduce"));
      N.Send = reinterpret_cast<decltype(N.Send)>(sym("ncclSend"));
      N.Recv = reinterpret_cast<decltype(N.Recv)>(sym("ncclRecv"));
      N.GroupStart = reinterpret_cast<decltype(N.GroupStart)>(sym("ncclGroupStart"));
      N.GroupEnd = reinterpret_cast<decltype(N.GroupEnd)>(sym("ncclGroupEnd"));
      N.ok = N.GetUniqueId && N.CommInitRank && N.CommDestroy && N.Broadcast && N.AllReduce && N.Send && N.Recv &&
             N.GroupStart && N.GroupEnd;
    }
  }
  return N;
}

}  // namespace

struct gj_dist_ctx {
  int nranks = 0, rank = 0, device = 0;
  ncclComm_t comm = nullptr;
  cudaStream_t side = nullptr;
  cudaEvent_t ev_upd = nullptr, ev_fac = nullptr, ev_b = nullptr;
  void* ws = nullptr;      // device workspace, kept between calls (grown on demand)
  size_t ws_bytes = 0;
};

namespace {

struct DeviceScope {   // run on the handle's device, restore the caller's
  int prev = 0;
  explicit DeviceScope(int d) {
    cudaGetDevice(&prev);
    cudaSetDevice(d);
  }
  ~DeviceScope() { cudaSetDevice(prev); }
};

#define GJ_CU(x)                                     \
  do {                                               \
    if ((x) != cudaSuccess) return GJ_ERR_CUDA;      \
  } while (0)
#define GJ_NC(x)                                     \
  do {                                               \
    if ((x) != 0) return GJ_ERR_NCCL;                \
  } while (0)

// Carves 256-byte aligned pieces from one workspace (a dry run sizes it).
struct Carve {
  char* base;
  size_t off = 0;
  explicit Carve(void* b) : base(static_cast<char*>(b)) {}
  template <typename T>
  T* get(size_t count) {
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += (count * sizeof(T) + 255) / 256 * 256;
    return p;
  }
};

}  // namespace

extern "C" {

gj_status gj_dist_get_unique_id(unsigned char unique_id[GJ_DIST_UNIQUE_ID_BYTES]) {
  if (!unique_id) return GJ_ERR_ARG;
  const Nccl& N = nccl();
  if (!N.ok) return GJ_ERR_NCCL;
  ncclUniqueId id;
  GJ_NC(N.GetUniqueId(&id));
  memcpy(unique_id, id.internal, GJ_DIST_UNIQUE_ID_BYTES);
  return GJ_OK;
}

gj_status gj_dist_init(int nranks, int rank, const unsigned char unique_id[GJ_DIST_UNIQUE_ID_BYTES], int device,
                       gj_dist_handle* handle) {
  if (!handle || !unique_id || nranks < 1 || nranks > GJ_DIST_MAX_RANKS || rank < 0 || rank >= nranks || device < 0)
    return GJ_ERR_ARG;
  *handle = nullptr;
  const Nccl& N = nccl();
  if (!N.ok) return GJ_ERR_NCCL;
  DeviceScope ds(device);
  gj_dist_ctx* c = new gj_dist_ctx;
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  ncclUniqueId id;
  memcpy(id.internal, unique_id, GJ_DIST_UNIQUE_ID_BYTES);
  if (N.CommInitRank(&c->comm, nranks, id, rank) != 0) {
    delete c;
    return GJ_ERR_NCCL;
  }
  if (cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_upd, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_fac, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_b, cudaEventDisableTiming) != cudaSuccess) {
    N.CommDestroy(c->comm);
    delete c;
    return GJ_ERR_CUDA;
  }
  *handle = c;
  return GJ_OK;
}

gj_status gj_dist_finalize(gj_dist_handle c) {
  if (!c) return GJ_OK;
  DeviceScope ds(c->device);
  const Nccl& N = nccl();
  gj_status st = GJ_OK;
  if (c->comm && N.ok && N.CommDestroy(c->comm) != 0) st = GJ_ERR_NCCL;
  if (c->ws) cudaFree(c->ws);
  if (c->side) cudaStreamDestroy(c->side);
  for (cudaEvent_t e : {c->ev_upd, c->ev_fac, c->ev_b})
    if (e) cudaEventDestroy(e);
  delete c;
  return st;
}

gj_status gj_invert_dist(gj_dist_handle c, int n, const double* A_local, int64_t lda, double* Ainv_local,
                         int64_t ldainv, int32_t* ipiv, double* logabsdet, int8_t* sign, int32_t* info, double tol,
                         void* stream) {
  if (!c || n <= GJ_BATCHED_MAX_N || n > GJ_LARGE_MAX_N) return GJ_ERR_ARG;
  const int P = c->nranks, rank = c->rank;
  int npad, nl, nr;
  gj::dist_sizes(n, P, rank, &npad, &nl, &nr);
  if (nr > 0 && (!A_local || !Ainv_local || lda < nr || ldainv < nr)) return GJ_ERR_ARG;
  const Nccl& N = nccl();
  if (!N.ok) return GJ_ERR_NCCL;
  DeviceScope ds(c->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int nb = npad / GJ_DIST_BLOCK;
  const int B = GJ_DIST_BLOCK;

  // workspace (kept in the handle): X, state x 2, W x 2, R, smax, outputs, plan, buffers
  auto carve = [&](Carve& cv, int ms, int mr) {
    struct Parts {
      double *X, *w0, *w1, *R, *lg, *sendbuf, *recvbuf;
      int32_t *i0, *i1, *ipiv, *info, *send_cols, *recv_cols, *counts;
      uint64_t* smax;
      int8_t* sg;
    } p;
    p.X = cv.get<double>((size_t)npad * (nl > 0 ? nl : 1));
    p.i0 = cv.get<int32_t>(6 * (size_t)npad);
    p.i1 = cv.get<int32_t>(6 * (size_t)npad);
    p.w0 = cv.get<double>((size_t)npad * B);
    p.w1 = cv.get<double>((size_t)npad * B);
    p.R = cv.get<double>((size_t)B * (nl > 0 ? nl : 1));
    p.smax = cv.get<uint64_t>(1);
    p.ipiv = cv.get<int32_t>(n);
    p.lg = cv.get<double>(1);
    p.sg = cv.get<int8_t>(1);
    p.info = cv.get<int32_t>(1);
    p.send_cols = cv.get<int32_t>(nl > 0 ? nl : 1);
    p.recv_cols = cv.get<int32_t>(nr > 0 ? nr : 1);
    p.counts = cv.get<int32_t>(2 * P);
    p.sendbuf = cv.get<double>((size_t)(ms > 0 ? ms : 1) * n);
    p.recvbuf = cv.get<double>((size_t)(mr > 0 ? mr : 1) * n);
    return p;
  };
  // the all-to-all buffers are at most one local column block set each: size for the worst
  // case (every local column / every output column) so the workspace is sized up front
  Carve dry(nullptr);
  carve(dry, nl, nr);
  if (dry.off > c->ws_bytes) {
    if (c->ws) {
      GJ_CU(cudaStreamSynchronize(s));
      cudaFree(c->ws);
      c->ws = nullptr;
      c->ws_bytes = 0;
    }
    GJ_CU(cudaMalloc(&c->ws, dry.off));
    c->ws_bytes = dry.off;
  }
  Carve cv(c->ws);
  const auto pp = carve(cv, nl, nr);
  double* X = pp.X;
  int32_t* ibuf[2] = {pp.i0, pp.i1};
  double* wbuf[2] = {pp.w0, pp.w1};
  double* R = pp.R;
  uint64_t* smax = pp.smax;
  int32_t* o_ipiv = ipiv ? ipiv : pp.ipiv;
  double* o_lg = logabsdet ? logabsdet : pp.lg;
  int8_t* o_sg = sign ? sign : pp.sg;
  int32_t* o_info = info ? info : pp.info;
  int32_t* send_cols = pp.send_cols;
  int32_t* recv_cols = pp.recv_cols;
  int32_t* counts = pp.counts;
  // replicated state views: pos | pivstep | rec_q | rec_row | rec_p (fp64 as 2 x int32)
  struct View {
    int32_t *pos, *piv, *rq, *rr;
    double* rp;
  };
  auto view = [&](int32_t* b) {
    return View{b, b + npad, b + 2 * npad, b + 3 * npad, reinterpret_cast<double*>(b + 4 * npad)};
  };
  auto cu = [](cudaError_t e) { return e == cudaSuccess ? GJ_OK : GJ_ERR_CUDA; };

  View v0 = view(ibuf[0]);
  GJ_CU(cudaMemsetAsync(smax, 0, 8, s));
  GJ_CU(gj::dist_init(n, P, rank, nr > 0 ? A_local : nullptr, nr > 0 ? lda : 1, X, v0.pos, v0.piv,
                      reinterpret_cast<unsigned long long*>(smax), s));
  if (P > 1) GJ_NC(N.AllReduce(smax, smax, 1, nccl_uint64, nccl_max, c->comm, s));
  double* Xo = nl > 0 ? X : nullptr;
  double* Ro = nl > 0 ? R : nullptr;
  if (rank == 0) GJ_CU(gj::dist_factor(n, P, rank, 0, X, v0.pos, v0.piv, v0.rp, v0.rq, v0.rr, wbuf[0], s));
  if (P > 1) {
    GJ_NC(N.Broadcast(ibuf[0], ibuf[0], 6 * (size_t)npad, nccl_int32, 0, c->comm, s));
    GJ_NC(N.Broadcast(wbuf[0], wbuf[0], (size_t)npad * B, nccl_float64, 0, c->comm, s));
  }
  GJ_CU(cudaEventRecord(c->ev_upd, s));
  for (int k = 0; k < nb; ++k) {
    const View vk = view(ibuf[k & 1]);
    double* W = wbuf[k & 1];
    const bool nxt = k + 1 < nb;
    const bool own_next = nxt && (k + 1) % P == rank;
    if (own_next) {
      GJ_CU(gj::dist_update(n, P, rank, k, 1, Xo, W, vk.piv, vk.rr, Ro, s));
      GJ_CU(cudaMemcpyAsync(ibuf[(k + 1) & 1], ibuf[k & 1], 6 * (size_t)npad * 4, cudaMemcpyDeviceToDevice, s));
      const View vn = view(ibuf[(k + 1) & 1]);
      GJ_CU(gj::dist_factor(n, P, rank, k + 1, X, vn.pos, vn.piv, vn.rp, vn.rq, vn.rr, wbuf[(k + 1) & 1], s));
      GJ_CU(cudaEventRecord(c->ev_fac, s));
      GJ_CU(gj::dist_update(n, P, rank, k, 2, Xo, W, vk.piv, vk.rr, Ro, s));
    } else {
      GJ_CU(gj::dist_update(n, P, rank, k, 0, Xo, W, vk.piv, vk.rr, Ro, s));
    }
    if (nxt && P > 1) {
      // panel k+1 into the buffers of parity k+1 on the side stream: after its factorisation
      // (owner) and after panel k-1's update (their last reader), not after panel k's
      GJ_CU(cudaStreamWaitEvent(c->side, c->ev_upd, 0));
      if (own_next) GJ_CU(cudaStreamWaitEvent(c->side, c->ev_fac, 0));
      const int root = (k + 1) % P;
      GJ_NC(N.GroupStart());
      GJ_NC(N.Broadcast(ibuf[(k + 1) & 1], ibuf[(k + 1) & 1], 6 * (size_t)npad, nccl_int32, root, c->comm, c->side));
      GJ_NC(N.Broadcast(wbuf[(k + 1) & 1], wbuf[(k + 1) & 1], (size_t)npad * B, nccl_float64, root, c->comm,
                        c->side));
      GJ_NC(N.GroupEnd());
      GJ_CU(cudaEventRecord(c->ev_b, c->side));
      GJ_CU(cudaEventRecord(c->ev_upd, s));
      GJ_CU(cudaStreamWaitEvent(s, c->ev_b, 0));
    } else {
      GJ_CU(cudaEventRecord(c->ev_upd, s));
    }
  }
  const View vf = view(ibuf[(nb - 1) & 1]);
  GJ_CU(gj::dist_finalize(n, vf.rp, vf.rq, tol, reinterpret_cast<const unsigned long long*>(smax), o_ipiv, o_lg,
                          o_sg, o_info, s));
  // un-permutation: Ainv[i][j] = X[rec_row[i]][pivstep[j]], one all-to-all of columns
  GJ_CU(gj::dist_unpermute_plan(n, P, rank, vf.piv, send_cols, recv_cols, counts, s));
  std::vector<int32_t> cnt(2 * P);
  GJ_CU(cudaMemcpyAsync(cnt.data(), counts, 2 * P * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  GJ_CU(cudaStreamSynchronize(s));
  int ms = 0, mr = 0;
  for (int p = 0; p < P; ++p) {
    ms += cnt[p];
    mr += cnt[P + p];
  }
  double* sendbuf = pp.sendbuf;
  double* recvbuf = P > 1 ? pp.recvbuf : sendbuf;
  if (ms > 0) GJ_CU(gj::dist_unpermute_pack(n, P, rank, X, vf.rr, send_cols, ms, sendbuf, s));
  if (P > 1) {
    GJ_NC(N.GroupStart());
    size_t so = 0, ro = 0;
    for (int p = 0; p < P; ++p) {
      if (cnt[p] > 0) GJ_NC(N.Send(sendbuf + so, (size_t)cnt[p] * n, nccl_float64, p, c->comm, s));
      if (cnt[P + p] > 0) GJ_NC(N.Recv(recvbuf + ro, (size_t)cnt[P + p] * n, nccl_float64, p, c->comm, s));
      so += (size_t)cnt[p] * n;
      ro += (size_t)cnt[P + p] * n;
    }
    GJ_NC(N.GroupEnd());
  }
  if (mr > 0) GJ_CU(gj::dist_unpermute_unpack(n, recvbuf, recv_cols, mr, Ainv_local, ldainv, s));
  return cu(cudaGetLastError());
}

}  // extern "C"
