// K2 — batched Gauss–Jordan inversion for 32 < n <= 64 on sm_100a: one matrix per CTA
// of 64 threads (two warps), thread i holds row i of the compact working array in
// registers; n < 64 runs padded with identity rows/columns (padded steps pick the
// padding rows and change nothing real).
//
// The method per step k is K1's (gj_batched.cu; §2 Eqs. (14)-(15), Obs. 2-3,
// listing L150-L177): max-|x_ik| pivot search over un-pivoted rows with ties to the
// smallest physical position (reading G3), logical swaps tracked on positions, deferred
// pivot-row normalisation, Eq. (15) update with the compact D column, rotated registers
// in a rolled two-step loop, per-step (p, q) record, un-permuted store (L179-L198).
// What differs from K1 is the cross-warp part: each warp reduces its 32 candidates with
// redux.sync, the two warp winners meet in shared memory across one CTA barrier, and the
// pivot row is published across a second barrier.
// I/O: n = 64 and 16-byte aligned buffers stream each matrix with TMA (four or two
// 128-byte-swizzled boxes of 64 rows); otherwise coalesced loads through a padded buffer.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "gj_internal.h"
#include "gj_ptx.cuh"
#include "gj_rowops.cuh"

namespace gj {
namespace {

using namespace ptx;
using namespace rowops;

constexpr int NP = 64;
constexpr int kThreads = 64;

template <typename T>
struct L64 {
  static constexpr int RB = NP * (int)sizeof(T);           // 256 or 512 bytes per row
  static constexpr int SPAN = 128;
  static constexpr int REG = RB / SPAN;                    // TMA boxes per matrix
  static constexpr int BOX_COLS = SPAN / (int)sizeof(T);
  static constexpr int TMA_BYTES = NP * RB;
  static constexpr int PAD_BYTES = NP * (NP + 1) * (int)sizeof(T);
  static constexpr int STAGE = (PAD_BYTES + 1023) / 1024 * 1024;   // >= TMA_BYTES
  static constexpr int PROW = 2 * NP * (int)sizeof(T);
  static constexpr int XS = 2 * 2 * 16;                     // [buf][warp] candidate triples
  static constexpr int REC = NP * 16;
  static constexpr int PERM = NP * 4;
  static constexpr int MISC = 128;                          // mbarrier + epilogue exchange
  static constexpr int TOTAL = STAGE + PROW + XS + REC + PERM + MISC;
};

template <typename T, bool TMA>
struct Addr64 {
  uint32_t rb, rx;
  __device__ __forceinline__ explicit Addr64(int row) {
    if constexpr (TMA) {
      rb = (uint32_t)(row * 128);
      rx = (uint32_t)((row & 7) << 4);
    } else {
      rb = (uint32_t)(row * (NP + 1) * (int)sizeof(T));
      rx = 0;
    }
  }
  __device__ __forceinline__ uint32_t at_b(uint32_t cb) const {
    if constexpr (TMA) {
      return (cb >> 7) * (NP * 128) + rb + ((cb & 127u) ^ rx);
    } else {
      return rb + cb;
    }
  }
};

// Warp-level best candidate: (hi, lo) of |x| and the smallest position among the tied.
__device__ __forceinline__ uint4 warp_best(float v, uint32_t kmask, int pos) {
  const uint32_t key = __float_as_uint(v) & 0x7fffffffu & kmask;
  const uint32_t m = __reduce_max_sync(0xffffffffu, key);
  const uint32_t pc = (key == m && kmask != 0u) ? (uint32_t)pos : 0xffffu;
  const uint32_t pw = __reduce_min_sync(0xffffffffu, pc);
  return make_uint4(m, 0u, pw, 0u);
}
__device__ __forceinline__ uint4 warp_best(double v, uint32_t kmask, int pos) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  const uint32_t hi = (uint32_t)(b >> 32) & 0x7fffffffu & kmask;
  const uint32_t lo = (uint32_t)b & kmask;
  const uint32_t mh = __reduce_max_sync(0xffffffffu, hi);
  const uint32_t ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
  const uint32_t pc = (hi == mh && lo == ml && kmask != 0u) ? (uint32_t)pos : 0xffffu;
  const uint32_t pw = __reduce_min_sync(0xffffffffu, pc);
  return make_uint4(mh, ml, pw, 0u);
}

template <typename T, int PC, bool SECOND>
__device__ __forceinline__ void step64(int k, T (&x)[NP], T* prow, uint4* xs, unsigned char* rec, uint32_t& kmask,
                                       int& pos, int tid, int warp, int lane) {
  // a2: per-warp winner, then the two warp winners compared in shared memory
  const uint4 wb = warp_best(x[PC], kmask, pos);
  if (lane == 0) xs[PC * 2 + warp] = wb;
  __syncthreads();
  const uint4 b0 = xs[PC * 2 + 0], b1 = xs[PC * 2 + 1];
  const bool gt = (b0.x > b1.x) || (b0.x == b1.x && b0.y > b1.y);
  const bool eq = (b0.x == b1.x) && (b0.y == b1.y);
  const int q = (int)(eq ? min(b0.z, b1.z) : (gt ? b0.z : b1.z));
  const bool is_piv = pos == q;
  // a3: the listing's swap of rows k and q (L156-L162), on positions only
  if (pos == k) pos = q;
  if (is_piv) pos = k;
  // a4: publish the un-normalised pivot row (only the warp that holds it issues stores)
  T* pr = prow + PC * NP;
  if (__any_sync(0xffffffffu, is_piv)) st_row_if<T, NP>(is_piv, pr, x);
  __syncthreads();
  const T p = pr[PC];
  if (tid == 0) rec_store(rec, k, p, q);
  const T rp = rcp(p);
  kmask = is_piv ? 0u : kmask;
  // a5: Eq. (15) with the deferred pivot-row scale; column k becomes the D column.
  // The pivot row is streamed from shared memory in chunks (a full fp64 row in registers
  // next to the working row would exceed the register file).
  const T nf = is_piv ? T(0) : -(x[PC] * rp);
  const T dcol = is_piv ? T(1) : nf;
  constexpr int CH = 16 / (int)sizeof(T) * 4;   // 8 doubles / 16 floats per chunk
  if constexpr (!SECOND) {
#pragma unroll
    for (int c = 0; c < NP; c += CH) {
      T y[CH];
#pragma unroll
      for (int j = 0; j < CH; ++j) y[j] = pr[c + j];
#pragma unroll
      for (int j = 0; j < CH; ++j)
        if (c + j != 0) x[c + j] = fma(nf, y[j], x[c + j]);
      asm volatile("" ::: "memory");
    }
    x[0] = dcol;
  } else {
    const T c0 = fma(nf, pr[0], x[0]);
#pragma unroll
    for (int c = 0; c < NP; c += CH) {
      T y[CH];
#pragma unroll
      for (int j = 0; j < CH; ++j) y[j] = pr[c + j];
#pragma unroll
      for (int j = 0; j < CH; ++j)
        if (c + j >= 2) x[c + j - 2] = fma(nf, y[j], x[c + j]);
      asm volatile("" ::: "memory");
    }
    x[NP - 2] = c0;
    x[NP - 1] = dcol;
  }
}

struct Maps64 {
  CUtensorMap a, x;
};

template <typename T, bool TMA>
__global__ void __launch_bounds__(kThreads)
gj_batched64_kernel(BatchedArgs a, const __grid_constant__ Maps64 tm) {
  using LY = L64<T>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* stage = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  T* prow = reinterpret_cast<T*>(stage + LY::STAGE);
  uint4* xs = reinterpret_cast<uint4*>(reinterpret_cast<unsigned char*>(prow) + LY::PROW);
  unsigned char* rec = reinterpret_cast<unsigned char*>(xs) + LY::XS;
  int* perm = reinterpret_cast<int*>(rec + LY::REC);
  uint64_t* bar = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(perm) + LY::PERM);
  uint32_t* ex = reinterpret_cast<uint32_t*>(bar + 1);   // epilogue exchange [warp][4]

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int n = a.n;
  const int nn = n * n;
  const T* __restrict__ Ag = static_cast<const T*>(a.A);
  T* __restrict__ Xg = static_cast<T*>(a.Ainv);

  if constexpr (TMA) {
    if (tid == 0) {
      mbar_init(bar, 1);
      fence_mbar_init();
    }
    __syncthreads();
  }

  int it = 0;
  for (int64_t m = blockIdx.x; m < a.batch; m += gridDim.x, ++it) {
    // ---- a1: load ----
    if constexpr (TMA) {
      if (tid == 0) {
        bulk_wait_read0();   // the previous matrix's TMA store has read the stage
        mbar_expect_tx(bar, LY::TMA_BYTES);
#pragma unroll
        for (int rg = 0; rg < LY::REG; ++rg)
          tma_load_2d(stage + rg * NP * 128, &tm.a, rg * LY::BOX_COLS, (int)(m * NP), bar);
      }
      while (!mbar_try_wait(bar, it & 1)) {
      }
      __syncwarp();
    } else {
      const int64_t gofs = m * nn;
      for (int e0 = 0; e0 < nn; e0 += kThreads * 8) {
        T v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int e = e0 + u * kThreads + tid;
          v[u] = e < nn ? __ldcs(Ag + gofs + e) : T(0);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int e = e0 + u * kThreads + tid;
          if (e < nn) {
            const int r = e / n;
            *reinterpret_cast<T*>(stage + Addr64<T, false>(r).at_b((e - r * n) * sizeof(T))) = v[u];
          }
        }
      }
      __syncthreads();
    }
    T x[NP];
    const bool real_row = tid < n;
    {
      const Addr64<T, TMA> ra(tid);
      if constexpr (TMA) {
#pragma unroll
        for (int j = 0; j < NP; j += 16 / (int)sizeof(T)) {
          const uint4 u = *reinterpret_cast<const uint4*>(stage + ra.at_b(j * sizeof(T)));
          if constexpr (sizeof(T) == 4) {
            x[j] = __uint_as_float(u.x); x[j + 1] = __uint_as_float(u.y);
            x[j + 2] = __uint_as_float(u.z); x[j + 3] = __uint_as_float(u.w);
          } else {
            x[j] = __longlong_as_double((long long)(((unsigned long long)u.y << 32) | u.x));
            x[j + 1] = __longlong_as_double((long long)(((unsigned long long)u.w << 32) | u.z));
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < NP; ++j)
          x[j] = (real_row && j < n) ? *reinterpret_cast<const T*>(stage + ra.at_b(j * sizeof(T)))
                                     : ((tid == j) ? T(1) : T(0));
      }
    }
    // zero threshold tau = tol * max|a_ij| (Obs. 2, reading G1)
    T rowmax = T(0);
#pragma unroll
    for (int j = 0; j < NP; ++j)
      if (real_row && j < n) rowmax = fmax(rowmax, fabs(x[j]));
    {
      const unsigned long long rb =
          sizeof(T) == 4 ? (unsigned long long)__float_as_uint((float)rowmax) << 32
                         : (unsigned long long)__double_as_longlong((double)rowmax);
      const uint32_t mh = __reduce_max_sync(0xffffffffu, (uint32_t)(rb >> 32));
      const uint32_t ml = __reduce_max_sync(0xffffffffu, (uint32_t)(rb >> 32) == mh ? (uint32_t)rb : 0u);
      if (lane == 0) {
        ex[warp * 4 + 0] = mh;
        ex[warp * 4 + 1] = ml;
      }
    }
    __syncthreads();   // also: the stage has been fully read
    double smax;
    {
      const unsigned long long w0 = ((unsigned long long)ex[0] << 32) | ex[1];
      const unsigned long long w1 = ((unsigned long long)ex[4] << 32) | ex[5];
      const unsigned long long w = w0 > w1 ? w0 : w1;
      smax = sizeof(T) == 4 ? (double)__uint_as_float((uint32_t)(w >> 32)) : __longlong_as_double((long long)w);
    }
    const T tau = round_down_to(a.tol * smax, T(0));

    uint32_t kmask = 0xffffffffu;
    int pos = tid;
#pragma unroll 1
    for (int k = 0; k < NP; k += 2) {
      step64<T, 0, false>(k, x, prow, xs, rec, kmask, pos, tid, warp, lane);
      step64<T, 1, true>(k + 1, x, prow, xs, rec, kmask, pos, tid, warp, lane);
    }
    __syncthreads();

    // ---- a6: det / ipiv / singular flag from the per-step record ----
    T p_own, p_k;
    int q_own, q_k;
    rec_load(rec, pos, p_own, q_own);
    rec_load(rec, tid, p_k, q_k);
    (void)q_own;
    const T myrp = rcp(p_own);
    const bool stepk = tid < n;
    const unsigned fb = __ballot_sync(0xffffffffu, stepk && fabs(p_k) <= tau);
    const int ns = __popc(__ballot_sync(0xffffffffu, stepk && q_k != tid));
    const int ng = __popc(__ballot_sync(0xffffffffu, stepk && p_k < T(0)));
    double lg = stepk ? log_abs(p_k) : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lg += __shfl_xor_sync(0xffffffffu, lg, o);
    if (lane == 0) {
      ex[8 + warp * 4 + 0] = fb;
      ex[8 + warp * 4 + 1] = (uint32_t)(ns + ng * 256);
      *reinterpret_cast<double*>(&ex[16 + warp * 2]) = lg;
    }
    if (a.ipiv && stepk) a.ipiv[m * n + tid] = q_k + 1;
    perm[pos] = tid * (int)sizeof(T);   // output column (bytes) of compact column `pos`
    __syncthreads();
    if (tid == 0) {
      const unsigned f0 = ex[8], f1 = ex[12];
      const int info = f0 ? __ffs(f0) : (f1 ? 32 + __ffs(f1) : 0);
      const int nsw = (int)((ex[9] & 255u) + (ex[13] & 255u));
      const int nng = (int)((ex[9] >> 8) + (ex[13] >> 8));
      const double lgs = *reinterpret_cast<double*>(&ex[16]) + *reinterpret_cast<double*>(&ex[18]);
      const int sgn = ((nsw ^ nng) & 1) ? -1 : 1;
      if (a.info) a.info[m] = info;
      if (a.logabsdet) a.logabsdet[m] = info ? -INFINITY : lgs;
      if (a.sign) a.sign[m] = info ? 0 : (int8_t)sgn;
      if (a.det) static_cast<T*>(a.det)[m] = info ? T(0) : (T)(sgn * exp(lgs));
    }

    // ---- a7 + a8: un-permuted store ----
    if (Xg != nullptr) {
      const Addr64<T, TMA> dst(pos);
#pragma unroll
      for (int kp = 0; kp < NP; kp += 4) {
        const int4 cb = *reinterpret_cast<const int4*>(perm + kp);
        const int cbs[4] = {cb.x, cb.y, cb.z, cb.w};
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (real_row && kp + u < n) *reinterpret_cast<T*>(stage + dst.at_b((uint32_t)cbs[u])) = myrp * x[kp + u];
      }
      if constexpr (TMA) {
        fence_async_smem();
        __syncthreads();
        if (tid == 0) {
#pragma unroll
          for (int rg = 0; rg < LY::REG; ++rg)
            tma_store_2d(&tm.x, rg * LY::BOX_COLS, (int)(m * NP), stage + rg * NP * 128);
          bulk_commit();
        }
      } else {
        __syncthreads();
        const int64_t gofs = m * nn;
        for (int e = tid; e < nn; e += kThreads) {
          const int r = e / n;
          __stcs(Xg + gofs + e, *reinterpret_cast<const T*>(stage + Addr64<T, false>(r).at_b((e - r * n) * sizeof(T))));
        }
      }
    }
    __syncthreads();
  }
  if constexpr (TMA) {
    if (tid == 0) bulk_wait0();
  }
}

template <typename T, bool TMA>
cudaError_t launch64(const BatchedArgs& a, const Maps64& maps, cudaStream_t s) {
  const size_t smem = (size_t)L64<T>::TOTAL + 1024;
  auto kern = gj_batched64_kernel<T, TMA>;
  static unsigned long long configured = 0;
  const unsigned long long dbit = device_bit();
  if (!(configured & dbit)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured |= dbit;
  }
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const int64_t cap = (int64_t)device_sm_count() * per_sm;
  const int grid = (int)(a.batch < cap ? a.batch : cap);
  kern<<<grid, kThreads, smem, s>>>(a, maps);
  return cudaGetLastError();
}

template <typename T>
cudaError_t dispatch64(const BatchedArgs& a, cudaStream_t s) {
  Maps64 maps;
  using LY = L64<T>;
  const bool aligned = (reinterpret_cast<uintptr_t>(a.A) % 16 == 0) &&
                       (a.Ainv == nullptr || reinterpret_cast<uintptr_t>(a.Ainv) % 16 == 0);
  const bool f64 = sizeof(T) == 8;
  const uint64_t rows = (uint64_t)a.batch * NP;
  if (a.n == NP && aligned && rows < (1ull << 31) &&
      make_tma_map_2d(&maps.a, f64, a.A, NP, rows, NP * sizeof(T), LY::BOX_COLS, NP, 128) &&
      (a.Ainv == nullptr || make_tma_map_2d(&maps.x, f64, a.Ainv, NP, rows, NP * sizeof(T), LY::BOX_COLS, NP, 128))) {
    if (a.Ainv == nullptr) maps.x = maps.a;
    return launch64<T, true>(a, maps, s);
  }
  return launch64<T, false>(a, maps, s);
}

}  // namespace

cudaError_t launch_batched64(gj_dtype dt, const BatchedArgs& a, cudaStream_t s) {
  if (a.batch == 0) return cudaSuccess;
  if (dt == GJ_F64 && a.n == 64) {
    // K2e (gj_batched64e.cu); an unaligned batch falls back to the generic K2 below
    const cudaError_t e = launch_batched64e(a, s);
    if (e != cudaErrorNotSupported) return e;
  }
  return dt == GJ_F32 ? dispatch64<float>(a, s) : dispatch64<double>(a, s);
}

}  // namespace gj
