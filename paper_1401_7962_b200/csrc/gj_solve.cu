// K7 — batched multi-RHS solve X = A^-1 B by Gauss–Jordan on [A | B], n <= 32, m <= 32
// right-hand sides (Eq. (12) with B in place of I: the elimination of
// Eqs. (14)-(15), applied to the n + m columns of [A | B]).
//
// K1's layout and step (lane = row, partial pivoting on the listing's rule with ties to the
// smallest physical position (G3), logical row swaps, deferred pivot-row normalisation),
// but the A part is not kept in compact form: the k loop is fully unrolled, step k's pivot
// column is register k and only the columns right of it are published, loaded and
// updated (the A part shrinks: ~n^3/2 + n^2 m FMAs instead of the inverse's n^3).  The B
// part (m registers) takes every step's update.  At the end the row pivoted at step k holds p_k x_k, so
// X[k][:] = b_row / p_k — a row gather, no column permutation (B's columns never move).
#include <cuda_runtime.h>
#include <cmath>
#include <cstdint>

#include "gj_internal.h"
#include "gj_ptx.cuh"
#include "gj_rowops.cuh"

namespace gj {
namespace {

using namespace ptx;
using namespace rowops;

constexpr int kSolveWarps = 4;

template <int L>
__device__ __forceinline__ uint32_t smax_u32(uint32_t v) {
  if constexpr (L == 32) {
    return __reduce_max_sync(0xffffffffu, v);
  } else {
#pragma unroll
    for (int o = L / 2; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
  }
}
template <int L>
__device__ __forceinline__ uint32_t smin_u32(uint32_t v) {
  if constexpr (L == 32) {
    return __reduce_min_sync(0xffffffffu, v);
  } else {
#pragma unroll
    for (int o = L / 2; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
  }
}
template <int L>
__device__ __forceinline__ double ssum(double v) {
#pragma unroll
  for (int o = L / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// a2: max |v| over the group's eligible rows (IEEE bit patterns; fp64 high word, then low
// word among the winners), ties -> the smallest physical position; returns that position
__device__ __forceinline__ void skey(float v, bool ok, uint32_t& hi, uint32_t& lo) {
  hi = ok ? (__float_as_uint(v) & 0x7fffffffu) : 0u;
  lo = 0u;
}
__device__ __forceinline__ void skey(double v, bool ok, uint32_t& hi, uint32_t& lo) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  hi = ok ? ((uint32_t)(b >> 32) & 0x7fffffffu) : 0u;
  lo = ok ? (uint32_t)b : 0u;
}
template <typename T, int L>
__device__ __forceinline__ int s_pivot(T v, bool ok, int pos) {
  uint32_t hi, lo;
  skey(v, ok, hi, lo);
  const uint32_t mh = smax_u32<L>(hi);
  uint32_t ml = 0u;
  if constexpr (sizeof(T) == 8) ml = smax_u32<L>(hi == mh ? lo : 0u);
  const bool cand = ok && hi == mh && lo == ml;
  return (int)smin_u32<L>(cand ? (uint32_t)pos : 0xffffu);
}

// cp.async.bulk.prefetch of the 16-byte aligned interior of [lo, hi)
__device__ __forceinline__ void prefetch_l2_range(const void* lo, const void* hi) {
  const uintptr_t a = ((uintptr_t)lo + 15) & ~(uintptr_t)15, b = (uintptr_t)hi & ~(uintptr_t)15;
  if (b > a) bulk_prefetch_l2(reinterpret_cast<const void*>(a), (uint32_t)(b - a));
}

template <typename T, int NP, int NR>
struct SolveSmem {
  static constexpr int MPW = 32 / NP;
  static constexpr int ROWS = 32;
  static constexpr int SA = ROWS * (NP + 1) * (int)sizeof(T);     // A staging (padded rows)
  static constexpr int SB = ROWS * (NR + 1) * (int)sizeof(T);     // B / X staging
  static constexpr int PA = 2 * MPW * (NP + 4) * (int)sizeof(T);  // pivot row, A part + pivot (2 buffers)
  static constexpr int PB = 2 * MPW * NR * (int)sizeof(T);        // pivot row, B part
  static constexpr int REC = ROWS * 16;
  static constexpr int per_warp = ((SA + SB + PA + PB + REC) + 15) / 16 * 16;
};

// rows [0, nrows) of length len (row-major, contiguous) <-> padded staging rows of the task
template <typename T, int STRIDE, bool LOAD>
__device__ __forceinline__ void move_rows(T* g, T* stage, int nrows, int len, int n, int NPr, int lane) {
  const int rpi = 32 / len;
  const int lr = lane / len, lc = lane - lr * len;
  const bool act = lr < rpi;
  const int iters = (nrows + rpi - 1) / rpi;
  const float rn = 1.0f / (float)n;
  for (int it0 = 0; it0 < iters; it0 += 8) {
    T v[8];
    if constexpr (LOAD) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int R = (it0 + u) * rpi + lr;
        v[u] = (act && R < nrows) ? __ldcs(g + R * len + lc) : T(0);
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int R = (it0 + u) * rpi + lr;
      if (act && R < nrows) {
        const int m = (int)(((float)R + 0.5f) * rn);   // matrix of row R (exact: R < 32)
        T* s = stage + (m * NPr + (R - m * n)) * STRIDE + lc;
        if constexpr (LOAD) {
          *s = v[u];
        } else {
          __stcs(g + R * len + lc, *s);
        }
      }
    }
  }
}

// One step K (static: the k loop is fully unrolled, so the pivot column is register K and
// only the columns right of it are live — the A part shrinks as the elimination proceeds).
template <typename T, int NP, int NR, int K>
__device__ __forceinline__ void solve_step(T (&x)[NP], T (&b)[NR], bool& done, int& pos, T* pa, T* pb,
                                           unsigned char* rec_g, int li) {
  constexpr int L = NP;
  constexpr int J0 = (K + 1) & ~3;   // first published / loaded column (16-byte aligned)
  const int q = s_pivot<T, L>(x[K], !done, pos);
  const bool piv = !done && pos == q;
  if (pos == K) pos = q;   // a3: the listing's swap of positions k and q (L156-L162)
  if (piv) pos = K;
  // a4: publish the pivot row's live A columns and its B part
  if constexpr (J0 < NP) {
    const uint32_t a0 = smem_u32(pa);
#pragma unroll
    for (int j = J0; j < NP; j += 16 / (int)sizeof(T)) {
      if constexpr (sizeof(T) == 4) {
        st_shared_v4_if(piv, a0 + 4u * j, x[j], x[j + 1], x[j + 2], x[j + 3]);
      } else {
        st_shared_v2_if(piv, a0 + 8u * j, x[j], x[j + 1]);
      }
    }
  }
  st_row_if<T, NR>(piv, pb, b);
  if (piv) pa[NP] = x[K];   // the pivot itself (slot NP)
  __syncwarp();
  const T pk = pa[NP];
  if (li == 0) rec_store(rec_g, K, pk, q);
  const T nf = piv ? T(0) : -(x[K] * rcp(pk));
  done = done || piv;
  // a5: A columns right of K (16-byte loads from J0), then every B column
  if constexpr (J0 < NP) {
    T y[NP];
#pragma unroll
    for (int j = J0; j < NP; j += 16 / (int)sizeof(T)) {
      if constexpr (sizeof(T) == 4) {
        const float4 v = *reinterpret_cast<const float4*>(pa + j);
        y[j] = v.x; y[j + 1] = v.y; y[j + 2] = v.z; y[j + 3] = v.w;
      } else {
        const double2 v = *reinterpret_cast<const double2*>(pa + j);
        y[j] = v.x; y[j + 1] = v.y;
      }
    }
#pragma unroll
    for (int j = K + 1; j < NP; ++j) x[j] = fma(nf, y[j], x[j]);
  }
  T yb[NR];
  ld_row<T, NR>(yb, pb);
  if constexpr (sizeof(T) == 4 && NR % 2 == 0) {
#pragma unroll
    for (int j = 0; j < NR; j += 2) ffma2(b[j], b[j + 1], nf, yb[j], yb[j + 1]);
  } else {
#pragma unroll
    for (int j = 0; j < NR; ++j) b[j] = fma(nf, yb[j], b[j]);
  }
}

template <typename T, int NP, int NR, int K>
__device__ __forceinline__ void solve_steps(T (&x)[NP], T (&b)[NR], bool& done, int& pos, T* pa0, T* pb0,
                                            unsigned char* rec_g, int li, int g) {
  if constexpr (K < NP) {
    constexpr int MPW = 32 / NP;
    constexpr int PAW = NP + 4;   // pivot-row buffer width (A columns + the pivot, 16-byte rows)
    // two buffers alternate, so step K+1's publish cannot overwrite what a slow lane of
    // step K still reads
    T* pa = pa0 + (K & 1) * MPW * PAW + g * PAW;
    T* pb = pb0 + (K & 1) * MPW * NR + g * NR;
    solve_step<T, NP, NR, K>(x, b, done, pos, pa, pb, rec_g, li);
    solve_steps<T, NP, NR, K + 1>(x, b, done, pos, pa0, pb0, rec_g, li, g);
  }
}

template <typename T, int NP, int NR>
__global__ void __launch_bounds__(kSolveWarps * 32) gj_solve_kernel(SolveArgs a) {
  using S = SolveSmem<T, NP, NR>;
  constexpr int L = NP, MPW = S::MPW;
  constexpr int RECW = sizeof(T) == 4 ? 8 : 16;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char* wb = smem_raw + warp * S::per_warp;
  T* sa = reinterpret_cast<T*>(wb);
  T* sb = reinterpret_cast<T*>(wb + S::SA);
  T* pa0 = reinterpret_cast<T*>(wb + S::SA + S::SB);
  T* pb0 = reinterpret_cast<T*>(wb + S::SA + S::SB + S::PA);
  unsigned char* rec = wb + S::SA + S::SB + S::PA + S::PB;

  const int n = a.n, m = a.m;
  const int g = lane / L, li = lane % L;
  const unsigned gmask = (L == 32 ? 0xffffffffu : ((1u << L) - 1u)) << (L * g);
  unsigned char* rec_g = rec + g * NP * RECW;
  const T* __restrict__ Ag = static_cast<const T*>(a.A);
  const T* Bg = static_cast<const T*>(a.B);   // X may alias B: no __restrict__
  T* Xg = static_cast<T*>(a.X);

  const int64_t ntasks = (a.batch + MPW - 1) / MPW;
  for (int64_t task = (int64_t)blockIdx.x * kSolveWarps + warp; task < ntasks;
       task += (int64_t)gridDim.x * kSolveWarps) {
    const int64_t item0 = task * MPW;
    const int64_t left = a.batch - item0;
    const int vi = left < MPW ? (int)left : MPW;
    const bool item_ok = g < vi;
    // the next task's A and B into L2 while this one runs (the 16-byte aligned interior)
    if (lane == 0 && task + (int64_t)gridDim.x * kSolveWarps < ntasks) {
      const int64_t nx0 = (task + (int64_t)gridDim.x * kSolveWarps) * MPW;
      const int64_t nx1 = nx0 + MPW < a.batch ? nx0 + MPW : a.batch;
      prefetch_l2_range(Ag + nx0 * n * n, Ag + nx1 * n * n);
      prefetch_l2_range(Bg + nx0 * n * m, Bg + nx1 * n * m);
    }
    // ---- a1: A and B rows of the task into the padded staging rows
    move_rows<T, NP + 1, true>(const_cast<T*>(Ag) + item0 * n * n, sa, vi * n, n, n, NP, lane);
    move_rows<T, NR + 1, true>(const_cast<T*>(Bg) + item0 * n * m, sb, vi * n, m, n, NP, lane);
    __syncwarp();
    const bool real = li < n;
    T x[NP], b[NR];
#pragma unroll
    for (int j = 0; j < NP; ++j) x[j] = (item_ok && real && j < n) ? sa[(g * NP + li) * (NP + 1) + j] : T(li == j ? 1 : 0);
#pragma unroll
    for (int j = 0; j < NR; ++j) b[j] = (item_ok && real && j < m) ? sb[(g * NP + li) * (NR + 1) + j] : T(0);
    __syncwarp();
    T rowmax = T(0);
#pragma unroll
    for (int j = 0; j < NP; ++j)
      if (real && j < n) rowmax = fmax(rowmax, fabs(x[j]));
    double smax;
    if constexpr (sizeof(T) == 4) {
      smax = (double)__uint_as_float(smax_u32<L>(__float_as_uint(rowmax)));
    } else {
      const unsigned long long bb = (unsigned long long)__double_as_longlong(rowmax);
      const uint32_t mh = smax_u32<L>((uint32_t)(bb >> 32));
      const uint32_t ml = smax_u32<L>((uint32_t)(bb >> 32) == mh ? (uint32_t)bb : 0u);
      smax = __longlong_as_double((long long)(((unsigned long long)mh << 32) | ml));
    }
    const T tau = round_down_to(a.tol * smax, T(0));

    bool done = false;
    int pos = li;
    // padded steps k >= n pick the identity padding rows and change nothing real
    solve_steps<T, NP, NR, 0>(x, b, done, pos, pa0, pb0, rec_g, li, g);
    __syncwarp();

    // ---- a6: det / ipiv / singular flag (lane li <-> step li)
    T p_own, p_k;
    int q_own, q_k;
    rec_load(rec_g, pos, p_own, q_own);
    rec_load(rec_g, li, p_k, q_k);
    (void)q_own;
    const bool stepk = li < n;
    const unsigned fb = __ballot_sync(0xffffffffu, stepk && fabs(p_k) <= tau) & gmask;
    const int info = fb ? (__ffs(fb) - g * L) : 0;
    const int nswap = __popc(__ballot_sync(0xffffffffu, stepk && q_k != li) & gmask);
    const int nneg = __popc(__ballot_sync(0xffffffffu, stepk && p_k < T(0)) & gmask);
    const double lg = ssum<L>(stepk ? log_abs(p_k) : 0.0);
    if (item_ok && stepk && a.ipiv) a.ipiv[(item0 + g) * n + li] = q_k + 1;
    if (item_ok && li == 0) {
      const int64_t item = item0 + g;
      if (a.info) a.info[item] = info;
      if (a.logabsdet) a.logabsdet[item] = info ? -INFINITY : lg;
      if (a.sign) a.sign[item] = info ? 0 : (int8_t)(((nswap ^ nneg) & 1) ? -1 : 1);
    }
    // ---- a7 + a8: X[k][:] = (row pivoted at step k)[B part] / p_k
    if (real) {
      const T rp = rcp(p_own);
      T* dst = sb + (g * NP + pos) * (NR + 1);
#pragma unroll
      for (int j = 0; j < NR; ++j)
        if (j < m) dst[j] = b[j] * rp;
    }
    __syncwarp();
    move_rows<T, NR + 1, false>(Xg + item0 * n * m, sb, vi * n, m, n, NP, lane);
    __syncwarp();
  }
}

template <typename T, int NP, int NR>
cudaError_t launch_solve_t(const SolveArgs& a, cudaStream_t s) {
  using S = SolveSmem<T, NP, NR>;
  const int smem = kSolveWarps * S::per_warp;
  static unsigned long long configured = 0;   // > 48 KB for fp64 with many right-hand sides
  const unsigned long long dbit = device_bit();
  if (!(configured & dbit)) {
    cudaError_t e = cudaFuncSetAttribute(gj_solve_kernel<T, NP, NR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    configured |= dbit;
  }
  const int64_t ntasks = (a.batch + S::MPW - 1) / S::MPW;
  const int64_t need = (ntasks + kSolveWarps - 1) / kSolveWarps;
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gj_solve_kernel<T, NP, NR>, kSolveWarps * 32, smem);
  if (e != cudaSuccess) return e;
  const int64_t cap = (int64_t)device_sm_count() * (per_sm > 0 ? per_sm : 1);
  const int grid = (int)(need < cap ? need : cap);
  gj_solve_kernel<T, NP, NR><<<grid, kSolveWarps * 32, smem, s>>>(a);
  return cudaGetLastError();
}

template <typename T, int NP>
cudaError_t launch_solve_np(const SolveArgs& a, cudaStream_t s) {
  if (a.m <= 1) return launch_solve_t<T, NP, 1>(a, s);
  if (a.m <= 4) return launch_solve_t<T, NP, 4>(a, s);
  if (a.m <= 8) return launch_solve_t<T, NP, 8>(a, s);
  if (a.m <= 16) return launch_solve_t<T, NP, 16>(a, s);
  return launch_solve_t<T, NP, 32>(a, s);
}

template <typename T>
cudaError_t launch_solve_dt(const SolveArgs& a, cudaStream_t s) {
  if (a.n <= 4) return launch_solve_np<T, 4>(a, s);
  if (a.n <= 8) return launch_solve_np<T, 8>(a, s);
  if (a.n <= 16) return launch_solve_np<T, 16>(a, s);
  return launch_solve_np<T, 32>(a, s);
}

}  // namespace

cudaError_t launch_solve_batched(gj_dtype dt, const SolveArgs& a, cudaStream_t s) {
  if (a.n < 1 || a.n > 32 || a.m < 1 || a.m > 32) return cudaErrorInvalidValue;
  if (dt == GJ_F32) {
    const cudaError_t e = launch_blk32_solve(a, s);
    if (e != cudaErrorNotSupported) return e;
  }
  return dt == GJ_F32 ? launch_solve_dt<float>(a, s) : launch_solve_dt<double>(a, s);
}

}  // namespace gj
