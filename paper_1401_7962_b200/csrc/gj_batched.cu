// K1 — batched Gauss–Jordan inversion for n <= 32 on sm_100a: one matrix per group of
// NP lanes (NP = next power of two >= n, so 32/NP matrices per warp), lane = matrix row,
// the row held in registers for the whole elimination.
//
// Per step k (§2, Eqs. (14)-(15), L61-L72; listing L150-L177), per group:
//   a2  pivot search over the rows not yet pivoted: max |x_ik| via one redux.sync on the
//       IEEE bit pattern of |x| (monotone for non-negative floats; fp64: high word, then
//       low word); among equal candidates the row at the smallest PHYSICAL position wins
//       (second redux.sync min) — exactly the listing's first-maximum scan over the
//       physically swapped rows k..n (L151-L153, Obs. 3 L60; reading G3).
//   a3  logical swap: rows never move; each lane tracks the physical position its row
//       would have in the listing's swapped array, which yields LAPACK-style ipiv (the
//       listing's p[k] = j, L154) and, at the end, the step at which the row was pivot.
//   a4  pivot-row normalisation is DEFERRED: the pivot row is published un-normalised and
//       keeps the scale 1/p; every other row uses f_i = x_ik * (1/p), which is exactly the
//       multiplier of Eq. (15) (-a_ik^{k-1} times a_kj^k = a_kj^{k-1} / p).
//   a5  x_ij -= f_i * x_rj for j != k (Eq. (15)), FFMA2 (fma.rn.f32x2) for fp32; compact
//       storage: column k becomes the new D column (-f_i; 1 on the pivot row).
//   a6  log|det| = sum log|p_k| (fp64), sign = (-1)^swaps * prod sign(p_k) (Eq. (13), G4).
//   a7  un-permutation on store: Ainv[k][perm[k']] = (1/p_{perm[k]}) * X[perm[k]][k']
//       (the listing's reverse-order column swaps L179-L198 as one gather/scatter).
// I/O: for n = NP (powers of two) and 16-byte aligned buffers, each warp streams its 32
// rows per task with TMA (cp.async.bulk.tensor, 128/64/32-byte swizzle so that every
// lane's row read and the scatter are bank-conflict free) double-buffered against the
// compute; the output is staged in the same buffer and written with a TMA store.
// Other n use coalesced vector loads into a padded staging buffer.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cmath>
#include <cstdint>

#include "gj_internal.h"

namespace gj {
namespace {

constexpr int kWarpsPerBlock = 4;

// ------------------------------------------------------------------ small PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// All lanes wait, then reconverge (the per-lane try_wait loop may exit at different
// iterations; everything after it relies on a converged warp).
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
  __syncwarp();
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, int c0, int r0, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(r0), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* tm, int c0, int r0, const void* src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(tm)),
               "r"(c0), "r"(r0), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

// 1/p: MUFU approximation + one Newton step (branch-free, within 1 ulp; exact for powers
// of two).  fp64 keeps the IEEE round-to-nearest reciprocal.
__device__ __forceinline__ float rcp_rn(float p) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(p));
  const float e = fmaf(-p, r, 1.0f);
  return fmaf(r, e, r);
}
__device__ __forceinline__ double rcp_rn(double p) { return __drcp_rn(p); }

// Largest T <= t (t >= 0), so that |p| <= tau is decided exactly in T's precision.
__device__ __forceinline__ float round_down_to(double t, float) { return __double2float_rd(t); }
__device__ __forceinline__ double round_down_to(double t, double) { return t; }

template <int NP>
__device__ __forceinline__ double group_max(double v) {
#pragma unroll
  for (int o = NP / 2; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
template <int NP>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int o = NP / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ------------------------------------------------------------------ a5: elimination
// x[j] -= f * y[j] for j != K; fp32 pairs use FFMA2.
__device__ __forceinline__ void ffma2(float& x0, float& x1, float nf, float y0, float y1) {
  unsigned long long xv, yv, fv;
  asm("mov.b64 %0, {%1,%2};" : "=l"(xv) : "f"(x0), "f"(x1));
  asm("mov.b64 %0, {%1,%2};" : "=l"(yv) : "f"(y0), "f"(y1));
  asm("mov.b64 %0, {%1,%1};" : "=l"(fv) : "f"(nf));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(xv) : "l"(fv), "l"(yv));
  asm("mov.b64 {%0,%1}, %2;" : "=f"(x0), "=f"(x1) : "l"(xv));
}

template <int NP, int K>
__device__ __forceinline__ void elim_pair(float (&x)[NP], const float (&y)[NP], float nf, int j) {
  if (j != K && j + 1 != K) {
    ffma2(x[j], x[j + 1], nf, y[j], y[j + 1]);
  } else if (j == K) {
    x[j + 1] = fmaf(nf, y[j + 1], x[j + 1]);
  } else {
    x[j] = fmaf(nf, y[j], x[j]);
  }
}
// The pair holding column K+1 (the next step's pivot column) goes first so the next
// pivot search can start while the rest of the update is still issuing.
template <int NP, int K>
__device__ __forceinline__ void eliminate(float (&x)[NP], const float (&y)[NP], float nf) {
  constexpr int first = ((K + 1) % NP) & ~1;
  elim_pair<NP, K>(x, y, nf, first);
#pragma unroll
  for (int j = 0; j + 1 < NP; j += 2)
    if (j != first) elim_pair<NP, K>(x, y, nf, j);
}
template <int NP, int K>
__device__ __forceinline__ void eliminate(double (&x)[NP], const double (&y)[NP], double nf) {
  constexpr int first = (K + 1) % NP;
  if (first != K) x[first] = fma(nf, y[first], x[first]);
#pragma unroll
  for (int j = 0; j < NP; ++j)
    if (j != K && j != first) x[j] = fma(nf, y[j], x[j]);
}

// ------------------------------------------------------------------ configuration
// R rows per lane (two rows share every pivot-row load and every publish/search
// instruction), L = NP/R lanes per matrix, MPW matrices per warp, ROWS = 32*R rows
// per warp task.
template <typename T, int NP>
struct Cfg {
  static constexpr int R = (NP >= 4 && NP * (int)sizeof(T) * 2 <= 256) ? 2 : 1;
  static constexpr int L = NP / R;
  static constexpr int MPW = 32 / L;
  static constexpr int ROWS = MPW * NP;
};

// ------------------------------------------------------------------ shared-memory layouts
// TMA path: the warp's ROWS rows stored as REG regions of [ROWS rows][SPAN bytes], each
// swizzled like CU_TENSOR_MAP_SWIZZLE_{SPAN}B (16-byte chunk index ^= address bits 7+).
template <typename T, int NP>
struct TmaLayout {
  static constexpr int ROWS = Cfg<T, NP>::ROWS;
  static constexpr int RB = NP * (int)sizeof(T);        // row bytes
  static constexpr int SPAN = RB < 128 ? RB : 128;       // swizzle span
  static constexpr int REG = RB / SPAN;                  // regions (TMA boxes) per row
  static constexpr int BOX_COLS = SPAN / (int)sizeof(T);
  static constexpr int BYTES = ROWS * RB;                // one stage buffer
  static constexpr int SWZ_MASK = SPAN == 128 ? 7 : SPAN == 64 ? 3 : SPAN == 32 ? 1 : 0;
  // used with RB >= 16 only (launch_np instantiates the TMA path for such rows)
  // per-row part of the address: row*SPAN and the XOR applied to the in-span byte offset
  __device__ static __forceinline__ uint32_t row_base(int row) { return (uint32_t)(row * SPAN); }
  __device__ static __forceinline__ uint32_t row_xor(int row) {
    return (((uint32_t)(row * SPAN) >> 7) & SWZ_MASK) << 4;
  }
  __device__ static __forceinline__ uint32_t off(uint32_t rb, uint32_t rx, int byte_in_row) {
    return (uint32_t)((byte_in_row / SPAN) * ROWS * SPAN) + rb + (((uint32_t)(byte_in_row % SPAN)) ^ rx);
  }
};

// Generic path: padded rows (pitch NP+1 elements), linear.
template <typename T, int NP, bool TMA>
struct Smem {
  using C = Cfg<T, NP>;
  static constexpr int PITCH = NP + 1;
  static constexpr int STAGE_BYTES = TMA ? TmaLayout<T, NP>::BYTES : C::ROWS * PITCH * (int)sizeof(T);
  static constexpr int NBUF = TMA ? 2 : 1;
  static constexpr int STAGE_ALIGNED = (STAGE_BYTES + 1023) / 1024 * 1024;
  static constexpr int PROW_BYTES = 2 * C::MPW * NP * (int)sizeof(T);
  static constexpr int PERM_BYTES = C::MPW * NP * 4;
  static constexpr int per_warp =
      ((NBUF * STAGE_ALIGNED + PROW_BYTES + PERM_BYTES + 16 * NBUF) + 1023) / 1024 * 1024;
};

template <typename T, int NP, bool TMA>
struct RowAddr {
  uint32_t rb = 0, rx = 0;
  __device__ __forceinline__ RowAddr() {}
  __device__ __forceinline__ explicit RowAddr(int row) {
    if constexpr (TMA) {
      rb = TmaLayout<T, NP>::row_base(row);
      rx = TmaLayout<T, NP>::row_xor(row);
    } else {
      rb = (uint32_t)(row * (NP + 1) * (int)sizeof(T));
      rx = 0;
    }
  }
  __device__ __forceinline__ uint32_t at(int col) const {
    if constexpr (TMA) {
      return TmaLayout<T, NP>::off(rb, rx, col * (int)sizeof(T));
    } else {
      return rb + (uint32_t)(col * (int)sizeof(T));
    }
  }
};

// Read a whole row (NP values) from the staging buffer.
template <typename T, int NP, bool TMA>
__device__ __forceinline__ void stage_ld_row(T (&x)[NP], const unsigned char* stage, int row) {
  const RowAddr<T, NP, TMA> ra(row);
  if constexpr (TMA) {
    constexpr int V = 16 / sizeof(T);
#pragma unroll
    for (int j = 0; j < NP; j += V) {
      const uint4 u = *reinterpret_cast<const uint4*>(stage + ra.at(j));
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
    for (int j = 0; j < NP; ++j) x[j] = *reinterpret_cast<const T*>(stage + ra.at(j));
  }
}

template <typename T, int NP>
__device__ __forceinline__ void st_row(T* dst, const T (&x)[NP]) {
  if constexpr ((NP * sizeof(T)) % 16 == 0) {
#pragma unroll
    for (int j = 0; j < NP; j += 16 / (int)sizeof(T)) {
      if constexpr (sizeof(T) == 4) {
        *reinterpret_cast<float4*>(dst + j) = make_float4(x[j], x[j + 1], x[j + 2], x[j + 3]);
      } else {
        *reinterpret_cast<double2*>(dst + j) = make_double2(x[j], x[j + 1]);
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < NP; ++j) dst[j] = x[j];
  }
}
template <typename T, int NP>
__device__ __forceinline__ void ld_row(T (&y)[NP], const T* src) {
  if constexpr ((NP * sizeof(T)) % 16 == 0) {
#pragma unroll
    for (int j = 0; j < NP; j += 16 / (int)sizeof(T)) {
      if constexpr (sizeof(T) == 4) {
        const float4 v = *reinterpret_cast<const float4*>(src + j);
        y[j] = v.x; y[j + 1] = v.y; y[j + 2] = v.z; y[j + 3] = v.w;
      } else {
        const double2 v = *reinterpret_cast<const double2*>(src + j);
        y[j] = v.x; y[j + 1] = v.y;
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < NP; ++j) y[j] = src[j];
  }
}

struct TmaMaps {
  CUtensorMap a, x;
};

// ------------------------------------------------------------------ a2: pivot search (R rows/lane)
// Per-matrix (lane-group) reductions.  redux.sync is only fast with a warp-uniform
// member mask, so with two matrices per warp each group runs a full-warp redux in which
// the other group contributes the identity; with more groups a shuffle butterfly over
// the group's L lanes is cheaper.
template <int MPW, int L>
__device__ __forceinline__ uint32_t group_max_u32(uint32_t v, int g) {
  if constexpr (MPW == 1) {
    return __reduce_max_sync(0xffffffffu, v);
  } else if constexpr (MPW == 2) {
    const uint32_t a = __reduce_max_sync(0xffffffffu, g == 0 ? v : 0u);
    const uint32_t b = __reduce_max_sync(0xffffffffu, g == 1 ? v : 0u);
    return g ? b : a;
  } else {
#pragma unroll
    for (int o = L / 2; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
  }
}
template <int MPW, int L>
__device__ __forceinline__ uint32_t group_min_u32(uint32_t v, int g) {
  if constexpr (MPW == 1) {
    return __reduce_min_sync(0xffffffffu, v);
  } else if constexpr (MPW == 2) {
    const uint32_t a = __reduce_min_sync(0xffffffffu, g == 0 ? v : 0xffffffffu);
    const uint32_t b = __reduce_min_sync(0xffffffffu, g == 1 ? v : 0xffffffffu);
    return g ? b : a;
  } else {
#pragma unroll
    for (int o = L / 2; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
  }
}

// On return q = physical position of the pivot row (uniform over the group) and
// is_piv[r] marks the slot holding it.
template <int R, int MPW, int L>
__device__ __forceinline__ void pivot_search(const float (&v)[R], const bool (&used)[R], const int (&pos)[R],
                                             int g, int& q, bool (&is_piv)[R]) {
  uint32_t key[R];
  uint32_t km = 0;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    key[r] = used[r] ? 0u : (__float_as_uint(v[r]) & 0x7fffffffu);
    km = max(km, key[r]);
  }
  const uint32_t m = group_max_u32<MPW, L>(km, g);
  uint32_t pc = 0xffffu;
#pragma unroll
  for (int r = 0; r < R; ++r)
    if (!used[r] && key[r] == m) pc = min(pc, (uint32_t)pos[r]);
  q = (int)group_min_u32<MPW, L>(pc, g);
#pragma unroll
  for (int r = 0; r < R; ++r) is_piv[r] = (pos[r] == q) && !used[r] && key[r] == m;
}

template <int R, int MPW, int L>
__device__ __forceinline__ void pivot_search(const double (&v)[R], const bool (&used)[R], const int (&pos)[R],
                                             int g, int& q, bool (&is_piv)[R]) {
  uint32_t hi[R], lo[R];
  uint32_t hm = 0;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v[r]) & 0x7fffffffffffffffull;
    hi[r] = used[r] ? 0u : (uint32_t)(b >> 32);
    lo[r] = used[r] ? 0u : (uint32_t)b;
    hm = max(hm, hi[r]);
  }
  const uint32_t mh = group_max_u32<MPW, L>(hm, g);
  uint32_t lm = 0;
#pragma unroll
  for (int r = 0; r < R; ++r)
    if (hi[r] == mh) lm = max(lm, lo[r]);
  const uint32_t ml = group_max_u32<MPW, L>(lm, g);
  uint32_t pc = 0xffffu;
#pragma unroll
  for (int r = 0; r < R; ++r)
    if (!used[r] && hi[r] == mh && lo[r] == ml) pc = min(pc, (uint32_t)pos[r]);
  q = (int)group_min_u32<MPW, L>(pc, g);
#pragma unroll
  for (int r = 0; r < R; ++r) is_piv[r] = (pos[r] == q) && !used[r] && hi[r] == mh && lo[r] == ml;
}

// Predicated row store (no branch, so the unrolled steps stay one basic block).
template <typename T, int NP>
__device__ __forceinline__ void st_row_if(bool pred, T* dst, const T (&x)[NP]) {
  if constexpr ((NP * sizeof(T)) % 16 == 0) {
    const uint32_t a = smem_u32(dst);
    const uint32_t p = pred ? 1u : 0u;
#pragma unroll
    for (int j = 0; j < NP; j += 16 / (int)sizeof(T)) {
      if constexpr (sizeof(T) == 4) {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %0, 0;\n\t@p st.shared.v4.f32 [%1], {%2, %3, %4, %5};\n}"
                     ::"r"(p), "r"(a + 4u * j), "f"(x[j]), "f"(x[j + 1]), "f"(x[j + 2]), "f"(x[j + 3]) : "memory");
      } else {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %0, 0;\n\t@p st.shared.v2.f64 [%1], {%2, %3};\n}"
                     ::"r"(p), "r"(a + 8u * j), "d"(x[j]), "d"(x[j + 1]) : "memory");
      }
    }
  } else {
    if (pred) st_row<T, NP>(dst, x);
  }
}

// Rotated elimination update.  The k loop is rolled (two steps per iteration) and the
// register file is kept ROTATED so that the pivot column of the first step of a pair is
// always register 0 and of the second step register 1: the second step writes its
// results two registers to the left (x'[j] = x[j+2] - f*y[j+2]) and appends the two new
// D columns at the end.  After NP steps (NP even) the rotation is back to identity and
// register j holds compact column j (the D column of step j).
// fp32 pairs stay 8-byte aligned (rotation by 2), so FFMA2 is used throughout.
template <int NP>
__device__ __forceinline__ void update_first(float (&x)[NP], const float (&y)[NP], float nf) {
  x[1] = fmaf(nf, y[1], x[1]);
#pragma unroll
  for (int j = 2; j < NP; j += 2) ffma2(x[j], x[j + 1], nf, y[j], y[j + 1]);
}
template <int NP>
__device__ __forceinline__ void update_first(double (&x)[NP], const double (&y)[NP], double nf) {
#pragma unroll
  for (int j = 1; j < NP; ++j) x[j] = fma(nf, y[j], x[j]);
}
template <int NP>
__device__ __forceinline__ void update_second_rot(float (&x)[NP], const float (&y)[NP], float nf, float dcol) {
  const float c0 = fmaf(nf, y[0], x[0]);
#pragma unroll
  for (int j = 0; j + 3 < NP; j += 2) {
    float a = x[j + 2], b = x[j + 3];
    ffma2(a, b, nf, y[j + 2], y[j + 3]);
    x[j] = a;
    x[j + 1] = b;
  }
  x[NP - 2] = c0;
  x[NP - 1] = dcol;
}
template <int NP>
__device__ __forceinline__ void update_second_rot(double (&x)[NP], const double (&y)[NP], double nf, double dcol) {
  const double c0 = fma(nf, y[0], x[0]);
#pragma unroll
  for (int j = 0; j + 2 < NP; ++j) x[j] = fma(nf, y[j + 2], x[j + 2]);
  x[NP - 2] = c0;
  x[NP - 1] = dcol;
}

// One elimination step (a2-a5) at runtime step index k; the pivot column is register
// PC (0 or 1); SECOND selects the rotating update.
template <typename T, int NP, int PC, bool SECOND>
__device__ __forceinline__ void gj_step(int k, int n, T (&x)[Cfg<T, NP>::R][NP], T* prow_g,
                                        bool (&used)[Cfg<T, NP>::R], int (&pos)[Cfg<T, NP>::R],
                                        T (&myrp)[Cfg<T, NP>::R], int (&myipiv)[Cfg<T, NP>::R], int& info, T tau,
                                        int li, int g) {
  using C = Cfg<T, NP>;
  constexpr int R = C::R;
  T col[R];
#pragma unroll
  for (int r = 0; r < R; ++r) col[r] = x[r][PC];
  int q;
  bool is_piv[R];
  pivot_search<R, C::MPW, C::L>(col, used, pos, g, q, is_piv);
  // a3: listing's swap of rows k and q (L156-L162), tracked on positions only
#pragma unroll
  for (int r = 0; r < R; ++r) {
    if (li + r * C::L == k) myipiv[r] = q + 1;
    if (pos[r] == k) pos[r] = q;
  }
  // a4: publish the pivot row (one buffer per step of the pair: one __syncwarp per step)
  T* pr = prow_g + PC * C::MPW * NP;
#pragma unroll
  for (int r = 0; r < R; ++r) st_row_if<T, NP>(is_piv[r], pr, x[r]);
  __syncwarp();
  T y[NP];
  ld_row<T, NP>(y, pr);
  const T p = y[PC];
  // Obs. 2: largest candidate at or below the zero threshold -> singular at step k+1
  if (fabs(p) <= tau && info == 0 && k < n) info = k + 1;
  const T rp = rcp_rn(p);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    if (is_piv[r]) {
      pos[r] = k;
      used[r] = true;
      myrp[r] = rp;
    }
    // a5: Eq. (15) with the deferred pivot-row scale; column k becomes the D column
    const T nf = is_piv[r] ? T(0) : -(x[r][PC] * rp);
    const T dcol = is_piv[r] ? T(1) : nf;
    if constexpr (!SECOND) {
      update_first<NP>(x[r], y, nf);
      x[r][0] = dcol;
    } else {
      update_second_rot<NP>(x[r], y, nf, dcol);
    }
  }
}

template <int L>
__device__ __forceinline__ unsigned lane_group_mask(int lane) {
  if constexpr (L == 32) {
    return 0xffffffffu;
  } else {
    return ((1u << L) - 1u) << (lane & ~(L - 1));
  }
}

template <typename T, int NP, bool TMA>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
gj_batched_warp_kernel(BatchedArgs a, const __grid_constant__ TmaMaps tm) {
  using C = Cfg<T, NP>;
  using S = Smem<T, NP, TMA>;
  using TL = TmaLayout<T, (TMA ? NP : 4 * (int)(16 / sizeof(T)))>;   // only used when TMA
  constexpr int R = C::R, L = C::L, MPW = C::MPW, ROWS = C::ROWS;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  // 1024-byte alignment for the swizzled TMA boxes (the launch adds 1 KB of slack)
  unsigned char* sbase = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* wbase = sbase + warp * S::per_warp;
  unsigned char* stage0 = wbase;
  T* prow = reinterpret_cast<T*>(wbase + S::NBUF * S::STAGE_ALIGNED);
  int* permS = reinterpret_cast<int*>(reinterpret_cast<unsigned char*>(prow) + S::PROW_BYTES);
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(permS) + S::PERM_BYTES);

  const int n = TMA ? NP : a.n;
  const int nn = n * n;
  const int g = lane / L;        // matrix within the warp task
  const int li = lane % L;       // slot r holds row li + r*L
  const unsigned gmask = lane_group_mask<L>(lane);
  const T* __restrict__ Ag = static_cast<const T*>(a.A);
  T* __restrict__ Xg = static_cast<T*>(a.Ainv);
  T* prow_g = prow + g * NP;     // + (k&1)*MPW*NP selects the buffer

  const int64_t ntasks = (a.batch + MPW - 1) / MPW;
  const int64_t wstride = (int64_t)gridDim.x * kWarpsPerBlock;
  const int64_t task0 = (int64_t)blockIdx.x * kWarpsPerBlock + warp;

  if constexpr (TMA) {
    if (lane == 0) {
      mbar_init(&bars[0], 1);
      mbar_init(&bars[1], 1);
      fence_mbar_init();
    }
    __syncwarp();
    if (lane == 0 && task0 < ntasks) {
      mbar_expect_tx(&bars[0], TL::BYTES);
#pragma unroll
      for (int rg = 0; rg < TL::REG; ++rg)
        tma_load_2d(stage0 + rg * ROWS * TL::SPAN, &tm.a, rg * TL::BOX_COLS, (int)(task0 * ROWS), &bars[0]);
    }
  }

  int it = 0;
  for (int64_t task = task0; task < ntasks; task += wstride, ++it) {
    const int64_t item0 = task * MPW;
    const int64_t left = a.batch - item0;
    const int valid_items = left < MPW ? (int)left : MPW;
    unsigned char* stage = stage0 + (TMA ? (it & 1) * S::STAGE_ALIGNED : 0);

    // ---- a1: load ----
    if constexpr (TMA) {
      const int64_t nxt = task + wstride;
      if (lane == 0 && nxt < ntasks) {
        unsigned char* ns = stage0 + ((it + 1) & 1) * S::STAGE_ALIGNED;
        bulk_wait_read0();   // the TMA store that last read `ns` has finished reading smem
        mbar_expect_tx(&bars[(it + 1) & 1], TL::BYTES);
#pragma unroll
        for (int rg = 0; rg < TL::REG; ++rg)
          tma_load_2d(ns + rg * ROWS * TL::SPAN, &tm.a, rg * TL::BOX_COLS, (int)(nxt * ROWS), &bars[(it + 1) & 1]);
      }
      mbar_wait(&bars[it & 1], (it >> 1) & 1);
    } else {
      const int tot = valid_items * nn;
      const int64_t gofs = item0 * nn;
      for (int e0 = 0; e0 < tot; e0 += 256) {
        T v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int e = e0 + u * 32 + lane;
          v[u] = e < tot ? __ldcs(Ag + gofs + e) : T(0);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int e = e0 + u * 32 + lane;
          if (e < tot) {
            const int m = e / nn;
            const int rem = e - m * nn;
            const int r = rem / n;
            *reinterpret_cast<T*>(stage + RowAddr<T, NP, false>(m * NP + r).at(rem - r * n)) = v[u];
          }
        }
      }
      __syncwarp();
    }
    T x[R][NP];
    bool real[R];
    const bool item_ok = g < valid_items;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int row = li + r * L;
      real[r] = row < n;
      stage_ld_row<T, NP, TMA>(x[r], stage, g * NP + row);
      if (!TMA || !item_ok) {
#pragma unroll
        for (int j = 0; j < NP; ++j) {
          const bool rl = item_ok && real[r] && j < n;
          if (!rl) x[r][j] = (row == j) ? T(1) : T(0);
        }
      }
    }
    __syncwarp();   // staging buffer fully read: free for the output scatter

    // zero threshold tau = tol * max|a_ij| (Obs. 2, reading G1)
    T rowmax = T(0);
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int j = 0; j < NP; ++j)
        if (real[r] && j < n) rowmax = fmax(rowmax, fabs(x[r][j]));
    const T tau = round_down_to(a.tol * group_max<L>((double)rowmax), T(0));

    bool used[R];
    int pos[R];      // physical position; after the loop = the step this row was pivot
    T myrp[R];       // 1/p of that step (deferred normalisation scale)
    int myipiv[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      used[r] = false;      // padding rows only ever win the padded steps k >= n
      pos[r] = li + r * L;
      myrp[r] = T(1);
      myipiv[r] = li + r * L + 1;
    }
    int info = 0;
    // padded steps k >= n pick the (identity) padding rows and change nothing real
#pragma unroll 1
    for (int k = 0; k < NP; k += 2) {
      gj_step<T, NP, 0, false>(k, n, x, prow_g, used, pos, myrp, myipiv, info, tau, li, g);
      gj_step<T, NP, 1, true>(k + 1, n, x, prow_g, used, pos, myrp, myipiv, info, tau, li, g);
    }

    // ---- a6: determinant (Eq. (13) with the swap sign, G4) ----
    double lgl = 0.0;
    int nneg = 0, nswap = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (real[r]) lgl -= log(fabs((double)myrp[r]));
      nneg += __popc(__ballot_sync(0xffffffffu, real[r] && myrp[r] < T(0)) & gmask);
      nswap += __popc(__ballot_sync(0xffffffffu, real[r] && myipiv[r] != li + r * L + 1) & gmask);
    }
    const double lg = group_sum<L>(lgl);
    const int sgn = ((nswap ^ nneg) & 1) ? -1 : 1;
    if (item_ok) {
      const int64_t item = item0 + g;
      if (li == 0) {
        if (a.info) a.info[item] = info;
        if (a.logabsdet) a.logabsdet[item] = info ? -INFINITY : lg;
        if (a.sign) a.sign[item] = info ? 0 : (int8_t)sgn;
        if (a.det) static_cast<T*>(a.det)[item] = info ? T(0) : (T)(sgn * exp(lg));
      }
      if (a.ipiv) {
#pragma unroll
        for (int r = 0; r < R; ++r)
          if (real[r]) a.ipiv[item * n + li + r * L] = myipiv[r];
      }
    }

    // ---- a7 + a8: un-permuted store through the staging buffer ----
    if (Xg != nullptr) {
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (real[r]) permS[g * NP + pos[r]] = li + r * L;
      __syncwarp();
      RowAddr<T, NP, TMA> dst[R];
#pragma unroll
      for (int r = 0; r < R; ++r) dst[r] = RowAddr<T, NP, TMA>(g * NP + pos[r]);
#pragma unroll
      for (int kp = 0; kp < NP; ++kp) {
        if (kp < n) {
          const int c = permS[g * NP + kp];
#pragma unroll
          for (int r = 0; r < R; ++r)
            if (real[r]) *reinterpret_cast<T*>(stage + dst[r].at(c)) = myrp[r] * x[r][kp];
        }
      }
      if constexpr (TMA) {
        fence_async_smem();
        __syncwarp();
        if (lane == 0) {
#pragma unroll
          for (int rg = 0; rg < TL::REG; ++rg)
            tma_store_2d(&tm.x, rg * TL::BOX_COLS, (int)(task * ROWS), stage + rg * ROWS * TL::SPAN);
          bulk_commit();
        }
      } else {
        __syncwarp();
        const int tot = valid_items * nn;
        const int64_t gofs = item0 * nn;
        for (int e = lane; e < tot; e += 32) {
          const int m = e / nn;
          const int rem = e - m * nn;
          const int r = rem / n;
          __stcs(Xg + gofs + e, *reinterpret_cast<const T*>(stage + RowAddr<T, NP, false>(m * NP + r).at(rem - r * n)));
        }
      }
    }
    __syncwarp();
  }
  if constexpr (TMA) {
    if (lane == 0) bulk_wait0();
  }
}

// ------------------------------------------------------------------ host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

template <typename T, int NP>
bool make_map(CUtensorMap* m, const void* base, int64_t batch) {
  using TL = TmaLayout<T, NP>;
  EncodeTiledFn enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)NP, (cuuint64_t)(batch * NP)};
  cuuint64_t strides[1] = {(cuuint64_t)NP * sizeof(T)};
  cuuint32_t box[2] = {(cuuint32_t)TL::BOX_COLS, (cuuint32_t)TL::ROWS};
  cuuint32_t es[2] = {1u, 1u};
  CUtensorMapSwizzle sw = TL::SPAN == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                          : TL::SPAN == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                          : TL::SPAN == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                           : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUtensorMapDataType dt = sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
  return enc(m, dt, 2, const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <typename T, int NP, bool TMA>
cudaError_t launch_warp(const BatchedArgs& a, const TmaMaps& maps, cudaStream_t s) {
  using S = Smem<T, NP, TMA>;
  const size_t smem = (size_t)S::per_warp * kWarpsPerBlock + 1024;
  auto kern = gj_batched_warp_kernel<T, NP, TMA>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kWarpsPerBlock * 32, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const int64_t ntasks = (a.batch + Cfg<T, NP>::MPW - 1) / Cfg<T, NP>::MPW;
  const int64_t need = (ntasks + kWarpsPerBlock - 1) / kWarpsPerBlock;
  const int64_t cap = (int64_t)device_sm_count() * per_sm;
  const int grid = (int)(need < cap ? need : cap);
  kern<<<grid, kWarpsPerBlock * 32, smem, s>>>(a, maps);
  return cudaGetLastError();
}

template <typename T, int NP>
cudaError_t launch_np(const BatchedArgs& a, cudaStream_t s) {
  TmaMaps maps;
  const bool full = a.n == NP;
  const bool aligned = (reinterpret_cast<uintptr_t>(a.A) % 16 == 0) &&
                       (a.Ainv == nullptr || reinterpret_cast<uintptr_t>(a.Ainv) % 16 == 0);
  const bool rows_ok = (NP * sizeof(T)) % 16 == 0 && a.batch * NP < (int64_t(1) << 31);
  if constexpr ((NP * sizeof(T)) % 16 == 0) {
    if (full && aligned && rows_ok && make_map<T, NP>(&maps.a, a.A, a.batch) &&
        (a.Ainv == nullptr || make_map<T, NP>(&maps.x, a.Ainv, a.batch))) {
      if (a.Ainv == nullptr) maps.x = maps.a;
      return launch_warp<T, NP, true>(a, maps, s);
    }
  }
  return launch_warp<T, NP, false>(a, maps, s);
}

template <typename T>
cudaError_t dispatch_np(const BatchedArgs& a, cudaStream_t s) {
  const int n = a.n;
  if (n <= 2) return launch_np<T, 2>(a, s);   // n = 1 runs padded to 2
  if (n <= 4) return launch_np<T, 4>(a, s);
  if (n <= 8) return launch_np<T, 8>(a, s);
  if (n <= 16) return launch_np<T, 16>(a, s);
  if (n <= 32) return launch_np<T, 32>(a, s);
  return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t launch_batched(gj_dtype dt, const BatchedArgs& a, cudaStream_t s) {
  if (a.batch == 0) return cudaSuccess;
  if (a.n <= 32) return dt == GJ_F32 ? dispatch_np<float>(a, s) : dispatch_np<double>(a, s);
  return cudaErrorInvalidValue;
}

}  // namespace gj
