// K1 — batched Gauss–Jordan inversion for n <= 32 on sm_100a.
//
// One matrix per group of NP lanes (NP = next power of two >= n; 32/NP matrices per
// warp), lane i holds row i of the compact working array in registers for the whole
// elimination.  Per step k (§2, Eqs. (14)-(15), L61-L72; listing L150-L177):
//   a2  pivot search over the rows not yet pivoted: max |x_ik| by one redux.sync on the
//       IEEE bit pattern of |x| (monotone for non-negative floats; fp64: high word then
//       low word); among equal candidates the row at the smallest PHYSICAL position wins
//       (second redux.sync, min) — exactly the listing's first-maximum scan over the
//       physically swapped rows k..n (L151-L153, Obs. 3 L60; reading G3).
//   a3  logical swap: rows never move; each lane tracks the position its row would have
//       in the listing's swapped array (swap k <-> q, L156-L162).  One lane records
//       (p, q) per step in shared memory: ipiv, the swap parity, the singular flag and
//       log|det| are all derived from that record after the loop.
//   a4  pivot-row normalisation is DEFERRED: the pivot lane publishes its row
//       un-normalised; every other row uses f_i = x_ik * (1/p), which is exactly the
//       multiplier of Eq. (15) (-a_ik^{k-1} times a_kj^k = a_kj^{k-1}/p); each row is
//       scaled by 1/p of its own pivot step once, at the store.
//   a5  x_ij -= f_i x_rj (Eq. (15)) with FFMA2 (fma.rn.f32x2) for fp32; compact storage:
//       column k becomes the new D column (-f_i, and 1 on the pivot row).
//   The k loop is rolled, two steps per iteration, with the register file ROTATED: the
//   pivot column of the first step of a pair is register 0, of the second register 1,
//   and the second step writes its results two registers to the left (x'[j] = x[j+2] -
//   f y[j+2]) appending the two new D columns at the end.  After NP steps register j
//   holds compact column j.  (The loop body stays ~100 instructions per step pair: no
//   I-cache pressure.)  n < NP runs padded with identity rows/columns: padded steps pick
//   the padding rows and change nothing real.
//   a6  log|det| = sum log|p_k| (fp64), sign = (-1)^swaps prod sign(p_k) (Eq. (13), G4).
//   a7  un-permutation on store: Ainv[k][perm[k']] = (1/p_{perm[k]}) X[perm[k]][k'] (the
//       listing's reverse-order column swaps, L179-L198, as one gather/scatter).
// fp32 n = 32 runs the blocked K1b (blk_panel_step, BS = 4); a call without ipiv runs it in
// two passes (K1f, launch_blk32): first with the pivot row taken from ballots when it is
// unique — no positions, no tie-break — giving a task up at its first exact tie, then the
// exact kernel over the tasks given up (bitwise the same outputs).
// I/O: for n = NP and 16-byte aligned buffers each warp streams its 32 rows per task with
// TMA (cp.async.bulk.tensor; 128/64/32-byte swizzle so every lane's row read and the
// scatter are bank-conflict free), double-buffered against the compute; the output is
// staged in the same buffer and written with a TMA store.  Other n use coalesced vector
// loads into a padded staging buffer.
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

#ifndef GJ_K1_WPB
#define GJ_K1_WPB 4
#endif
constexpr int kWarpsPerBlock = GJ_K1_WPB;   // warps per CTA of the batched kernels (A/B build option)
// K1b block loop unrolling (build option -DGJ_K1B_UNROLL=n, A/B measurements)
#ifndef GJ_K1B_LDS64
#define GJ_K1B_LDS64 0
#endif
#ifndef GJ_K1B_WSYNC
#define GJ_K1B_WSYNC 0
#endif
#if GJ_K1B_WSYNC
#define K1B_SYNC() asm volatile("bar.warp.sync 0xffffffff;" ::: "memory")
#else
#define K1B_SYNC() __syncwarp()
#endif
#ifndef GJ_K1B_NST
#define GJ_K1B_NST 2   // TMA stages per warp (A/B build option: 1 = 16 warps per SM at 128 registers)
#endif
#ifndef GJ_K1B_PUB1
#define GJ_K1B_PUB1 1   // the block publish as one asm block of predicated stores (A/B option)
#endif
#ifndef GJ_K1B_PUBM
#define GJ_K1B_PUBM 1   // block publish with the two register slots merged (A/B option)
#endif
#ifndef GJ_K1B_UNROLL
#define GJ_K1B_UNROLL 1
#endif
constexpr int kK1bUnroll = GJ_K1B_UNROLL;

// R rows per lane: two rows share every pivot-row load (halving the shared-memory
// traffic of the broadcast, which bounds the fp32 n = 32 case); L = NP/R lanes per matrix.
template <typename T, int NP>
struct Cfg {
  static constexpr int R = (NP == 32 && sizeof(T) == 4) ? 2 : 1;
  static constexpr int L = NP / R;      // lanes per matrix
  static constexpr int MPW = 32 / L;    // matrices per warp
  static constexpr int ROWS = MPW * NP; // rows per warp task
};

// ------------------------------------------------------------------ group reductions
// redux.sync is only fast with a warp-uniform member mask: one matrix per warp uses it
// directly, two matrices run one full-warp redux per group (the other group contributes
// the identity), more groups use a shuffle butterfly over the group's lanes.
// A/B build options (round 2 measurements, tools/time_c2_lib.py on C2, bitwise-equal
// outputs): GJ_K1_GRPREDUX=1 reduces each 16-lane group with a non-uniform member mask instead
// of two full-warp reductions (4.76 ms against 3.53: the masked redux's ~168-cycle latency sits
// on the pivot chain); GJ_K1_RECPRED=1 (default) stores the per-step record with one predicated
// st.shared instead of an `if (li == 0)` branch (3.485 against 3.531 ms).
#ifndef GJ_K1_GRPREDUX
#define GJ_K1_GRPREDUX 0
#endif
#ifndef GJ_K1_RECPRED
#define GJ_K1_RECPRED 1
#endif
template <int MPW, int L>
__device__ __forceinline__ uint32_t group_max_u32(uint32_t v, int g) {
  if constexpr (MPW == 2 && GJ_K1_GRPREDUX) {
    return __reduce_max_sync(g ? 0xffff0000u : 0x0000ffffu, v);
  } else if constexpr (MPW == 1) {
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
  if constexpr (MPW == 2 && GJ_K1_GRPREDUX) {
    return __reduce_min_sync(g ? 0xffff0000u : 0x0000ffffu, v);
  } else if constexpr (MPW == 1) {
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
template <int L>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int o = L / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <int L>
__device__ __forceinline__ unsigned lane_group_mask(int lane) {
  if constexpr (L == 32) {
    return 0xffffffffu;
  } else {
    return ((1u << L) - 1u) << (lane & ~(L - 1));
  }
}

// ------------------------------------------------------------------ a2: pivot search
// Eligible rows carry kmask = all ones, pivoted rows kmask = 0.  On return q = the pivot
// row's physical position (group-uniform) and is_piv[r] marks the slot holding it.
template <int R, int MPW, int L>
__device__ __forceinline__ void pivot_search(const float (&v)[R], const uint32_t (&kmask)[R], const int (&pos)[R],
                                             int g, int& q, bool (&is_piv)[R]) {
  uint32_t key[R];
  uint32_t km = 0;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    key[r] = __float_as_uint(v[r]) & 0x7fffffffu & kmask[r];
    km = max(km, key[r]);
  }
  const uint32_t m = group_max_u32<MPW, L>(km, g);
  uint32_t pc = 0xffffu;
#pragma unroll
  for (int r = 0; r < R; ++r)
    if (key[r] == m && kmask[r] != 0u) pc = min(pc, (uint32_t)pos[r]);
  q = (int)group_min_u32<MPW, L>(pc, g);
#pragma unroll
  for (int r = 0; r < R; ++r) is_piv[r] = pos[r] == q;
}
template <int R, int MPW, int L>
__device__ __forceinline__ void pivot_search(const double (&v)[R], const uint32_t (&kmask)[R], const int (&pos)[R],
                                             int g, int& q, bool (&is_piv)[R]) {
  uint32_t hi[R], lo[R];
  uint32_t hm = 0;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v[r]);
    hi[r] = (uint32_t)(b >> 32) & 0x7fffffffu & kmask[r];
    lo[r] = (uint32_t)b & kmask[r];
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
    if (hi[r] == mh && lo[r] == ml && kmask[r] != 0u) pc = min(pc, (uint32_t)pos[r]);
  q = (int)group_min_u32<MPW, L>(pc, g);
#pragma unroll
  for (int r = 0; r < R; ++r) is_piv[r] = pos[r] == q;
}

// ------------------------------------------------------------------ shared-memory layouts
// TMA path: the warp's 32 rows stored as REG regions of [32 rows][SPAN bytes], each
// swizzled like CU_TENSOR_MAP_SWIZZLE_{SPAN}B (16-byte chunk index ^= address bits 7+).
template <typename T, int NP>
struct TmaLayout {
  static constexpr int ROWS = Cfg<T, NP>::ROWS;
  static constexpr int RB = NP * (int)sizeof(T);   // row bytes (>= 16 on this path)
  static constexpr int SPAN = RB < 128 ? RB : 128;  // swizzle span
  static constexpr int REG = RB / SPAN;             // regions (TMA boxes) per row
  static constexpr int BOX_COLS = SPAN / (int)sizeof(T);
  static constexpr int BYTES = ROWS * RB;           // one stage buffer
  static constexpr int SWZ_MASK = SPAN == 128 ? 7 : SPAN == 64 ? 3 : SPAN == 32 ? 1 : 0;
};

template <typename T, int NP, bool TMA>
struct Smem {
  static constexpr int ROWS = Cfg<T, NP>::ROWS;
  static constexpr int STAGE_BYTES = TMA ? ROWS * NP * (int)sizeof(T) : ROWS * (NP + 1) * (int)sizeof(T);
  static constexpr int NBUF = TMA ? 2 : 1;
  static constexpr int STAGE_ALIGNED = (STAGE_BYTES + 1023) / 1024 * 1024;
  static constexpr int PROW_BYTES = 2 * ROWS * (int)sizeof(T);   // two pivot-row buffers (all groups)
  static constexpr int REC_BYTES = ROWS * 16;                     // per-step (p, q) record
  static constexpr int PERM_BYTES = ROWS * 4;
  static constexpr int per_warp =
      ((NBUF * STAGE_ALIGNED + PROW_BYTES + REC_BYTES + PERM_BYTES + 16 * NBUF) + 1023) / 1024 * 1024;
};

// Address of (row, col) inside a staging buffer: per-row part (rb, rx) + column bytes.
template <typename T, int NP, bool TMA>
struct RowAddr {
  uint32_t rb = 0, rx = 0;
  __device__ __forceinline__ explicit RowAddr(int row) {
    if constexpr (TMA) {
      using TL = TmaLayout<T, NP>;
      rb = (uint32_t)(row * TL::SPAN);
      rx = ((rb >> 7) & TL::SWZ_MASK) << 4;
    } else {
      rb = (uint32_t)(row * (NP + 1) * (int)sizeof(T));
    }
  }
  __device__ __forceinline__ uint32_t at_b(uint32_t cb) const {
    if constexpr (TMA) {
      using TL = TmaLayout<T, NP>;
      if constexpr (TL::REG == 1) {
        return rb + (cb ^ rx);
      } else {
        return (cb / TL::SPAN) * (TL::ROWS * TL::SPAN) + rb + ((cb % TL::SPAN) ^ rx);
      }
    } else {
      return rb + cb;
    }
  }
};

template <typename T, int NP, bool TMA>
__device__ __forceinline__ void stage_ld_row(T (&x)[NP], const unsigned char* stage, int row) {
  const RowAddr<T, NP, TMA> ra(row);
  if constexpr (TMA) {
    constexpr int V = 16 / sizeof(T);
#pragma unroll
    for (int j = 0; j < NP; j += V) {
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
    for (int j = 0; j < NP; ++j) x[j] = *reinterpret_cast<const T*>(stage + ra.at_b(j * sizeof(T)));
  }
}

struct TmaMaps {
  CUtensorMap a, x;
};

// One elimination step (a2-a5) at runtime step index k; pivot column = register PC.
template <typename T, int NP, int PC, bool SECOND>
__device__ __forceinline__ void gj_step(int k, T (&x)[Cfg<T, NP>::R][NP], T* prow_g, unsigned char* rec_g,
                                        uint32_t (&kmask)[Cfg<T, NP>::R], int (&pos)[Cfg<T, NP>::R], int li, int g) {
  using C = Cfg<T, NP>;
  constexpr int R = C::R;
  T col[R];
#pragma unroll
  for (int r = 0; r < R; ++r) col[r] = x[r][PC];
  int q;
  bool is_piv[R];
  pivot_search<R, C::MPW, C::L>(col, kmask, pos, g, q, is_piv);
  // a3: the listing's swap of rows k and q (L156-L162), on positions only
#pragma unroll
  for (int r = 0; r < R; ++r) {
    if (pos[r] == k) pos[r] = q;
    if (is_piv[r]) pos[r] = k;
  }
  // a4: publish the (un-normalised) pivot row; one buffer per step of the pair
  T* pr = prow_g + PC * C::MPW * NP;
#pragma unroll
  for (int r = 0; r < R; ++r) st_row_if<T, NP>(is_piv[r], pr, x[r]);
  __syncwarp();
  T y[NP];
  ld_row<T, NP>(y, pr);
  const T p = y[PC];
  if (li == 0) rec_store(rec_g, k, p, q);
  const T rp = rcp(p);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    kmask[r] = is_piv[r] ? 0u : kmask[r];
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

template <typename T, int NP, bool TMA>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
gj_batched_warp_kernel(BatchedArgs a, const __grid_constant__ TmaMaps tm) {
  using C = Cfg<T, NP>;
  using S = Smem<T, NP, TMA>;
  using TL = TmaLayout<T, (TMA ? NP : 16 / (int)sizeof(T))>;   // only used when TMA
  constexpr int L = C::L, MPW = C::MPW, R = C::R, ROWS = C::ROWS;
  constexpr int RECW = sizeof(T) == 4 ? 8 : 16;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  // 1024-byte alignment for the swizzled TMA boxes (the launch adds 1 KB of slack)
  unsigned char* sbase = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* wbase = sbase + warp * S::per_warp;
  unsigned char* stage0 = wbase;
  T* prow = reinterpret_cast<T*>(wbase + S::NBUF * S::STAGE_ALIGNED);
  unsigned char* rec = reinterpret_cast<unsigned char*>(prow) + S::PROW_BYTES;
  int* permS = reinterpret_cast<int*>(rec + S::REC_BYTES);
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(permS) + S::PERM_BYTES);

  const int n = TMA ? NP : a.n;
  const int nn = n * n;
  const int g = lane / L;        // matrix within the warp task
  const int li = lane % L;       // row within the matrix
  const unsigned gmask = lane_group_mask<L>(lane);
  const T* __restrict__ Ag = static_cast<const T*>(a.A);
  T* __restrict__ Xg = static_cast<T*>(a.Ainv);
  T* prow_g = prow + g * NP;
  unsigned char* rec_g = rec + g * NP * RECW;   // one record of NP steps per matrix
  int* perm_g = permS + g * NP;

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

    // ---- a1: load the task's rows into the staging buffer ----
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
      mbar_wait_warp(&bars[it & 1], (it >> 1) & 1);
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
            *reinterpret_cast<T*>(stage + RowAddr<T, NP, false>(m * NP + r).at_b((rem - r * n) * sizeof(T))) = v[u];
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
        for (int j = 0; j < NP; ++j)
          if (!(item_ok && real[r] && j < n)) x[r][j] = (row == j) ? T(1) : T(0);
      }
    }
    __syncwarp();   // staging buffer fully read: free for the output scatter

    // zero threshold tau = tol * max|a_ij| (Obs. 2, reading G1); padding excluded
    T rowmax = T(0);
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int j = 0; j < NP; ++j)
        if (real[r] && j < n) rowmax = fmax(rowmax, fabs(x[r][j]));
    double smax;
    if constexpr (sizeof(T) == 4) {
      smax = (double)__uint_as_float(group_max_u32<MPW, L>(__float_as_uint(rowmax), g));
    } else {
      // exact max of non-negative doubles: high words, then low words among the winners
      const unsigned long long b = (unsigned long long)__double_as_longlong(rowmax);
      const uint32_t mh = group_max_u32<MPW, L>((uint32_t)(b >> 32), g);
      const uint32_t ml = group_max_u32<MPW, L>((uint32_t)(b >> 32) == mh ? (uint32_t)b : 0u, g);
      smax = __longlong_as_double((long long)(((unsigned long long)mh << 32) | ml));
    }
    const T tau = round_down_to(a.tol * smax, T(0));

    uint32_t kmask[R];
    int pos[R];   // physical position; after the loop = the step this row was pivot
#pragma unroll
    for (int r = 0; r < R; ++r) {
      kmask[r] = 0xffffffffu;
      pos[r] = li + r * L;
    }
    // padded steps k >= n pick the (identity) padding rows and change nothing real
#pragma unroll 1
    for (int k = 0; k < NP; k += 2) {
      gj_step<T, NP, 0, false>(k, x, prow_g, rec_g, kmask, pos, li, g);
      gj_step<T, NP, 1, true>(k + 1, x, prow_g, rec_g, kmask, pos, li, g);
    }
    __syncwarp();

    // ---- a6: det / ipiv / singular flag from the per-step record ----
    T myrp[R];
    unsigned failb = 0;
    int nswap = 0, nneg = 0;
    double lgl = 0.0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int row = li + r * L;
      T p_own, p_k;
      int q_own, q_k;
      rec_load(rec_g, pos[r], p_own, q_own);   // this row's own pivot step
      rec_load(rec_g, row, p_k, q_k);          // step `row` of the record
      (void)q_own;
      myrp[r] = rcp(p_own);
      const bool stepk = row < n;
      // steps li + r*L: bit li of slot r's ballot; first failing step = lowest (r, li)
      const unsigned fb = __ballot_sync(0xffffffffu, stepk && fabs(p_k) <= tau) & gmask;
      if (failb == 0 && fb != 0) failb = (unsigned)(__ffs(fb) - g * L + r * L);
      nswap += __popc(__ballot_sync(0xffffffffu, stepk && q_k != row) & gmask);
      nneg += __popc(__ballot_sync(0xffffffffu, stepk && p_k < T(0)) & gmask);
      if (stepk) lgl += log_abs(p_k);
      if (a.ipiv && item_ok && stepk) a.ipiv[(item0 + g) * n + row] = q_k + 1;
    }
    const int info = (int)failb;   // first failing step, 1-based (0: regular)
    const double lg = group_sum<L>(lgl);
    const int sgn = ((nswap ^ nneg) & 1) ? -1 : 1;
    if (item_ok && li == 0) {
      const int64_t item = item0 + g;
      if (a.info) a.info[item] = info;
      if (a.logabsdet) a.logabsdet[item] = info ? -INFINITY : lg;
      if (a.sign) a.sign[item] = info ? 0 : (int8_t)sgn;
      if (a.det) static_cast<T*>(a.det)[item] = info ? T(0) : (T)(sgn * exp(lg));
    }

    // ---- a7 + a8: un-permuted store through the staging buffer ----
    if (Xg != nullptr) {
#pragma unroll
      for (int r = 0; r < R; ++r) perm_g[pos[r]] = (li + r * L) * (int)sizeof(T);   // output column (bytes)
      __syncwarp();
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const RowAddr<T, NP, TMA> dst(g * NP + pos[r]);
        if constexpr (NP >= 4) {
#pragma unroll
          for (int kp = 0; kp < NP; kp += 4) {
            const int4 cb = *reinterpret_cast<const int4*>(perm_g + kp);
            const int cbs[4] = {cb.x, cb.y, cb.z, cb.w};
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (real[r] && kp + u < n)
                *reinterpret_cast<T*>(stage + dst.at_b((uint32_t)cbs[u])) = myrp[r] * x[r][kp + u];
          }
        } else {
#pragma unroll
          for (int kp = 0; kp < NP; ++kp)
            if (real[r] && kp < n) *reinterpret_cast<T*>(stage + dst.at_b((uint32_t)perm_g[kp])) = myrp[r] * x[r][kp];
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
          __stcs(Xg + gofs + e,
                 *reinterpret_cast<const T*>(stage + RowAddr<T, NP, false>(m * NP + r).at_b((rem - r * n) * sizeof(T))));
        }
      }
    }
    __syncwarp();
  }
  if constexpr (TMA) {
    if (lane == 0) bulk_wait0();
  }
}

// ------------------------------------------------------------------ K1b: blocked, fp32 n = 32
// The same elimination taken in blocks of BS steps (the aggregation of Eqs. (14)-(15) the
// large-n path uses, applied inside one register-resident matrix).  Within a block, step
// s only updates the BS panel columns (all the next pivot search needs); the pivot row's
// panel values travel by one shuffle each.  At the end of the block the BS pivot rows'
// other 32-BS values — untouched since the block began — are published to shared memory
// ONCE and every row applies the block's BS rank-1 updates to its other columns at once:
//     x_i[J'] += sum_s (W_is - S_is) R_s[J']
// (W = the panel's compact columns after the block, R_s = the block-start row pivoted at
// step s, S_is = 1 iff row i is that row; DESIGN.md §7 derives it).  The panel registers
// hold W - S directly: a pivot row's own compact entry starts at 1 - 1 = 0, later updates
// are additive, and the 1 is added back at the store.  Why: the per-step publish of a
// whole pivot row (8 predicated STS.128 per slot, 4 smem cycles each whatever the lane
// count; tools/ubench/smem_bench.cu) bounded the unblocked K1; here it happens once per
// block.  Tie-break, logical swaps, record and epilogue are K1's.
// R rows per lane (R = 2: 16 lanes and 2 matrices per warp; R = 4: 8 lanes and 4
// matrices per warp: every shared-memory read of the trailing update then feeds four rows).
template <int R>
struct BlkGeo {
  static constexpr int L = 32 / R;       // lanes per matrix
  static constexpr int M = R;            // matrices per warp task
  static constexpr int ROWS = 32 * M;    // rows per warp task
  static constexpr int STAGE = ROWS * 128;
};

template <int R, int BS>
struct BlkMisc {
  static constexpr int RW = 32 - BS;
  static constexpr int RBUF = BlkGeo<R>::M * BS * RW * 4;   // [matrix][block step][RW] pivot-row tails
  static constexpr int REC = BlkGeo<R>::M * 32 * 8;         // [matrix][step] (p, q)
  static constexpr int PERM = BlkGeo<R>::M * 32 * 4;
  static constexpr int BYTES = RBUF + REC + PERM + 16;
  static constexpr int smem(int nst) { return kWarpsPerBlock * (nst * BlkGeo<R>::STAGE + BYTES) + 1024; }
};

// group reductions over the L lanes of a matrix
template <int R>
__device__ __forceinline__ uint32_t blk_gmax(uint32_t v, int g) {
  return group_max_u32<BlkGeo<R>::M, BlkGeo<R>::L>(v, g);
}
template <int R>
__device__ __forceinline__ uint32_t blk_gmin(uint32_t v, int g) {
  return group_min_u32<BlkGeo<R>::M, BlkGeo<R>::L>(v, g);
}

// One panel step s (static) at global step k on the panel registers P (branch-free, so
// that a whole block stays one basic block and the scheduler can interleave the previous
// block's trailing update into the latency of this chain).
// FAST (K1f, the pass that assumes no exact ties): the pivot row of each matrix is the one
// row whose key equals the group maximum, found from two ballots; no physical positions are
// tracked (pos[] holds the step at which the row was pivoted) and the record keeps only p.
// A step where some matrix of the warp has more than one row at its maximum (an exact tie,
// or an all-zero column) sets `tie`; the task is then discarded and redone by the exact
// kernel (the tie-break G3 needs the positions).  Without a tie both variants take the same
// pivot and do the same arithmetic, so their outputs are bitwise equal.
template <int R, int BS, bool FAST>
__device__ __forceinline__ void blk_panel_step(const int s, const int k, float (&P)[R][BS], uint32_t (&kmask)[R],
                                               int (&pos)[R], int (&bs)[R], unsigned& tie, float (&pblk)[BS],
                                               unsigned char* rec_g, int li, int g, int lane) {
  constexpr int SB = R == 2 ? 1 : 2;   // slot bits in the winner code
  constexpr int L = BlkGeo<R>::L;
  // a2: max |x_ik| over the un-pivoted rows (IEEE bit pattern of |x|, monotone)
  uint32_t key[R];
  uint32_t km = 0;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    key[r] = __float_as_uint(P[r][s]) & kmask[r];
    km = max(km, key[r]);
  }
  const uint32_t m = blk_gmax<R>(km, g);
  // |1/p| and the unsigned multipliers start while the tie-break runs (|p| = m exactly)
  const float ra = rcp(__uint_as_float(m));
  float t[R];
#pragma unroll
  for (int r = 0; r < R; ++r) t[r] = P[r][s] * ra;
  int q, src, slot;
  bool pv[R];
  if constexpr (FAST) {
    // every matrix has at least one row at its maximum, so a total of M candidates over the
    // warp means exactly one per matrix
    unsigned ball[R], any = 0;
    int tot = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      pv[r] = key[r] == m;
      ball[r] = __ballot_sync(0xffffffffu, pv[r]);
      tot += __popc(ball[r]);
      any |= ball[r];
    }
    tie |= (unsigned)(tot != BlkGeo<R>::M);
    const unsigned gm = (L == 32 ? 0xffffffffu : ((1u << L) - 1u)) << (L * g);
    const unsigned su = 31u - (unsigned)__clz(any & gm);   // FLO: the candidate's lane
    src = (int)su;
    slot = 0;
#pragma unroll
    for (int r = 1; r < R; ++r) slot = (ball[r] & gm) ? r : slot;
    q = src;   // recorded in place of the position (K1f's epilogue reads only p from the record)
  } else {
    // ties -> smallest physical position (G3); the winner code carries (position, lane, slot)
    uint32_t cmin = 0xffffffu;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const uint32_t c = (key[r] == m && kmask[r] != 0u)
                             ? ((uint32_t)pos[r] << (5 + SB) | (uint32_t)lane << SB | (uint32_t)r) : 0xffffffu;
      cmin = min(cmin, c);
    }
    const uint32_t win = blk_gmin<R>(cmin, g);
    q = (int)(win >> (5 + SB));
    src = (int)((win >> SB) & 31u);
    slot = (int)(win & ((1u << SB) - 1u));
#pragma unroll
    for (int r = 0; r < R; ++r) pv[r] = pos[r] == q;
  }
  // the pivot row's panel values (one shuffle each from the pivot lane)
  float z[BS];
#pragma unroll
  for (int j = 0; j < BS; ++j) {
    float v = P[0][j];
#pragma unroll
    for (int r = 1; r < R; ++r) v = slot == r ? P[r][j] : v;
    z[j] = __shfl_sync(0xffffffffu, v, src);
  }
  const float p = z[s];
  const uint32_t psign = __float_as_uint(p) & 0x80000000u;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    // a5 on the panel: Eq. (15) with the deferred pivot-row scale, multiplier x_ik / p
    const float nf = pv[r] ? 0.0f : __uint_as_float((__float_as_uint(t[r]) ^ psign) ^ 0x80000000u);
#pragma unroll
    for (int j = 0; j < BS; j += 2) {
      if (j == s) {
        P[r][j + 1] = fmaf(nf, z[j + 1], P[r][j + 1]);
      } else if (j + 1 == s) {
        P[r][j] = fmaf(nf, z[j], P[r][j]);
      } else {
        ffma2(P[r][j], P[r][j + 1], nf, z[j], z[j + 1]);
      }
    }
    P[r][s] = nf;   // compact D entry; 0 on the pivot row (W - S: its 1 is held as 0)
    kmask[r] = pv[r] ? 0u : kmask[r];
    bs[r] = pv[r] ? s : bs[r];
    if constexpr (FAST) {
      // pos[] (the step this row is pivoted at = its final position) is set from bs[] once
      // per block, where the block's pivot rows are published (k0_pos_from_bs)
    } else {
      // a3: the listing's swap of positions k and q (L156-L162), positions only
      pos[r] = (pos[r] == k) ? q : pos[r];
      pos[r] = pv[r] ? k : pos[r];
    }
  }
  if constexpr (FAST) {
    (void)q;
    pblk[s] = p;   // K1f: the block's four pivots are recorded at once (rec_store_block)
  } else if constexpr (GJ_K1_RECPRED) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.eq.u32 p, %0, 0;\n\t@p st.shared.v2.u32 [%1], {%2, %3};\n}" ::"r"(li),
                 "r"(smem_u32(rec_g) + 8u * k), "r"(__float_as_uint(p)), "r"(q)
                 : "memory");
  } else {
    if (li == 0) rec_store(rec_g, k, p, q);
  }
}

// K1f's record: p of steps k0 .. k0 + 3 as one 16-byte store by the group's lane 0 (the
// record is then p only, 4 bytes per step; one store per block instead of one per step)
__device__ __forceinline__ void rec_store_block(unsigned char* rec_g, int k0, const float (&pb)[4], int li) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.eq.u32 p, %0, 0;\n\t@p st.shared.v4.f32 [%1], {%2, %3, %4, %5};\n}" ::"r"(li),
               "r"(smem_u32(rec_g) + 4u * k0), "f"(pb[0]), "f"(pb[1]), "f"(pb[2]), "f"(pb[3])
               : "memory");
}

// K1f: the steps of block k0's pivot rows, from their block-step slots
template <int R>
__device__ __forceinline__ void k0_pos_from_bs(int (&pos)[R], const int (&bs)[R], int k0) {
#pragma unroll
  for (int r = 0; r < R; ++r) pos[r] = bs[r] >= 0 ? k0 + bs[r] : pos[r];
}

// Seven predicated 16-byte shared stores of v[0..27] at dst (one asm block: ptxas keeps them
// predicated instead of turning the run into a branch ladder).
__device__ __forceinline__ void st7_if(bool pred, uint32_t dst, const float (&v)[28]) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %0, 0;\n\t"
      "@p st.shared.v4.f32 [%1], {%2, %3, %4, %5};\n\t"
      "@p st.shared.v4.f32 [%1+16], {%6, %7, %8, %9};\n\t"
      "@p st.shared.v4.f32 [%1+32], {%10, %11, %12, %13};\n\t"
      "@p st.shared.v4.f32 [%1+48], {%14, %15, %16, %17};\n\t"
      "@p st.shared.v4.f32 [%1+64], {%18, %19, %20, %21};\n\t"
      "@p st.shared.v4.f32 [%1+80], {%22, %23, %24, %25};\n\t"
      "@p st.shared.v4.f32 [%1+96], {%26, %27, %28, %29};\n}" ::"r"(pred ? 1u : 0u), "r"(dst),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
      "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]), "f"(v[17]), "f"(v[18]),
      "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]), "f"(v[25]), "f"(v[26]), "f"(v[27])
      : "memory");
}

// Publish the block's pivot rows: their other RW values T (unchanged since the block began).
template <int R, int BS>
__device__ __forceinline__ void blk_publish(const float (&T)[R][32 - BS], const int (&bs)[R], float* rbuf_g) {
  constexpr int RW = 32 - BS;
  if constexpr (R == 2 && RW == 28 && GJ_K1B_PUBM) {
    // merged slots: one store sequence carries the lane's (first) pivot row of the block, so
    // that the active lanes of both slots share each wavefront; the rare lane whose two rows
    // both pivot in the block stores its second one in a sequence that is predicated off
    // (no wavefront) everywhere else
    const bool p0 = bs[0] >= 0;
    const int sb = p0 ? bs[0] : bs[1];
    float D[28];
#pragma unroll
    for (int j = 0; j < 28; ++j) D[j] = p0 ? T[0][j] : T[1][j];
    st7_if(sb >= 0, smem_u32(rbuf_g) + (uint32_t)(sb < 0 ? 0 : sb) * (RW * 4), D);
    st7_if(p0 && bs[1] >= 0, smem_u32(rbuf_g) + (uint32_t)(bs[1] < 0 ? 0 : bs[1]) * (RW * 4), T[1]);
  } else {
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const uint32_t dst = smem_u32(rbuf_g) + (uint32_t)(bs[r] < 0 ? 0 : bs[r]) * (RW * 4);
    if constexpr (RW == 28 && GJ_K1B_PUB1) {
      // the seven predicated 16-byte stores in one asm block (one predicate)
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ge.s32 p, %0, 0;\n\t"
          "@p st.shared.v4.f32 [%1], {%2, %3, %4, %5};\n\t"
          "@p st.shared.v4.f32 [%1+16], {%6, %7, %8, %9};\n\t"
          "@p st.shared.v4.f32 [%1+32], {%10, %11, %12, %13};\n\t"
          "@p st.shared.v4.f32 [%1+48], {%14, %15, %16, %17};\n\t"
          "@p st.shared.v4.f32 [%1+64], {%18, %19, %20, %21};\n\t"
          "@p st.shared.v4.f32 [%1+80], {%22, %23, %24, %25};\n\t"
          "@p st.shared.v4.f32 [%1+96], {%26, %27, %28, %29};\n}" ::"r"(bs[r]), "r"(dst),
          "f"(T[r][0]), "f"(T[r][1]), "f"(T[r][2]), "f"(T[r][3]), "f"(T[r][4]), "f"(T[r][5]), "f"(T[r][6]),
          "f"(T[r][7]), "f"(T[r][8]), "f"(T[r][9]), "f"(T[r][10]), "f"(T[r][11]), "f"(T[r][12]), "f"(T[r][13]),
          "f"(T[r][14]), "f"(T[r][15]), "f"(T[r][16]), "f"(T[r][17]), "f"(T[r][18]), "f"(T[r][19]),
          "f"(T[r][20]), "f"(T[r][21]), "f"(T[r][22]), "f"(T[r][23]), "f"(T[r][24]), "f"(T[r][25]),
          "f"(T[r][26]), "f"(T[r][27])
          : "memory");
    } else {
#pragma unroll
      for (int j = 0; j < RW; j += 4)
        st_shared_v4_if(bs[r] >= 0, dst + 4u * j, T[r][j], T[r][j + 1], T[r][j + 2], T[r][j + 3]);
    }
  }
  }
}

// Rank-1 term s of the trailing update on columns [J0, J1) of T: T += (W - S)[:, s] R_s.
// SHIFT: write the result BS registers to the left (T[j - BS] = T[j] + ...), in increasing
// j, which realises the block's register rotation without moves (the last term does it).
template <int R, int BS, int J0, int J1, int N, bool SHIFT = false>
__device__ __forceinline__ void blk_trail_term(float (&T)[R][N], const float (&P)[R][BS], int s, const float* rbuf_g,
                                               int tofs) {
  constexpr int RW = 32 - BS;
  float Rs[J1 - J0];
  if constexpr (GJ_K1B_LDS64) {
    const uint32_t ab = smem_u32(rbuf_g + s * RW + J0);
#pragma unroll
    for (int j = 0; j < J1 - J0; j += 2)
      asm volatile("ld.volatile.shared.v2.f32 {%0, %1}, [%2];" : "=f"(Rs[j]), "=f"(Rs[j + 1]) : "r"(ab + 4u * j));
  } else {
    ld_row<float, J1 - J0>(Rs, rbuf_g + s * RW + J0);
  }
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int j = 0; j < J1 - J0; j += 2) {
      if constexpr (SHIFT) {
        float u0 = T[r][tofs + j], u1 = T[r][tofs + j + 1];
        ffma2(u0, u1, P[r][s], Rs[j], Rs[j + 1]);
        T[r][tofs + j - BS] = u0;
        T[r][tofs + j + 1 - BS] = u1;
      } else {
        ffma2(T[r][tofs + j], T[r][tofs + j + 1], P[r][s], Rs[j], Rs[j + 1]);
      }
    }
}

// Number of cycles of the permutation sigma of a matrix's 32 rows (row li + L r -> sig[r]; L = 16
// lanes x 2 rows): pointer jumping, 5 rounds, each row's label = the smallest row of its
// cycle; a row is its cycle's representative iff its label is itself.  (lab, next) travel
// packed in one word.
template <int L>
__device__ __forceinline__ int perm_cycles(const int (&sig)[2], int li, int g, unsigned gmask) {
  static_assert(L == 16, "two rows per lane");
  int lab[2] = {li, li + L}, nx[2] = {sig[0], sig[1]};
#pragma unroll
  for (int it = 0; it < 5; ++it) {
    const int pk0 = (lab[0] << 8) | nx[0], pk1 = (lab[1] << 8) | nx[1];
    int nl[2], nn[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int b = nx[r];
      const int srcl = (g * L) | (b & (L - 1));
      const int v0 = __shfl_sync(0xffffffffu, pk0, srcl), v1 = __shfl_sync(0xffffffffu, pk1, srcl);
      const int v = b >= L ? v1 : v0;
      nl[r] = min(lab[r], v >> 8);
      nn[r] = v & 0xff;
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      lab[r] = nl[r];
      nx[r] = nn[r];
    }
  }
  return __popc(__ballot_sync(0xffffffffu, lab[0] == li) & gmask) + __popc(__ballot_sync(0xffffffffu, lab[1] == li + L) & gmask);
}

// NST = TMA stages per warp: 2 = the next task streams in during this one; 1 = half the
// shared memory (more resident warps), the next task is prefetched into L2 instead.
// MODE (the two-pass run of launch_blk32, used when no ipiv is requested):
//   0  exact (G3 tie-break on physical positions) over every task;
//   1  K1f: FAST panel steps over every task; a task in which a step found an exact tie
//      writes nothing and is appended to tlist (tlist[0] = count, tlist[1..] = tasks);
//   2  exact over the tasks of tlist only (the tasks MODE 1 gave up, read from A again —
//      A is intact there even when the inverse aliases it).
template <int R, int BS, int NST, int MODE>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, (R == 4 ? 8 : (NST == 1 ? 16 : 12)) / kWarpsPerBlock)
gj_blk32_kernel(BatchedArgs a, const __grid_constant__ TmaMaps tm, int* __restrict__ tlist) {
  constexpr bool FAST = MODE == 1;
  if constexpr (MODE == 2) {
    if (tlist[0] == 0) return;   // the usual case: K1f met no tie
  }
  using Geo = BlkGeo<R>;
  using M = BlkMisc<R, BS>;
  constexpr int RW = M::RW, L = Geo::L, MT = Geo::M;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  unsigned char* sbase = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* stage0 = sbase + warp * NST * Geo::STAGE;
  unsigned char* misc = sbase + kWarpsPerBlock * NST * Geo::STAGE + warp * M::BYTES;
  float* rbuf = reinterpret_cast<float*>(misc);
  unsigned char* rec = misc + M::RBUF;
  int* permS = reinterpret_cast<int*>(rec + M::REC);
  uint64_t* bars = reinterpret_cast<uint64_t*>(misc + M::RBUF + M::REC + M::PERM);

  const int g = lane / L;
  const int li = lane % L;
  const unsigned gmask = (L == 32 ? 0xffffffffu : ((1u << L) - 1u)) << (L * g);
  float* rbuf_g = rbuf + g * BS * RW;
  unsigned char* rec_g = rec + g * 32 * 8;
  int* perm_g = permS + g * 32;

  // task index ti -> task (MODE 2: the list of tasks the FAST pass gave up)
  const int64_t ntasks = MODE == 2 ? (int64_t)tlist[0] : (a.batch + MT - 1) / MT;
  auto task_of = [&](int64_t ti) -> int64_t { return MODE == 2 ? (int64_t)tlist[1 + ti] : ti; };
  const int64_t wstride = (int64_t)gridDim.x * kWarpsPerBlock;
  const int64_t ti0 = (int64_t)blockIdx.x * kWarpsPerBlock + warp;

  if (lane == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  K1B_SYNC();
  if (lane == 0 && ti0 < ntasks) {
    mbar_expect_tx(&bars[0], Geo::STAGE);
    tma_load_2d(stage0, &tm.a, 0, (int)(task_of(ti0) * Geo::ROWS), &bars[0]);
  }

  int it = 0;
  for (int64_t ti = ti0; ti < ntasks; ti += wstride, ++it) {
    const int64_t task = task_of(ti);
    const int64_t item0 = task * MT;
    const bool item_ok = item0 + g < a.batch;
    unsigned char* stage = stage0 + (NST == 2 ? (it & 1) * Geo::STAGE : 0);
    const int64_t nti = ti + wstride;
    if constexpr (NST == 2) {
      if (lane == 0 && nti < ntasks) {
        unsigned char* ns = stage0 + ((it + 1) & 1) * Geo::STAGE;
        bulk_wait_read0();
        mbar_expect_tx(&bars[(it + 1) & 1], Geo::STAGE);
        tma_load_2d(ns, &tm.a, 0, (int)(task_of(nti) * Geo::ROWS), &bars[(it + 1) & 1]);
      }
      mbar_wait_warp(&bars[it & 1], (it >> 1) & 1);
    } else {
      if (lane == 0 && nti < ntasks)
        bulk_prefetch_l2(static_cast<const float*>(a.A) + task_of(nti) * Geo::ROWS * 32, Geo::STAGE);
      mbar_wait_warp(&bars[0], it & 1);
    }
    // ---- a1: rows li + L r of matrix g into registers ----
    float x[R][32];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int row = li + L * r;
      stage_ld_row<float, 32, true>(x[r], stage, g * 32 + row);
      if (!item_ok) {
#pragma unroll
        for (int j = 0; j < 32; ++j) x[r][j] = (row == j) ? 1.0f : 0.0f;
      }
    }
    K1B_SYNC();
    float rowmax = 0.0f;
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int j = 0; j < 32; ++j) rowmax = fmaxf(rowmax, fabsf(x[r][j]));
    const double smax = (double)__uint_as_float(blk_gmax<R>(__float_as_uint(rowmax), g));
    const float tau = round_down_to(a.tol * smax, 0.0f);

    uint32_t kmask[R];
    int pos[R], bs[R];
    unsigned tie = 0;
    // P: panel columns of the current block; T: the other 32 - BS columns, rotated so
    // that T[0..BS) is the next panel and the finished compact D columns sit at the end
    float P[R][BS], T[R][RW];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      kmask[r] = 0x7fffffffu;
      pos[r] = li + L * r;
      bs[r] = -1;
#pragma unroll
      for (int j = 0; j < BS; ++j) P[r][j] = x[r][j];
#pragma unroll
      for (int j = 0; j < RW; ++j) T[r][j] = x[r][BS + j];
    }
    float pb[BS];
#pragma unroll
    for (int s = 0; s < BS; ++s) blk_panel_step<R, BS, FAST>(s, s, P, kmask, pos, bs, tie, pb, rec_g, li, g, lane);
    if constexpr (FAST) rec_store_block(rec_g, 0, pb, li);
    // look-ahead: per iteration, publish block kb's pivot rows, apply its update to the
    // next panel first, then factor that panel while the rest of block kb's update runs
#pragma unroll kK1bUnroll
    for (int kb = 0; kb + BS < 32; kb += BS) {
      blk_publish<R, BS>(T, bs, rbuf_g);
      if constexpr (FAST) k0_pos_from_bs<R>(pos, bs, kb);
      K1B_SYNC();
      float NP[R][BS];
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int j = 0; j < BS; ++j) NP[r][j] = T[r][j];
#pragma unroll
      for (int s = 0; s < BS; ++s) blk_trail_term<R, BS, 0, BS, BS>(NP, P, s, rbuf_g, 0);
#pragma unroll
      for (int r = 0; r < R; ++r) bs[r] = -1;
#pragma unroll
      for (int s = 0; s < BS; ++s) {
        blk_panel_step<R, BS, FAST>(s, kb + BS + s, NP, kmask, pos, bs, tie, pb, rec_g, li, g, lane);
        if (s + 1 < BS)
          blk_trail_term<R, BS, BS, RW, RW>(T, P, s, rbuf_g, BS);
        else
          blk_trail_term<R, BS, BS, RW, RW, true>(T, P, s, rbuf_g, BS);   // + the rotation
      }
      if constexpr (FAST) rec_store_block(rec_g, kb + BS, pb, li);
      K1B_SYNC();   // every lane has read rbuf before the next publish
#pragma unroll
      for (int r = 0; r < R; ++r) {
#pragma unroll
        for (int j = 0; j < BS; ++j) {
          T[r][RW - BS + j] = P[r][j];
          P[r][j] = NP[r][j];
        }
      }
      // K1f gives a task up at the end of the block that met its first tie (warp-uniform):
      // the rest is not worth computing, the exact pass redoes the task
      if (FAST && tie) break;
    }
    // last block: its whole update, then x = [T | P] (register j = compact column j)
    blk_publish<R, BS>(T, bs, rbuf_g);
    if constexpr (FAST) k0_pos_from_bs<R>(pos, bs, 32 - BS);
    K1B_SYNC();
#pragma unroll
    for (int s = 0; s < BS; ++s) blk_trail_term<R, BS, 0, RW, RW>(T, P, s, rbuf_g, 0);
#pragma unroll
    for (int r = 0; r < R; ++r) {
#pragma unroll
      for (int j = 0; j < RW; ++j) x[r][j] = T[r][j];
#pragma unroll
      for (int j = 0; j < BS; ++j) x[r][RW + j] = P[r][j];
    }

    // ---- a6: det / ipiv / singular flag from the per-step record ----
    float myrp[R];
    unsigned failb = 0;
    int nswap = 0, nneg = 0;
    double lgl = 0.0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int row = li + L * r;
      float p_own, p_k;
      int q_own, q_k = 0;
      if constexpr (FAST) {
        p_own = reinterpret_cast<const float*>(rec_g)[pos[r]];
        p_k = reinterpret_cast<const float*>(rec_g)[row];
      } else {
        rec_load(rec_g, pos[r], p_own, q_own);
        rec_load(rec_g, row, p_k, q_k);
        (void)q_own;
      }
      myrp[r] = rcp(p_own);
      const unsigned fb = __ballot_sync(0xffffffffu, fabsf(p_k) <= tau) & gmask;
      if (failb == 0 && fb != 0) failb = (unsigned)(__ffs(fb) - g * L + r * L);
      if constexpr (!FAST) nswap += __popc(__ballot_sync(0xffffffffu, q_k != row) & gmask);
      nneg += __popc(__ballot_sync(0xffffffffu, p_k < 0.0f) & gmask);
      lgl += log_abs(p_k);
      if constexpr (!FAST) {
        if (a.ipiv && item_ok) a.ipiv[(item0 + g) * 32 + row] = q_k + 1;
      }
    }
    // K1f keeps no positions: the swaps' parity is that of the permutation row -> pivot step
    if constexpr (FAST) nswap = 32 - perm_cycles<L>(pos, li, g, gmask);
    const int info = (int)failb;
    const double lg = group_sum<L>(lgl);
    const int sgn = ((nswap ^ nneg) & 1) ? -1 : 1;
    if (item_ok && li == 0 && !tie) {
      const int64_t item = item0 + g;
      if (a.info) a.info[item] = info;
      if (a.logabsdet) a.logabsdet[item] = info ? -INFINITY : lg;
      if (a.sign) a.sign[item] = info ? 0 : (int8_t)sgn;
      if (a.det) static_cast<float*>(a.det)[item] = info ? 0.0f : (float)(sgn * exp(lg));
    }
    if constexpr (FAST) {
      // a task with an exact tie: nothing written; the exact pass redoes it (tie is warp-uniform)
      if (tie && lane == 0) tlist[1 + atomicAdd(tlist, 1)] = (int)task;
    }

    // ---- a7 + a8: un-permuted store through the staging buffer ----
    if (a.Ainv != nullptr && !tie) {
#pragma unroll
      for (int r = 0; r < R; ++r) perm_g[pos[r]] = (li + L * r) * 4;   // output column (bytes)
      K1B_SYNC();
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const RowAddr<float, 32, true> dst(g * 32 + pos[r]);
#pragma unroll
        for (int kp = 0; kp < 32; kp += 4) {
          const int4 cb = *reinterpret_cast<const int4*>(perm_g + kp);
          const int cbs[4] = {cb.x, cb.y, cb.z, cb.w};
#pragma unroll
          for (int u = 0; u < 4; ++u) *reinterpret_cast<float*>(stage + dst.at_b((uint32_t)cbs[u])) = myrp[r] * x[r][kp + u];
        }
        // the row's own compact entry was held as W - 1 (see above): add the 1 back
        float* own = reinterpret_cast<float*>(stage + dst.at_b((uint32_t)((li + L * r) * 4)));
        *own = *own + myrp[r];
      }
      fence_async_smem();
      K1B_SYNC();
      if (lane == 0) {
        tma_store_2d(&tm.x, 0, (int)(task * Geo::ROWS), stage);
        bulk_commit();
      }
    }
    K1B_SYNC();
    if constexpr (NST == 1) {
      if (lane == 0 && nti < ntasks) {
        bulk_wait_read0();   // the store has read the stage
        mbar_expect_tx(&bars[0], Geo::STAGE);
        tma_load_2d(stage0, &tm.a, 0, (int)(task_of(nti) * Geo::ROWS), &bars[0]);
      }
    }
  }
  if (lane == 0) bulk_wait0();
}

template <int R, int BS, int NST, int MODE>
cudaError_t launch_blk32_mode(const BatchedArgs& a, const TmaMaps& maps, int* tlist, cudaStream_t s) {
  const size_t smem = BlkMisc<R, BS>::smem(NST);
  auto kern = gj_blk32_kernel<R, BS, NST, MODE>;
  static unsigned long long configured = 0;
  const unsigned long long dbit = device_bit();
  if (!(configured & dbit)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured |= dbit;
  }
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kWarpsPerBlock * 32, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const int64_t ntasks = (a.batch + R - 1) / R;
  const int64_t need = (ntasks + kWarpsPerBlock - 1) / kWarpsPerBlock;
  const int64_t cap = (int64_t)device_sm_count() * per_sm;
  const int grid = (int)(need < cap ? need : cap);
  kern<<<grid, kWarpsPerBlock * 32, smem, s>>>(a, maps, tlist);
  return cudaGetLastError();
}

#ifndef GJ_K1F
#define GJ_K1F 1   // two-pass K1f + exact redo when no ipiv is requested (A/B build option)
#endif

// K1b entry.  Without ipiv (C2's outputs) it runs two passes: K1f over every task (no
// positions, no tie-break), then the exact kernel over the tasks in which K1f met an exact
// tie; the task list comes from a stream-ordered allocation of the library's memory pool.
// With ipiv (the LAPACK-style swap sequence needs the positions) it runs the exact kernel.
template <int R, int BS, int NST>
cudaError_t launch_blk32(const BatchedArgs& a, const TmaMaps& maps, cudaStream_t s) {
  if (GJ_K1F && a.ipiv == nullptr) {
    const int64_t ntasks = (a.batch + R - 1) / R;
    int* tl = static_cast<int*>(pool_alloc_async((size_t)(ntasks + 1) * sizeof(int), s));
    if (tl != nullptr) {
      cudaError_t e = cudaMemsetAsync(tl, 0, sizeof(int), s);
      if (e == cudaSuccess) e = launch_blk32_mode<R, BS, NST, 1>(a, maps, tl, s);
      if (e == cudaSuccess) e = launch_blk32_mode<R, BS, NST, 2>(a, maps, tl, s);
      const cudaError_t f = cudaFreeAsync(tl, s);
      return e != cudaSuccess ? e : f;
    }
  }
  return launch_blk32_mode<R, BS, NST, 0>(a, maps, nullptr, s);
}

// ------------------------------------------------------------------ K1s: blocked solve / det, fp32 n = 32
// [A | B] -> [diag(p) | P B] by K1b's blocked elimination (R = 2 rows per lane, two
// matrices per warp, BS = 4, the same panel step, tie-break, record and look-ahead), but
// nothing left of the current panel is kept: the compact D columns are dropped (the
// "skip the D half" of SURVEY.md §8f f4 — the det-only and solve variants never need
// A^-1), so block KB's trailing update covers only the columns right of the next panel plus
// the NR right-hand-side columns.  The eight blocks are unrolled (static column ranges, no
// register rotation).  At the end the row pivoted at step k holds p_k x_k (Eq. (12) with B
// in place of I): X[k][:] = b_row / p_k, a row gather.  NR = 0 is the determinant-only run.
struct BlkSolveArgs {
  int64_t batch;
  int m;                // right-hand sides actually present (<= NR)
  const float* B;       // [batch][32][m]
  float* X;             // [batch][32][m], may alias B
  int32_t* ipiv;
  double* logabsdet;
  int8_t* sign;
  float* det;
  int32_t* info;
  double tol;
};

template <int NR>
struct SolveBlk {
  static constexpr int R = 2, BS = 4, NST = 2;
  static constexpr int NRP = NR == 0 ? 0 : (NR + 3) / 4 * 4;
  static constexpr int RS = 32 + NRP;                                // pivot-row record: absolute column, then B
  static constexpr int RBUF = BlkGeo<R>::M * BS * RS * 4;
  static constexpr int REC = BlkGeo<R>::M * 32 * 8;
  static constexpr int BYTES = RBUF + REC + 16;
  static constexpr int smem() { return kWarpsPerBlock * (NST * BlkGeo<R>::STAGE + BYTES) + 1024; }
};

// the pivot rows of block KB publish their columns [(KB + 1) BS, 32) and their B part
template <int NR, int KB>
__device__ __forceinline__ void slv_publish(const float (&x)[2][32], const float (&b)[2][NR > 0 ? NR : 1],
                                            const int (&bs)[2], float* rb) {
  using S = SolveBlk<NR>;
  constexpr int C0 = (KB + 1) * S::BS;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const bool on = bs[r] >= 0;
    const uint32_t dst = smem_u32(rb) + (uint32_t)(on ? bs[r] : 0) * (S::RS * 4);
#pragma unroll
    for (int j = C0; j < 32; j += 4) st_shared_v4_if(on, dst + 4u * j, x[r][j], x[r][j + 1], x[r][j + 2], x[r][j + 3]);
    if constexpr (NR % 4 == 0 && NR > 0) {
#pragma unroll
      for (int j = 0; j < NR; j += 4) st_shared_v4_if(on, dst + 4u * (32 + j), b[r][j], b[r][j + 1], b[r][j + 2], b[r][j + 3]);
    } else if constexpr (NR > 0) {
      if (on) {
#pragma unroll
        for (int j = 0; j < NR; ++j) rb[bs[r] * S::RS + 32 + j] = b[r][j];
      }
    }
  }
}

// rank-1 term s of block KB's update on the A columns [J0, 32) and the B columns
template <int NR, int J0>
__device__ __forceinline__ void slv_trail(float (&x)[2][32], float (&b)[2][NR > 0 ? NR : 1], const float (&P)[2][4], int s,
                                          const float* rb) {
  using S = SolveBlk<NR>;
  if constexpr (J0 < 32) {
    float Rs[32 - J0];
    ld_row<float, 32 - J0>(Rs, rb + s * S::RS + J0);
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int j = 0; j < 32 - J0; j += 2) ffma2(x[r][J0 + j], x[r][J0 + j + 1], P[r][s], Rs[j], Rs[j + 1]);
  }
  if constexpr (NR > 0) {
    float Rb[NR];
    ld_row<float, NR>(Rb, rb + s * S::RS + 32);
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      if constexpr (NR % 2 == 0) {
#pragma unroll
        for (int j = 0; j < NR; j += 2) ffma2(b[r][j], b[r][j + 1], P[r][s], Rb[j], Rb[j + 1]);
      } else {
#pragma unroll
        for (int j = 0; j < NR; ++j) b[r][j] = fmaf(P[r][s], Rb[j], b[r][j]);
      }
    }
  }
}

// block KB has been factored (panel values P = W - S); apply its update, factoring block
// KB + 1 under it (look-ahead), then recurse
template <int NR, int KB, bool FAST>
__device__ __forceinline__ void slv_blocks(float (&x)[2][32], float (&b)[2][NR > 0 ? NR : 1], float (&P)[2][4],
                                           uint32_t (&kmask)[2], int (&pos)[2], int (&bs)[2], float* rb,
                                           unsigned& tie, unsigned char* rec_g, int li, int g, int lane) {
  constexpr int BS = 4;
  if constexpr (FAST) {
    if (tie) return;   // given up at an exact tie (warp-uniform): the exact pass redoes the task
  }
  slv_publish<NR, KB>(x, b, bs, rb);
  if constexpr (FAST) k0_pos_from_bs<2>(pos, bs, KB * BS);
  __syncwarp();
  if constexpr (KB + 1 < 32 / BS) {
    constexpr int C1 = (KB + 1) * BS;   // the next panel
    float NP[2][4];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int j = 0; j < BS; ++j) NP[r][j] = x[r][C1 + j];
#pragma unroll
    for (int s = 0; s < BS; ++s) {
      float Rs[4];
      ld_row<float, 4>(Rs, rb + s * SolveBlk<NR>::RS + C1);
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        ffma2(NP[r][0], NP[r][1], P[r][s], Rs[0], Rs[1]);
        ffma2(NP[r][2], NP[r][3], P[r][s], Rs[2], Rs[3]);
      }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) bs[r] = -1;
    float pb[BS];
#pragma unroll
    for (int s = 0; s < BS; ++s) {
      blk_panel_step<2, BS, FAST>(s, C1 + s, NP, kmask, pos, bs, tie, pb, rec_g, li, g, lane);
      slv_trail<NR, C1 + BS>(x, b, P, s, rb);
    }
    if constexpr (FAST) rec_store_block(rec_g, C1, pb, li);
    __syncwarp();   // every lane has read rb before the next publish
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int j = 0; j < BS; ++j) P[r][j] = NP[r][j];
    slv_blocks<NR, KB + 1, FAST>(x, b, P, kmask, pos, bs, rb, tie, rec_g, li, g, lane);
  } else {
#pragma unroll
    for (int s = 0; s < BS; ++s) slv_trail<NR, 32>(x, b, P, s, rb);
  }
}

template <int NR, int MODE>
// 3 CTAs per SM (168 registers) up to four right-hand sides; with eight the B registers
// spill there, and 2 CTAs (255 registers, no spill) measure faster (tools/ab_solve.py)
__global__ void __launch_bounds__(kWarpsPerBlock * 32, (NR >= 8 ? 8 : 12) / kWarpsPerBlock)
gj_blk32s_kernel(BlkSolveArgs a, const __grid_constant__ TmaMaps tm, int* __restrict__ tlist) {
  constexpr bool FAST = MODE == 1;   // MODE as in gj_blk32_kernel (K1f's two passes)
  if constexpr (MODE == 2) {
    if (tlist[0] == 0) return;
  }
  using S = SolveBlk<NR>;
  using Geo = BlkGeo<2>;
  constexpr int R = 2, BS = 4, L = Geo::L, MT = Geo::M, NB = NR > 0 ? NR : 1;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  unsigned char* sbase = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* stage0 = sbase + warp * S::NST * Geo::STAGE;
  unsigned char* misc = sbase + kWarpsPerBlock * S::NST * Geo::STAGE + warp * S::BYTES;
  float* rbuf = reinterpret_cast<float*>(misc);
  unsigned char* rec = misc + S::RBUF;
  uint64_t* bars = reinterpret_cast<uint64_t*>(misc + S::RBUF + S::REC);

  const int g = lane / L;
  const int li = lane % L;
  const unsigned gmask = ((1u << L) - 1u) << (L * g);
  float* rb = rbuf + g * BS * S::RS;
  unsigned char* rec_g = rec + g * 32 * 8;

  const int64_t ntasks = MODE == 2 ? (int64_t)tlist[0] : (a.batch + MT - 1) / MT;
  auto task_of = [&](int64_t ti) -> int64_t { return MODE == 2 ? (int64_t)tlist[1 + ti] : ti; };
  const int64_t wstride = (int64_t)gridDim.x * kWarpsPerBlock;
  const int64_t ti0 = (int64_t)blockIdx.x * kWarpsPerBlock + warp;
  const int m = a.m;

  if (lane == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  __syncwarp();
  if (lane == 0 && ti0 < ntasks) {
    mbar_expect_tx(&bars[0], Geo::STAGE);
    tma_load_2d(stage0, &tm.a, 0, (int)(task_of(ti0) * Geo::ROWS), &bars[0]);
  }

  int it = 0;
  for (int64_t ti = ti0; ti < ntasks; ti += wstride, ++it) {
    const int64_t task = task_of(ti);
    const int64_t item0 = task * MT;
    const bool item_ok = item0 + g < a.batch;
    unsigned char* stage = stage0 + (it & 1) * Geo::STAGE;
    const int64_t nti = ti + wstride;
    const int64_t nxt = nti < ntasks ? task_of(nti) : 0;
    if (lane == 0 && nti < ntasks) {
      mbar_expect_tx(&bars[(it + 1) & 1], Geo::STAGE);
      tma_load_2d(stage0 + ((it + 1) & 1) * Geo::STAGE, &tm.a, 0, (int)(nxt * Geo::ROWS), &bars[(it + 1) & 1]);
      if constexpr (NR > 0) {
        const int64_t i0 = nxt * MT, i1 = i0 + MT < a.batch ? i0 + MT : a.batch;
        const uintptr_t lo = ((uintptr_t)(a.B + i0 * 32 * m) + 15) & ~(uintptr_t)15;
        const uintptr_t hi = (uintptr_t)(a.B + i1 * 32 * m) & ~(uintptr_t)15;
        if (hi > lo) bulk_prefetch_l2(reinterpret_cast<const void*>(lo), (uint32_t)(hi - lo));
      }
    }
    // the right-hand sides of this lane's rows (before the wait: the loads overlap it)
    float b[R][NB];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int row = li + L * r;
#pragma unroll
      for (int j = 0; j < NB; ++j)
        b[r][j] = (NR > 0 && item_ok && j < m) ? __ldcs(a.B + ((item0 + g) * 32 + row) * m + j) : 0.0f;
    }
    mbar_wait_warp(&bars[it & 1], (it >> 1) & 1);
    float x[R][32];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int row = li + L * r;
      stage_ld_row<float, 32, true>(x[r], stage, g * 32 + row);
      if (!item_ok) {
#pragma unroll
        for (int j = 0; j < 32; ++j) x[r][j] = (row == j) ? 1.0f : 0.0f;
      }
    }
    __syncwarp();
    float rowmax = 0.0f;
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int j = 0; j < 32; ++j) rowmax = fmaxf(rowmax, fabsf(x[r][j]));
    const double smax = (double)__uint_as_float(blk_gmax<R>(__float_as_uint(rowmax), g));
    const float tau = round_down_to(a.tol * smax, 0.0f);

    uint32_t kmask[R];
    int pos[R], bs[R];
    unsigned tie = 0;
    float pb[BS];
    float P[R][BS];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      kmask[r] = 0x7fffffffu;
      pos[r] = li + L * r;
      bs[r] = -1;
#pragma unroll
      for (int j = 0; j < BS; ++j) P[r][j] = x[r][j];
    }
#pragma unroll
    for (int s = 0; s < BS; ++s) blk_panel_step<R, BS, FAST>(s, s, P, kmask, pos, bs, tie, pb, rec_g, li, g, lane);
    if constexpr (FAST) rec_store_block(rec_g, 0, pb, li);
    slv_blocks<NR, 0, FAST>(x, b, P, kmask, pos, bs, rb, tie, rec_g, li, g, lane);
    __syncwarp();

    // ---- a6: det / ipiv / singular flag from the per-step record (K1b's epilogue)
    float myrp[R];
    unsigned failb = 0;
    int nswap = 0, nneg = 0;
    double lgl = 0.0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int row = li + L * r;
      float p_own, p_k;
      int q_own, q_k = 0;
      if constexpr (FAST) {
        p_own = reinterpret_cast<const float*>(rec_g)[pos[r]];
        p_k = reinterpret_cast<const float*>(rec_g)[row];
      } else {
        rec_load(rec_g, pos[r], p_own, q_own);
        rec_load(rec_g, row, p_k, q_k);
        (void)q_own;
      }
      myrp[r] = rcp(p_own);
      const unsigned fb = __ballot_sync(0xffffffffu, fabsf(p_k) <= tau) & gmask;
      if (failb == 0 && fb != 0) failb = (unsigned)(__ffs(fb) - g * L + r * L);
      if constexpr (!FAST) nswap += __popc(__ballot_sync(0xffffffffu, q_k != row) & gmask);
      nneg += __popc(__ballot_sync(0xffffffffu, p_k < 0.0f) & gmask);
      lgl += log_abs(p_k);
      if constexpr (!FAST) {
        if (a.ipiv && item_ok) a.ipiv[(item0 + g) * 32 + row] = q_k + 1;
      }
    }
    if constexpr (FAST) nswap = 32 - perm_cycles<L>(pos, li, g, gmask);
    const int info = (int)failb;
    const double lg = group_sum<L>(lgl);
    const int sgn = ((nswap ^ nneg) & 1) ? -1 : 1;
    if constexpr (FAST) {
      if (tie && lane == 0) tlist[1 + atomicAdd(tlist, 1)] = (int)task;   // redone by the exact pass
    }
    if (item_ok && li == 0 && !tie) {
      const int64_t item = item0 + g;
      if (a.info) a.info[item] = info;
      if (a.logabsdet) a.logabsdet[item] = info ? -INFINITY : lg;
      if (a.sign) a.sign[item] = info ? 0 : (int8_t)sgn;
      if (a.det) a.det[item] = info ? 0.0f : (float)(sgn * exp(lg));
    }
    // ---- a7 + a8: X[k][:] = (row pivoted at step k)[B part] / p_k
    if constexpr (NR > 0) {
      if (item_ok && !tie) {
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
          for (int j = 0; j < NB; ++j)
            if (j < m) __stcs(a.X + ((item0 + g) * 32 + pos[r]) * m + j, b[r][j] * myrp[r]);
      }
    }
    __syncwarp();   // rec and rb are reused by the next task
  }
}

template <int NR, int MODE>
cudaError_t launch_blk32s_mode(const BlkSolveArgs& a, const TmaMaps& maps, int* tlist, cudaStream_t s) {
  const size_t smem = SolveBlk<NR>::smem();
  auto kern = gj_blk32s_kernel<NR, MODE>;
  static unsigned long long configured = 0;
  const unsigned long long dbit = device_bit();
  if (!(configured & dbit)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured |= dbit;
  }
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kWarpsPerBlock * 32, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const int64_t ntasks = (a.batch + 1) / 2;
  const int64_t need = (ntasks + kWarpsPerBlock - 1) / kWarpsPerBlock;
  const int64_t cap = (int64_t)device_sm_count() * per_sm;
  const int grid = (int)(need < cap ? need : cap);
  kern<<<grid, kWarpsPerBlock * 32, smem, s>>>(a, maps, tlist);
  return cudaGetLastError();
}

// K1s entry: without ipiv the two passes of K1f (FAST pass, then the exact kernel over the
// tasks it gave up), with ipiv the exact kernel (launch_blk32 explains why)
template <int NR>
cudaError_t launch_blk32s(const BlkSolveArgs& a, const TmaMaps& maps, cudaStream_t s) {
  if (GJ_K1F && a.ipiv == nullptr) {
    const int64_t ntasks = (a.batch + 1) / 2;
    int* tl = static_cast<int*>(pool_alloc_async((size_t)(ntasks + 1) * sizeof(int), s));
    if (tl != nullptr) {
      cudaError_t e = cudaMemsetAsync(tl, 0, sizeof(int), s);
      if (e == cudaSuccess) e = launch_blk32s_mode<NR, 1>(a, maps, tl, s);
      if (e == cudaSuccess) e = launch_blk32s_mode<NR, 2>(a, maps, tl, s);
      const cudaError_t f = cudaFreeAsync(tl, s);
      return e != cudaSuccess ? e : f;
    }
  }
  return launch_blk32s_mode<NR, 0>(a, maps, nullptr, s);
}

// K1s applicability: fp32, n = 32, m <= 8, 16-byte aligned A, rows indexable by the TMA map
bool blk32s_map(const void* A, int64_t batch, TmaMaps& maps) {
  if (reinterpret_cast<uintptr_t>(A) % 16 != 0 || batch * 32 >= (int64_t(1) << 31)) return false;
  if (!make_tma_map_2d(&maps.a, false, A, 32, (uint64_t)batch * 32, 128, 32, 64, 128)) return false;
  maps.x = maps.a;
  return true;
}

cudaError_t launch_blk32s_nr(const BlkSolveArgs& a, const TmaMaps& maps, cudaStream_t s) {
  if (a.B == nullptr) return launch_blk32s<0>(a, maps, s);
  if (a.m <= 1) return launch_blk32s<1>(a, maps, s);
  if (a.m <= 2) return launch_blk32s<2>(a, maps, s);
  if (a.m <= 4) return launch_blk32s<4>(a, maps, s);
  return launch_blk32s<8>(a, maps, s);
}

// ------------------------------------------------------------------ host side
template <typename T, int NP, bool TMA>
cudaError_t launch_warp(const BatchedArgs& a, const TmaMaps& maps, cudaStream_t s) {
  using S = Smem<T, NP, TMA>;
  const size_t smem = (size_t)S::per_warp * kWarpsPerBlock + 1024;
  auto kern = gj_batched_warp_kernel<T, NP, TMA>;
  static unsigned long long configured = 0;
  const unsigned long long dbit = device_bit();
  if (!(configured & dbit)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured |= dbit;
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
  if constexpr ((NP * sizeof(T)) % 16 == 0) {
    using TL = TmaLayout<T, NP>;
    const bool full = a.n == NP;
    const bool aligned = (reinterpret_cast<uintptr_t>(a.A) % 16 == 0) &&
                         (a.Ainv == nullptr || reinterpret_cast<uintptr_t>(a.Ainv) % 16 == 0);
    const bool rows_ok = a.batch * NP < (int64_t(1) << 31);
    const bool f64 = sizeof(T) == 8;
    const uint64_t rows = (uint64_t)a.batch * NP;
    const int swz = TL::SPAN >= 32 ? TL::SPAN : 0;
    if constexpr (NP == 32 && sizeof(T) == 4) {
      // determinant-only run: K1s without right-hand sides (no D half)
      if (full && a.Ainv == nullptr) {
        TmaMaps sm;
        if (blk32s_map(a.A, a.batch, sm)) {
          const BlkSolveArgs sa{a.batch, 0, nullptr, nullptr, a.ipiv, a.logabsdet, a.sign,
                                static_cast<float*>(a.det), a.info, a.tol};
          return launch_blk32s_nr(sa, sm, s);
        }
      }
      // K1b (blocked, BS = 4, two rows per lane, two TMA stages): box of 64 rows (2 matrices per warp task)
      if (full && aligned && rows_ok) {
        if (make_tma_map_2d(&maps.a, false, a.A, 32, rows, 128, 32, 64, 128) &&
            (a.Ainv == nullptr || make_tma_map_2d(&maps.x, false, a.Ainv, 32, rows, 128, 32, 64, 128))) {
          if (a.Ainv == nullptr) maps.x = maps.a;
          return launch_blk32<2, 4, GJ_K1B_NST>(a, maps, s);
        }
      }
    }
    if (full && aligned && rows_ok &&
        make_tma_map_2d(&maps.a, f64, a.A, NP, rows, NP * sizeof(T), TL::BOX_COLS, TL::ROWS, swz) &&
        (a.Ainv == nullptr || make_tma_map_2d(&maps.x, f64, a.Ainv, NP, rows, NP * sizeof(T), TL::BOX_COLS, TL::ROWS, swz))) {
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

cudaError_t launch_blk32_solve(const SolveArgs& a, cudaStream_t s) {
  if (a.n != 32 || a.m < 1 || a.m > 8) return cudaErrorNotSupported;
  TmaMaps maps;
  if (!blk32s_map(a.A, a.batch, maps)) return cudaErrorNotSupported;
  const BlkSolveArgs sa{a.batch, a.m, static_cast<const float*>(a.B), static_cast<float*>(a.X), a.ipiv,
                        a.logabsdet, a.sign, nullptr, a.info, a.tol};
  return launch_blk32s_nr(sa, maps, s);
}

cudaError_t launch_batched(gj_dtype dt, const BatchedArgs& a, cudaStream_t s) {
  if (a.batch == 0) return cudaSuccess;
  if (a.n <= 32) return dt == GJ_F32 ? dispatch_np<float>(a, s) : dispatch_np<double>(a, s);
  return cudaErrorInvalidValue;
}

}  // namespace gj
