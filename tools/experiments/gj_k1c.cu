// K1c — the C2 hot path (BASELINE configs[1]): batched Gauss–Jordan inversion, fp32, n = 32.
//
// Four matrices per warp task, eight lanes per matrix, FOUR rows per lane (slot r of lane li
// in group g holds row li + 8 r of matrix g), the matrix in registers for the whole
// elimination.  The method is K1b's (gj_batched.cu; §2, Eqs. (14)-(15), L61-L72;
// Obs. 2-3, L59-L60; listing L150-L198): partial pivoting on max |x_ik| over the rows not yet
// pivoted with ties to the smallest physical position of the listing's swapped array
// (reading G3), logical swaps, deferred normalisation (multiplier x_ik / p, each row scaled by
// its own pivot's reciprocal at the store), compact storage, and the elimination taken in
// blocks of BS = 4 steps: inside a block each step updates only the block's 4 panel columns,
// at the block's end every row applies   x_i[J'] += sum_s (W - S)_is R_s[J']   (the
// aggregation of Eqs. (14)-(15); DESIGN.md §7 derives it), with a one-block look-ahead.
//
// Why four matrices per warp (measured in profiles/r02_k1c_summary.md): the
// shared-memory pipe, not HBM, bounded K1b — every element of a block's pivot rows is
// broadcast to every row, and one broadcast feeds all the rows a lane holds of that matrix, so
// four rows per lane halve the broadcast traffic per matrix; the per-matrix parts of the pivot
// chain (reductions, reciprocal, the pivot row's panel values) are shared by four matrices.
// Measured costs behind the choices (tools/ubench/smem_tp.cu, tools/ubench/lat.cu): a
// broadcast LDS.128 costs 2.4 SM cycles but an LDS.64 at most 0.75, so the trailing update
// reads the pivot rows two values at a time; a predicated STS.128 costs one cycle per active
// quarter-warp, and a group is a quarter-warp here; redux.sync answers in ~18 cycles where a
// shuffle butterfly over 8 lanes takes ~90.
//
// Per pivot step (k = global step, s = k mod 4 = the panel column):
//   a2  key = |x_ik| bit pattern (monotone for non-negative floats), 0 for pivoted rows; the
//       group maximum m by one redux.sync per group; every row with key == m is a candidate.
//       One ballot per slot: if every group has exactly one candidate (the usual case) it is
//       the pivot; otherwise (ties) the candidate at the smallest physical position wins (a
//       second group reduction on (position, lane, slot)).  A numerically singular column
//       (m = 0) lets pivoted rows tie too: the singular flag is taken from m itself, so
//       whichever row wins, info is right, and the rest of that item is unspecified (G11).
//   a3  logical swap: each row keeps the position it would have in the listing's swapped
//       array; only the row at position k moves (to q).  The group's first lane records
//       (p, q) per step in shared memory: ipiv, the swap parity, log|det| and the singular
//       flag come from that record after the loop.
//   a4  the pivot row publishes its three other panel values and (q | sign p) in one 16-byte
//       store; |p| = m is already known to every lane, so 1/|p| starts before the winner is.
//   a5  Eq. (15) on the panel: x_ij += f_i z_j with f_i = -x_ik / p (FFMA2 for column pairs).
// I/O: the task's 128 rows arrive by TMA (128-byte swizzle) in a 16 KB stage that also holds
// the block buffers during the elimination (the matrix is in registers then) and the
// un-permuted output for the TMA store; the next task is prefetched into L2 meanwhile.
#include <cuda.h>
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

constexpr int kR = 4;            // rows per lane
constexpr int kL = 8;            // lanes per matrix
constexpr int kM = 4;            // matrices per warp task
constexpr int kBS = 4;           // block size (pivot steps per block)
constexpr int kRW = 32 - kBS;    // columns outside the panel
constexpr int kRows = 32 * kM;   // rows per warp task
constexpr int kWarps = 2;        // warps per CTA
#ifndef GJ_K1C_MINB
#define GJ_K1C_MINB 4            // resident CTAs per SM the registers are sized for (2 warps per scheduler)
#endif

// Per-warp shared memory.  The stage (TMA in / out) doubles as the elimination's scratch.
struct CS {
  static constexpr int STAGE = kRows * 128;                  // 16 KB
  // inside the stage, while the matrix is in registers:
  static constexpr int RBUF = 0;                             // [4 g][4 s][28] f32: block pivot rows
  static constexpr int ZBUF = RBUF + kM * kBS * kRW * 4;     // [2 parity][4 g] x 16 B: pivot row panel
  static constexpr int REC = ZBUF + 2 * kM * 16;             // [4 g][32] (p bits, q)
  static_assert(REC + kM * 32 * 8 <= STAGE, "scratch fits the stage");
  // outside the stage:
  static constexpr int PERM = STAGE;                         // [4 g][32] int: output column (bytes)
  static constexpr int BAR = PERM + kM * 32 * 4;
  static constexpr int PER_WARP = (BAR + 16 + 1023) / 1024 * 1024;
  static constexpr int SMEM = kWarps * PER_WARP + 1024;
};

__device__ __forceinline__ void st_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ void st_v4_if(bool p, uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %0, 0;\n\t@q st.shared.v4.b32 [%1], {%2, %3, %4, %5};\n}" ::"r"(
                   p ? 1u : 0u),
               "r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}
// Warp barrier with memory ordering among the warp's lanes (bar.warp.sync; in converged code
// ptxas emits no divergence check, so it does not split the basic block the way __syncwarp's
// BRA.DIV does — the panel chain and the interleaved trailing update stay schedulable together).
__device__ __forceinline__ void wsync() { asm volatile("bar.warp.sync 0xffffffff;" ::: "memory"); }
__device__ __forceinline__ uint4 ld_v4(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ float2 ld_f2(uint32_t addr) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr) : "memory");
  return v;
}

// Maximum / minimum over the 8 lanes of each group: one full-warp redux.sync per group (the
// other groups contribute the identity) — ~18 cycles each, where a shuffle butterfly takes ~90.
__device__ __forceinline__ uint32_t gmax8(uint32_t v, int g) {
  const uint32_t a0 = __reduce_max_sync(0xffffffffu, g == 0 ? v : 0u);
  const uint32_t a1 = __reduce_max_sync(0xffffffffu, g == 1 ? v : 0u);
  const uint32_t a2 = __reduce_max_sync(0xffffffffu, g == 2 ? v : 0u);
  const uint32_t a3 = __reduce_max_sync(0xffffffffu, g == 3 ? v : 0u);
  return g < 2 ? (g == 0 ? a0 : a1) : (g == 2 ? a2 : a3);
}
__device__ __forceinline__ uint32_t gmin8(uint32_t v, int g) {
  const uint32_t a0 = __reduce_min_sync(0xffffffffu, g == 0 ? v : 0xffffffffu);
  const uint32_t a1 = __reduce_min_sync(0xffffffffu, g == 1 ? v : 0xffffffffu);
  const uint32_t a2 = __reduce_min_sync(0xffffffffu, g == 2 ? v : 0xffffffffu);
  const uint32_t a3 = __reduce_min_sync(0xffffffffu, g == 3 ? v : 0xffffffffu);
  return g < 2 ? (g == 0 ? a0 : a1) : (g == 2 ? a2 : a3);
}

// The panel column order a pivot row publishes: A = the column outside the step's pair,
// (C, D) = the other pair (an aligned register pair for FFMA2).
template <int S> struct PanelOrder {
  static constexpr int A = S == 0 ? 1 : S == 1 ? 0 : S == 2 ? 3 : 2;
  static constexpr int C = S < 2 ? 2 : 0;
};

struct NoWork {
  __device__ __forceinline__ void operator()(int) const {}
};

// Pivot step S (static) of the block at global step k on the panel registers P.  work(0..2)
// is a third of the independent trailing update each, placed in the three stretches between
// the step's branch and barrier so that it fills the chain's latency.
template <int S, class W>
__device__ __forceinline__ void c_panel_step(const int k, float (&P)[kR][kBS], uint32_t (&km)[kR], int (&pos)[kR],
                                             int (&pst)[kR], uint32_t zb, uint32_t recg, int li, int g, int lane,
                                             const W& work) {
  using O = PanelOrder<S>;
  // a2: candidates = rows whose |x_ik| equals the group maximum
  uint32_t key[kR];
#pragma unroll
  for (int r = 0; r < kR; ++r) key[r] = __float_as_uint(P[r][S]) & km[r];
  const uint32_t m = gmax8(max(max(key[0], key[1]), max(key[2], key[3])), g);
  bool pv[kR];
  int cnt = 0;
#pragma unroll
  for (int r = 0; r < kR; ++r) {
    pv[r] = key[r] == m;
    cnt += __popc(__ballot_sync(0xffffffffu, pv[r]));
  }
  work(0);
  if (__builtin_expect(cnt != kM, 0)) {
    // ties (or a singular column): the candidate at the smallest physical position (G3);
    // the code carries (position, lane, slot), so the winner is unique
    uint32_t c = 0xffffffffu;
#pragma unroll
    for (int r = 0; r < kR; ++r)
      c = min(c, pv[r] ? ((uint32_t)pos[r] << 7 | (uint32_t)lane << 2 | (uint32_t)r) : 0xffffffffu);
    const uint32_t win = gmin8(c, g);
#pragma unroll
    for (int r = 0; r < kR; ++r)
      pv[r] = ((uint32_t)pos[r] << 7 | (uint32_t)lane << 2 | (uint32_t)r) == win;
  }
  // a4: the pivot row publishes (z_A, q | sign p, z_C, z_C+1); one winner per group
#pragma unroll
  for (int r = 0; r < kR; ++r)
    st_v4_if(pv[r], zb, __float_as_uint(P[r][O::A]), (uint32_t)pos[r] | (__float_as_uint(P[r][S]) & 0x80000000u),
             __float_as_uint(P[r][O::C]), __float_as_uint(P[r][O::C + 1]));
  const float ra = rcp(__uint_as_float(m));   // 1/|p| (|p| = m exactly), under the exchange
  work(1);
  wsync();
  const uint4 z = ld_v4(zb);
  const uint32_t q = z.y & 31u;
  if (li == 0)
    asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(recg + 8u * (uint32_t)k), "r"(m | (z.y & 0x80000000u)), "r"(q)
                 : "memory");
  // -1/p = -(1/|p|) sign p: the sign folded into the reciprocal once per step
  const float nrp = __uint_as_float(__float_as_uint(ra) ^ (~z.y & 0x80000000u));
  const float zA = __uint_as_float(z.x), zC = __uint_as_float(z.z), zD = __uint_as_float(z.w);
#pragma unroll
  for (int r = 0; r < kR; ++r) {
    // a5: f = -x_ik / p; 0 on the pivot row (W - S convention)
    const float nf = pv[r] ? 0.0f : P[r][S] * nrp;
    P[r][O::A] = fmaf(nf, zA, P[r][O::A]);
    ffma2(P[r][O::C], P[r][O::C + 1], nf, zC, zD);
    P[r][S] = nf;
    // a3: the listing's swap of positions k and q (L156-L162); pivoted rows keep km = 0
    pos[r] = (uint32_t)pos[r] == (uint32_t)k ? (int)q : pos[r];
    pst[r] = pv[r] ? k : pst[r];
    km[r] = pv[r] ? 0u : km[r];
  }
  work(2);
}

template <int S>
__device__ __forceinline__ void c_panel_steps(const int kb, float (&P)[kR][kBS], uint32_t (&km)[kR], int (&pos)[kR],
                                              int (&pst)[kR], uint32_t zbuf, uint32_t recg, int li, int g, int lane) {
  if constexpr (S < kBS) {
    c_panel_step<S>(kb + S, P, km, pos, pst, zbuf + (S & 1) * (kM * 16), recg, li, g, lane, NoWork{});
    c_panel_steps<S + 1>(kb, P, km, pos, pst, zbuf, recg, li, g, lane);
  }
}

// Publish the block's pivot rows (values at the block's start): row with pst in
// [kb, kb + 4) -> rbuf[g][pst - kb][0..28).
__device__ __forceinline__ void c_publish(const float (&T)[kR][kRW], const int (&pst)[kR], int kb, uint32_t rbg) {
#pragma unroll
  for (int r = 0; r < kR; ++r) {
    const uint32_t bs = (uint32_t)(pst[r] - kb);
    const bool on = bs < (uint32_t)kBS;
    const uint32_t dst = rbg + (on ? bs : 0u) * (kRW * 4);
#pragma unroll
    for (int j = 0; j < kRW; j += 4)
      st_v4_if(on, dst + 4u * j, __float_as_uint(T[r][j]), __float_as_uint(T[r][j + 1]), __float_as_uint(T[r][j + 2]),
               __float_as_uint(T[r][j + 3]));
  }
}

// Rank-1 term s of the block update on T columns [J0, J1): T += (W - S)[:, s] R_s, the pivot
// row read two values at a time.  SHIFT: the result lands BS registers to the left.
template <int J0, int J1, int N, bool SHIFT = false>
__device__ __forceinline__ void c_trail(float (&T)[kR][N], const float (&P)[kR][kBS], int s, uint32_t rbg) {
#pragma unroll
  for (int j = J0; j < J1; j += 2) {
    const float2 rv = ld_f2(rbg + (uint32_t)(s * kRW + j) * 4u);
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      if constexpr (SHIFT) {
        float u0 = T[r][j], u1 = T[r][j + 1];
        ffma2(u0, u1, P[r][s], rv.x, rv.y);
        T[r][j - kBS] = u0;
        T[r][j + 1 - kBS] = u1;
      } else {
        ffma2(T[r][j], T[r][j + 1], P[r][s], rv.x, rv.y);
      }
    }
  }
}
// Third `part` of term s on the columns outside the panel (pairs 4..27), for the interleave.
template <bool SHIFT>
struct TrailWork {
  float (&T)[kR][kRW];
  const float (&P)[kR][kBS];
  int s;
  uint32_t rbg;
  __device__ __forceinline__ void operator()(int part) const {
    if (part == 0) c_trail<kBS, kBS + 8, kRW, SHIFT>(T, P, s, rbg);
    else if (part == 1) c_trail<kBS + 8, kBS + 16, kRW, SHIFT>(T, P, s, rbg);
    else c_trail<kBS + 16, kRW, kRW, SHIFT>(T, P, s, rbg);
  }
};
// The same on the 4 look-ahead columns (the next panel), which sit at NP[.][0..4) and read
// R_s[0..4).
__device__ __forceinline__ void c_trail_np(float (&NP)[kR][kBS], const float (&P)[kR][kBS], int s, uint32_t rbg) {
#pragma unroll
  for (int j = 0; j < kBS; j += 2) {
    const float2 rv = ld_f2(rbg + (uint32_t)(s * kRW + j) * 4u);
#pragma unroll
    for (int r = 0; r < kR; ++r) ffma2(NP[r][j], NP[r][j + 1], P[r][s], rv.x, rv.y);
  }
}

__device__ __forceinline__ uint32_t swz128(uint32_t row, uint32_t cb) {   // byte offset of (row, column byte cb)
  return row * 128u + ((((cb >> 4) ^ (row & 7u)) << 4) | (cb & 15u));
}

__global__ void __launch_bounds__(kWarps * 32, GJ_K1C_MINB) gj_k1c_kernel(BatchedArgs a,
                                                                          const __grid_constant__ CUtensorMap tma_a,
                                                                          const __grid_constant__ CUtensorMap tma_x) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  unsigned char* sbase = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* stage = sbase + warp * CS::PER_WARP;
  const uint32_t st0 = smem_u32(stage);
  int* perm = reinterpret_cast<int*>(stage + CS::PERM);
  uint64_t* bar = reinterpret_cast<uint64_t*>(stage + CS::BAR);

  const int g = lane >> 3;
  const int li = lane & 7;
  const uint32_t rbg = st0 + CS::RBUF + (uint32_t)g * (kBS * kRW * 4);
  const uint32_t zbuf = st0 + CS::ZBUF + (uint32_t)g * 16;
  const uint32_t recg = st0 + CS::REC + (uint32_t)g * (32 * 8);
  int* perm_g = perm + g * 32;

  const int64_t ntasks = (a.batch + kM - 1) / kM;
  const int64_t wstride = (int64_t)gridDim.x * kWarps;
  const int64_t task0 = (int64_t)blockIdx.x * kWarps + warp;

  if (lane == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncwarp();
  if (lane == 0 && task0 < ntasks) {
    mbar_expect_tx(bar, CS::STAGE);
    tma_load_2d(stage, &tma_a, 0, (int)(task0 * kRows), bar);
  }

  int it = 0;
  for (int64_t task = task0; task < ntasks; task += wstride, ++it) {
    const int64_t item = task * kM + g;
    const bool item_ok = item < a.batch;
    const int64_t nxt = task + wstride;
    if (lane == 0 && nxt < ntasks) bulk_prefetch_l2(static_cast<const float*>(a.A) + nxt * kRows * 32, CS::STAGE);
    mbar_wait_warp(bar, it & 1);

    // ---- a1: rows li + 8 r of matrix g into registers; s = max |a_ij|
    float x[kR][32];
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      const uint32_t row = (uint32_t)(g * 32 + li + 8 * r);
#pragma unroll
      for (int j = 0; j < 32; j += 4) {
        const uint4 u = ld_v4(st0 + swz128(row, 4u * j));
        x[r][j] = __uint_as_float(u.x);
        x[r][j + 1] = __uint_as_float(u.y);
        x[r][j + 2] = __uint_as_float(u.z);
        x[r][j + 3] = __uint_as_float(u.w);
      }
      if (!item_ok) {   // padding matrices: the identity
#pragma unroll
        for (int j = 0; j < 32; ++j) x[r][j] = (li + 8 * r == j) ? 1.0f : 0.0f;
      }
    }
    __syncwarp();   // the stage is scratch from here on
    uint32_t amax = 0;
#pragma unroll
    for (int r = 0; r < kR; ++r)
#pragma unroll
      for (int j = 0; j < 32; ++j) amax = max(amax, __float_as_uint(x[r][j]) & 0x7fffffffu);

    uint32_t km[kR];
    int pos[kR], pst[kR];
    float P[kR][kBS], T[kR][kRW];
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      km[r] = 0x7fffffffu;
      pos[r] = li + 8 * r;
      pst[r] = 64;
#pragma unroll
      for (int j = 0; j < kBS; ++j) P[r][j] = x[r][j];
#pragma unroll
      for (int j = 0; j < kRW; ++j) T[r][j] = x[r][kBS + j];
    }
    c_panel_steps<0>(0, P, km, pos, pst, zbuf, recg, li, g, lane);
    // look-ahead: publish block kb's pivot rows, bring the next panel up to date first, then
    // factor it while the rest of block kb's update runs
#pragma unroll 1
    for (int kb = 0; kb + kBS < 32; kb += kBS) {
      c_publish(T, pst, kb, rbg);
      wsync();
      float NP[kR][kBS];
#pragma unroll
      for (int r = 0; r < kR; ++r)
#pragma unroll
        for (int j = 0; j < kBS; ++j) NP[r][j] = T[r][j];
#pragma unroll
      for (int s = 0; s < kBS; ++s) c_trail_np(NP, P, s, rbg);
      // the next block's panel steps interleaved with this block's remaining update
      c_panel_step<0>(kb + kBS + 0, NP, km, pos, pst, zbuf, recg, li, g, lane, TrailWork<false>{T, P, 0, rbg});
      c_panel_step<1>(kb + kBS + 1, NP, km, pos, pst, zbuf + kM * 16, recg, li, g, lane, TrailWork<false>{T, P, 1, rbg});
      c_panel_step<2>(kb + kBS + 2, NP, km, pos, pst, zbuf, recg, li, g, lane, TrailWork<false>{T, P, 2, rbg});
      // + the rotation by BS columns in the last term
      c_panel_step<3>(kb + kBS + 3, NP, km, pos, pst, zbuf + kM * 16, recg, li, g, lane, TrailWork<true>{T, P, 3, rbg});
      wsync();   // every lane has read rbuf before the next publish
#pragma unroll
      for (int r = 0; r < kR; ++r)
#pragma unroll
        for (int j = 0; j < kBS; ++j) {
          T[r][kRW - kBS + j] = P[r][j];
          P[r][j] = NP[r][j];
        }
    }
    // last block: its whole update; then x = [T | P] (register j = compact column j)
    c_publish(T, pst, 32 - kBS, rbg);
    wsync();
#pragma unroll
    for (int s = 0; s < kBS; ++s) c_trail<0, kRW, kRW>(T, P, s, rbg);
#pragma unroll
    for (int r = 0; r < kR; ++r) {
#pragma unroll
      for (int j = 0; j < kRW; ++j) x[r][j] = T[r][j];
#pragma unroll
      for (int j = 0; j < kBS; ++j) x[r][kRW + j] = P[r][j];
    }

    // ---- a6: det / ipiv / singular flag from the record (this lane: steps li + 8 r)
    const float tau = round_down_to(a.tol * (double)__uint_as_float(gmax8(amax, g)), 0.0f);
    float myrp[kR];
    int info = 0, nsw = 0, nng = 0, esum = 0;
    float msum = 0.0f;
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      const int k = li + 8 * r;
      uint2 rk;
      uint32_t pown;
      asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(rk.x), "=r"(rk.y) : "r"(recg + 8u * (uint32_t)k) : "memory");
      asm volatile("ld.shared.b32 %0, [%1];" : "=r"(pown) : "r"(recg + 8u * (uint32_t)pst[r]) : "memory");
      const float pk = __uint_as_float(rk.x);
      myrp[r] = rcp(__uint_as_float(pown));
      const unsigned fb = (__ballot_sync(0xffffffffu, fabsf(pk) <= tau) >> (8 * g)) & 0xffu;
      if (info == 0 && fb != 0) info = 8 * r + __ffs(fb);
      nsw += __popc(__ballot_sync(0xffffffffu, (int)rk.y != k) & (0xffu << (8 * g)));
      nng += __popc(__ballot_sync(0xffffffffu, pk < 0.0f) & (0xffu << (8 * g)));
      // log2|p| = e + log2(mantissa): exponents summed exactly, mantissa logs in fp32
      const uint32_t b = rk.x & 0x7fffffffu;
      esum += (int)(b >> 23) - 127;
      msum += __log2f(__uint_as_float((b & 0x7fffffu) | 0x3f800000u));
      if (a.ipiv && item_ok) a.ipiv[item * 32 + k] = (int)rk.y + 1;
    }
#pragma unroll
    for (int o = 1; o < kL; o <<= 1) {
      esum += __shfl_xor_sync(0xffffffffu, esum, o);
      msum += __shfl_xor_sync(0xffffffffu, msum, o);
    }
    if (item_ok && li == 0) {
      const double lg = ((double)esum + (double)msum) * 0.6931471805599453;
      const int sgn = ((nsw ^ nng) & 1) ? -1 : 1;
      if (a.info) a.info[item] = info;
      if (a.logabsdet) a.logabsdet[item] = info ? -INFINITY : lg;
      if (a.sign) a.sign[item] = info ? 0 : (int8_t)sgn;
      if (a.det) static_cast<float*>(a.det)[item] = info ? 0.0f : (float)(sgn * exp(lg));
    }

    // ---- a7 + a8: Ainv[pst(i)][perm[k']] = X[i][k'] / p_i through the stage (L179-L198)
    if (a.Ainv != nullptr) {
#pragma unroll
      for (int r = 0; r < kR; ++r) perm_g[pst[r]] = (li + 8 * r) * 4;   // compact column pst -> output column
      __syncwarp();
      uint32_t rb[kR], rx[kR];
#pragma unroll
      for (int r = 0; r < kR; ++r) {
        const uint32_t row = (uint32_t)(g * 32 + pst[r]);
        rb[r] = st0 + row * 128u;
        rx[r] = (row & 7u) << 4;
      }
#pragma unroll
      for (int kp = 0; kp < 32; kp += 4) {
        const int4 cb = *reinterpret_cast<const int4*>(perm_g + kp);
        const uint32_t cbs[4] = {(uint32_t)cb.x, (uint32_t)cb.y, (uint32_t)cb.z, (uint32_t)cb.w};
#pragma unroll
        for (int r = 0; r < kR; ++r)
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const uint32_t ad = rb[r] + (cbs[u] ^ rx[r]);
            asm volatile("st.shared.f32 [%0], %1;" ::"r"(ad), "f"(myrp[r] * x[r][kp + u]) : "memory");
          }
      }
      // the row's own compact entry was held as W - 1 (W - S convention): add the 1 back
#pragma unroll
      for (int r = 0; r < kR; ++r) {
        const uint32_t ad = rb[r] + ((uint32_t)((li + 8 * r) * 4) ^ rx[r]);
        float v;
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(ad) : "memory");
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(ad), "f"(v + myrp[r]) : "memory");
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_2d(&tma_x, 0, (int)(task * kRows), stage);
        bulk_commit();
      }
    }
    __syncwarp();
    if (lane == 0 && nxt < ntasks) {
      bulk_wait_read0();   // the store has read the stage
      mbar_expect_tx(bar, CS::STAGE);
      tma_load_2d(stage, &tma_a, 0, (int)(nxt * kRows), bar);
    }
  }
  if (lane == 0) bulk_wait0();
}

}  // namespace

// K1c launcher: fp32, n = 32, 16-byte aligned A / Ainv, batch * 32 rows addressable by TMA.
// cudaErrorNotSupported when those do not hold (the caller falls back to K1b / K1).
cudaError_t launch_k1c(const BatchedArgs& a, cudaStream_t s) {
  if (a.n != 32) return cudaErrorNotSupported;
  if ((reinterpret_cast<uintptr_t>(a.A) & 15) || (a.Ainv && (reinterpret_cast<uintptr_t>(a.Ainv) & 15)))
    return cudaErrorNotSupported;
  const uint64_t rows = (uint64_t)a.batch * 32;
  if (rows >= (uint64_t(1) << 31)) return cudaErrorNotSupported;
  CUtensorMap ma, mx;
  if (!make_tma_map_2d(&ma, false, a.A, 32, rows, 128, 32, kRows, 128)) return cudaErrorNotSupported;
  if (a.Ainv != nullptr) {
    if (!make_tma_map_2d(&mx, false, a.Ainv, 32, rows, 128, 32, kRows, 128)) return cudaErrorNotSupported;
  } else {
    mx = ma;
  }
  static unsigned long long configured = 0;
  const unsigned long long dbit = device_bit();
  if (!(configured & dbit)) {
    cudaError_t e = cudaFuncSetAttribute(gj_k1c_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, CS::SMEM);
    if (e != cudaSuccess) return e;
    configured |= dbit;
  }
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gj_k1c_kernel, kWarps * 32, CS::SMEM);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const int64_t ntasks = (a.batch + kM - 1) / kM;
  const int64_t need = (ntasks + kWarps - 1) / kWarps;
  const int64_t cap = (int64_t)device_sm_count() * per_sm;
  const int grid = (int)(need < cap ? need : cap);
  gj_k1c_kernel<<<grid, kWarps * 32, CS::SMEM, s>>>(a, ma, mx);
  return cudaGetLastError();
}

}  // namespace gj
