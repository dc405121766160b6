// EXPERIMENT (not built into the library): K2g, a register-resident trailing matrix for
// fp64 n = 64 (four trailing warps + the K2f panel warp), measured slower than K2f on C3 —
// profiles/r02_k2f_summary.md.  Kept for the record; the product kernel is K2f in
// paper_1401_7962_b200/csrc/gj_batched64e.cu (this file is a full copy with K2g added).
// K2e — the C3 hot path (BASELINE configs[2]): batched Gauss–Jordan for fp64 n = 64, one
// warp per matrix, the matrix resident in SHARED MEMORY, the blocked trailing update on the
// FP64 tensor pipe (DMMA, mma.sync m8n8k4 f64).
//
// The elimination (§2, Eqs. (14)-(15), L61-L72; Obs. 2-3 L59-L60; listing
// L150-L177) runs in blocks of BS = 8 pivot steps, the aggregation K1b uses:
//   1. the warp loads the block's 8 panel columns (rows lane, lane + 32) into registers and
//      factors them: max |x_ik| over the un-pivoted rows (fp64 keys: high word, then low
//      word), ties to the smallest physical position (reading G3), logical swaps, deferred
//      normalisation, the pivot row's own compact entry held as W - S = 0; the pivot row's
//      panel values travel through a small shared buffer (one writer, broadcast reads,
//      buffered by step parity) and 1/|p| starts from the winning key before the winner is
//      known; W - S goes back to shared memory with the block's record;
//   2. X[:, ~panel] += (W - S) R tile by tile: per 8-column tile the two B fragments are
//      read from the block's pivot rows (before the tile is written, so no copy of R), then
//      the eight m-tiles' C fragments go LDS.128 -> 2 DMMA -> STS.128.
// Layout: row stride 64 doubles with the 16-byte chunk index XOR f(row), f = ((row & 1) << 2)
// | ((row >> 1) & 3) — the panel's column access (8 rows per LDS.128 phase) and the
// accumulator-fragment access (rows 2p, 2p + 1 x 4 lanes per phase) both hit 8 distinct
// chunks.  A matrix costs ~34 KB of shared memory and 32 threads, so six run per SM.
// The un-permutation (L179-L198) and the deferred pivot-row scale happen in the store, and
// the next matrix's rows are loaded under this one's store.
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

constexpr int N64 = 64;
constexpr int BSD = 8;             // block size = one 8-column tile
#ifndef GJ_K2E_PSTORE
#define GJ_K2E_PSTORE 1            // K2e pivot-row publish as predicated stores, no selects (12.04 -> 11.23 ms)
#endif
#ifndef GJ_K2E_PHASED
#define GJ_K2E_PHASED 0            // loads / DMMA k0 / DMMA k1 / stores in phases: measured equal, off
#endif


__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ double shfl_dd(double v, int src) {
  const long long b = __double_as_longlong(v);
  const int lo = __shfl_sync(0xffffffffu, (int)(b & 0xffffffffll), src);
  const int hi = __shfl_sync(0xffffffffu, (int)(b >> 32), src);
  return __longlong_as_double(((long long)hi << 32) | (unsigned int)lo);
}
__device__ __forceinline__ double rcp64d(double p) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(p));
  double e = fma(-p, r, 1.0);
  r = fma(r, e, r);
  e = fma(-p, r, 1.0);
  return fma(r, e, r);
}


// Warp 0's pivot step S (static) at global step k on the panel rows lane and lane + 32.
// SROW (K2e): |p| is the winning key itself, so 1/|p| starts before the winner is known,
// and the pivot row travels through shared memory (one writer, broadcast reads, buffered by
// step parity) instead of sixteen shuffles.
template <int S, bool SROW = false>
__device__ __forceinline__ void d_panel_step(const int k, double (&x)[2][BSD], uint32_t (&kmask)[2], int (&pos)[2],
                                             int (&bs)[2], unsigned char* rec, int* rowk, int lane,
                                             double* prow = nullptr) {
  uint32_t hi[2], lo[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(x[r][S]);
    hi[r] = (uint32_t)(b >> 32) & 0x7fffffffu & kmask[r];
    lo[r] = (uint32_t)b & kmask[r];
  }
  const uint32_t mh = __reduce_max_sync(0xffffffffu, max(hi[0], hi[1]));
  uint32_t lm = 0;
#pragma unroll
  for (int r = 0; r < 2; ++r)
    if (hi[r] == mh) lm = max(lm, lo[r]);
  const uint32_t ml = __reduce_max_sync(0xffffffffu, lm);
  double rap = 0.0;
  if constexpr (SROW) rap = rcp64d(__longlong_as_double((long long)(((unsigned long long)mh << 32) | ml)));
  uint32_t c = 0xffffffu;
#pragma unroll
  for (int r = 0; r < 2; ++r)
    if (hi[r] == mh && lo[r] == ml && kmask[r] != 0u) c = min(c, (uint32_t)pos[r] << 6 | (uint32_t)lane << 1 | (uint32_t)r);
  const uint32_t win = __reduce_min_sync(0xffffffffu, c);
  const int q = (int)(win >> 6);
  const int src = (int)((win >> 1) & 31u);
  const int slot = (int)(win & 1u);
  double z[BSD];
  if constexpr (SROW) {
    double* pr = prow + (S & 1) * BSD;
#if GJ_K2E_PSTORE
    // two predicated store sets instead of selects: only the winner's slot stores
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      if (lane == src && slot == r) {
#pragma unroll
        for (int j = 0; j < BSD; j += 2) *reinterpret_cast<double2*>(pr + j) = make_double2(x[r][j], x[r][j + 1]);
      }
    }
#else
    if (lane == src) {
#pragma unroll
      for (int j = 0; j < BSD; j += 2)
        *reinterpret_cast<double2*>(pr + j) = slot ? make_double2(x[1][j], x[1][j + 1]) : make_double2(x[0][j], x[0][j + 1]);
    }
#endif
    __syncwarp();
#pragma unroll
    for (int j = 0; j < BSD; j += 2) {
      const double2 v = *reinterpret_cast<const double2*>(pr + j);
      z[j] = v.x;
      z[j + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < BSD; ++j) z[j] = shfl_dd(slot ? x[1][j] : x[0][j], src);
  }
  const double p = z[S];
  double rp;
  if constexpr (SROW) {
    rp = p < 0.0 ? -rap : rap;   // rcp64d is odd: bit-identical to rcp64d(p)
  } else {
    rp = rcp64d(p);
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const bool pv = pos[r] == q && kmask[r] != 0u;
    const double nf = pv ? 0.0 : -(x[r][S] * rp);
#pragma unroll
    for (int j = 0; j < BSD; ++j)
      if (j != S) x[r][j] = fma(nf, z[j], x[r][j]);
    x[r][S] = nf;   // compact D entry; 0 on the pivot row (W - S)
    kmask[r] = pv ? 0u : kmask[r];
    bs[r] = pv ? S : bs[r];
    pos[r] = (pos[r] == k) ? q : pos[r];   // a3: the listing's swap of positions k and q (L156-L162)
    pos[r] = pv ? k : pos[r];
  }
  if (lane == 0) {
    rec_store(rec, k, p, q);
    rowk[k] = src + 32 * slot;
  }
}
// Warp barrier with memory ordering among the lanes that ptxas does not turn into a
// divergence check + branch (as __syncwarp does): the panel step stays one basic block, so
// the interleaved trailing update (work) can be scheduled into its latency.
__device__ __forceinline__ void wsync() { asm volatile("bar.warp.sync 0xffffffff;" ::: "memory"); }
__device__ __forceinline__ void st2_if(bool p, double* addr, double a, double b) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %0, 0;\n\t@q st.shared.v2.f64 [%1], {%2, %3};\n}" ::"r"(p ? 1u : 0u),
               "r"((uint32_t)__cvta_generic_to_shared(addr)), "d"(a), "d"(b)
               : "memory");
}

struct NoWork {
  __device__ __forceinline__ void operator()(int) const {}
};

// K2e's pivot step S with a work hook: work(S) runs between the key reductions and the pivot
// row exchange (independent instructions for the scheduler to interleave with the chain).
template <int S, class Wk>
__device__ __forceinline__ void e_panel_step(const int k, double (&x)[2][BSD], uint32_t (&kmask)[2], int (&pos)[2],
                                             unsigned char* rec, int* rowk, int lane, double* prow, const Wk& work) {
  uint32_t hi[2], lo[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(x[r][S]);
    hi[r] = (uint32_t)(b >> 32) & 0x7fffffffu & kmask[r];
    lo[r] = (uint32_t)b & kmask[r];
  }
  const uint32_t mh = __reduce_max_sync(0xffffffffu, max(hi[0], hi[1]));
  const uint32_t lm = max(hi[0] == mh ? lo[0] : 0u, hi[1] == mh ? lo[1] : 0u);
  const uint32_t ml = __reduce_max_sync(0xffffffffu, lm);
  const double rap = rcp64d(__longlong_as_double((long long)(((unsigned long long)mh << 32) | ml)));
  uint32_t c = 0xffffffu;
#pragma unroll
  for (int r = 0; r < 2; ++r)
    c = min(c, (hi[r] == mh && lo[r] == ml && kmask[r] != 0u) ? ((uint32_t)pos[r] << 6 | (uint32_t)lane << 1 | (uint32_t)r)
                                                               : 0xffffffu);
  const uint32_t win = __reduce_min_sync(0xffffffffu, c);
  const int q = (int)(win >> 6);
  const int src = (int)((win >> 1) & 31u);
  const int slot = (int)(win & 1u);
  work(S);
  double* pr = prow + (S & 1) * BSD;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const bool me = lane == src && slot == r;
#pragma unroll
    for (int j = 0; j < BSD; j += 2) st2_if(me, pr + j, x[r][j], x[r][j + 1]);
  }
  wsync();
  double z[BSD];
#pragma unroll
  for (int j = 0; j < BSD; j += 2) {
    const double2 v = *reinterpret_cast<const double2*>(pr + j);
    z[j] = v.x;
    z[j + 1] = v.y;
  }
  const double p = z[S];
  const double rp = p < 0.0 ? -rap : rap;   // rcp64d is odd: bit-identical to rcp64d(p)
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const bool pv = pos[r] == q && kmask[r] != 0u;
    const double nf = pv ? 0.0 : -(x[r][S] * rp);
#pragma unroll
    for (int j = 0; j < BSD; ++j)
      if (j != S) x[r][j] = fma(nf, z[j], x[r][j]);
    x[r][S] = nf;   // compact D entry; 0 on the pivot row (W - S)
    kmask[r] = pv ? 0u : kmask[r];
    pos[r] = (pos[r] == k) ? q : pos[r];   // a3: the listing's swap of positions k and q (L156-L162)
    pos[r] = pv ? k : pos[r];
  }
  if (lane == 0) {
    rec_store(rec, k, p, q);
    rowk[k] = src + 32 * slot;
  }
}
template <int S, class Wk>
__device__ __forceinline__ void e_panel_steps(const int kb, double (&x)[2][BSD], uint32_t (&kmask)[2], int (&pos)[2],
                                              unsigned char* rec, int* rowk, int lane, double* prow, const Wk& work) {
  if constexpr (S < BSD) {
    e_panel_step<S>(kb + S, x, kmask, pos, rec, rowk, lane, prow, work);
    e_panel_steps<S + 1>(kb, x, kmask, pos, rec, rowk, lane, prow, work);
  }
}

template <int S, bool SROW = false>
__device__ __forceinline__ void d_panel_steps(const int kb, double (&x)[2][BSD], uint32_t (&kmask)[2], int (&pos)[2],
                                              int (&bs)[2], unsigned char* rec, int* rowk, int lane,
                                              double* prow = nullptr) {
  if constexpr (S < BSD) {
    d_panel_step<S, SROW>(kb + S, x, kmask, pos, bs, rec, rowk, lane, prow);
    d_panel_steps<S + 1, SROW>(kb, x, kmask, pos, bs, rec, rowk, lane, prow);
  }
}

// ------------------------------------------------------------------ K2e: one warp per matrix
// The same blocked elimination with the matrix resident in SHARED MEMORY (row stride 66
// doubles: a DMMA accumulator-fragment access of 8 rows x 4 lanes then spreads over all
// banks, 4 wavefronts per 512 B) and one warp doing everything for its matrix: the 8-step
// panel (d_panel_steps, K2d's chain), then per 8-column tile the block's B fragments (the
// pivot rows, read before the tile is written, so no copy of R is needed) and the 8 m-tiles'
// C fragments through DMMA.  Why: K2d's single panel warp per CTA holds the whole CTA at the
// per-step chain while the matrix occupies 4 warps' registers (4 CTAs per SM); here a
// matrix costs 35 KB of shared memory and 32 threads, so six panels run per SM.
#ifndef GJ_K2E_SWZ
#define GJ_K2E_SWZ 1
#endif
// Element (row, col) of the shared working array.  SWZ (default): row stride 64 doubles and
// the 16-byte chunk index XOR f(row), f = ((row & 1) << 2) | ((row >> 1) & 3): a bijection
// on 8 consecutive rows (a column access of 8 rows per LDS.128 phase hits 8 distinct
// chunks) with f(2p) ^ f(2p + 1) = 4 (the two rows of an accumulator-fragment phase use the
// two halves of the 128-byte line), so both access patterns run at 4 wavefronts per 512 B.
// Otherwise: padded stride 66 (8 wavefronts for the fragment pattern).
constexpr int MS = GJ_K2E_SWZ ? N64 : N64 + 2;
__device__ __forceinline__ int mix(int row, int col) {
  if constexpr (GJ_K2E_SWZ) {
    const int f = ((row & 1) << 2) | ((row >> 1) & 3);
    return row * N64 + ((((col >> 1) ^ f)) << 1) + (col & 1);
  } else {
    return row * MS + col;
  }
}
struct SmemE {
  static constexpr int M = 0;                              // [64][MS] the working array
  static constexpr int REC = M + N64 * MS * 8;             // [64] (p, q)
  static constexpr int ROW = REC + N64 * 16;               // [64] row pivoted at step k
  static constexpr int POS = ROW + N64 * 4;                // [64] final position of row i
  static constexpr int RP = POS + N64 * 4;                 // [64] 1 / p of step k
  static constexpr int PROW = RP + N64 * 8;                // [2][8] pivot-row broadcast
  static constexpr int BYTES = PROW + 2 * BSD * 8;
};
#ifndef GJ_K2E_SROW
#define GJ_K2E_SROW 1              // pivot row through shared memory + early 1/|p| (A/B option)
#endif
#ifndef GJ_K2E_NTU
#define GJ_K2E_NTU 2               // tile-loop unroll (measured: 1 13.5, 2 13.1, 4 13.2, 8 13.6 ms)
#endif
constexpr int kK2eNtu = GJ_K2E_NTU;
#ifndef GJ_K2G
#define GJ_K2G 1                   // K2g: register-resident trailing matrix (four trailing warps)
#endif
#ifndef GJ_K2E_TWO_WARPS
#define GJ_K2E_TWO_WARPS 1         // K2f: panel warp + trailing warp per matrix
#endif
#ifndef GJ_K2E_LA
#define GJ_K2E_LA 1                // look-ahead: panel kb + 1 factored under block kb's update (inverse)
#endif
#ifndef GJ_K2E_OVERLAP
#define GJ_K2E_OVERLAP 1           // load the next matrix under this one's store
#endif

// One 8-column tile of the block update: X[:, tile nt] += (W - S) R with the block's A
// fragments af and pivot rows rk0 / rk1 (B read before the tile is written: the pivot rows are
// rows of the tile).
__device__ __forceinline__ void e_tile_update(double* M, int nt, const double (&af)[8][2], int rk0, int rk1, int g,
                                              int t) {
  const double b0 = M[mix(rk0, 8 * nt + g)];   // B[t][g]: pivot row of step t, block start
  const double b1 = M[mix(rk1, 8 * nt + g)];
  wsync();
#pragma unroll
  for (int mt = 0; mt < 8; ++mt) {
    double2* cp = reinterpret_cast<double2*>(M + mix(8 * mt + g, 8 * nt + 2 * t));
    double2 c = *cp;
    dmma884(c.x, c.y, af[mt][0], b0);
    dmma884(c.x, c.y, af[mt][1], b1);
    *cp = c;
  }
}

// The six tiles other than the block's own and the look-ahead one, one per pivot step of the
// next panel (steps 0..5), in the order kb + 2, kb + 3, ... (mod 8).
struct TrailE {
  double* M;
  const double (&af)[8][2];
  int rk0, rk1, kb, g, t;
  __device__ __forceinline__ void operator()(int s) const {
    if (s < 6) e_tile_update(M, (kb + 2 + s) & 7, af, rk0, rk1, g, t);
  }
};

template <bool LA>
__global__ void __launch_bounds__(32, 6) gj_batched64e_kernel(BatchedArgs a) {
  extern __shared__ __align__(16) unsigned char smem_e[];
  double* M = reinterpret_cast<double*>(smem_e + SmemE::M);
  unsigned char* rec = smem_e + SmemE::REC;
  int* rowk = reinterpret_cast<int*>(smem_e + SmemE::ROW);
  int* posm = reinterpret_cast<int*>(smem_e + SmemE::POS);
  double* rpm = reinterpret_cast<double*>(smem_e + SmemE::RP);
  double* prow = reinterpret_cast<double*>(smem_e + SmemE::PROW);
  const int lane = threadIdx.x;
  const int g = lane >> 2, t = lane & 3;
  const double* __restrict__ Ag = static_cast<const double*>(a.A);
  double* __restrict__ Xg = static_cast<double*>(a.Ainv);

  bool loaded = false;   // this item's rows already in shared memory (loaded under the previous store)
  double rm_next = 0.0;
  for (int64_t item = blockIdx.x; item < a.batch; item += gridDim.x) {
    const double* Ai = Ag + item * (N64 * N64);
    if (item + gridDim.x < a.batch) {
      if (lane == 0) bulk_prefetch_l2(Ag + (item + gridDim.x) * (N64 * N64), N64 * N64 * 8);
    }
    // ---- a1: rows -> shared memory (one 512-byte row per instruction), max |a_ij|
    double rm = rm_next;
#pragma unroll 4
    for (int i0 = 0; i0 < (loaded ? 0 : N64); i0 += 8) {
      double2 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldcs(reinterpret_cast<const double2*>(Ai + (i0 + u) * N64) + lane);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        *reinterpret_cast<double2*>(M + mix(i0 + u, 2 * lane)) = v[u];
        rm = fmax(rm, fmax(fabs(v[u].x), fabs(v[u].y)));
      }
    }
    double tau;
    {
      const unsigned long long rb = (unsigned long long)__double_as_longlong(rm);
      const uint32_t mh = __reduce_max_sync(0xffffffffu, (uint32_t)(rb >> 32));
      const uint32_t ml = __reduce_max_sync(0xffffffffu, (uint32_t)(rb >> 32) == mh ? (uint32_t)rb : 0u);
      tau = a.tol * __longlong_as_double((long long)(((unsigned long long)mh << 32) | ml));
    }
    __syncwarp();
    uint32_t kmask[2] = {0xffffffffu, 0xffffffffu};
    int pos[2] = {lane, lane + 32};

    if constexpr (LA) {
      // look-ahead (inverse): block kb's update reaches tile kb + 1 first, then panel kb + 1
      // is factored while the other six tiles take block kb's update, one per pivot step
      double x[2][BSD];
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int j = 0; j < BSD; j += 2) {
          const double2 v = *reinterpret_cast<const double2*>(M + mix(lane + 32 * r, j));
          x[r][j] = v.x;
          x[r][j + 1] = v.y;
        }
      e_panel_steps<0>(0, x, kmask, pos, rec, rowk, lane, prow, NoWork{});
#pragma unroll 1
      for (int kb = 0; kb < N64 / BSD; ++kb) {
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int j = 0; j < BSD; j += 2)
            *reinterpret_cast<double2*>(M + mix(lane + 32 * r, 8 * kb + j)) = make_double2(x[r][j], x[r][j + 1]);
        wsync();
        double af[8][2];
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
          af[mt][0] = M[mix(8 * mt + g, 8 * kb + t)];       // A[g][t]
          af[mt][1] = M[mix(8 * mt + g, 8 * kb + 4 + t)];   // A[g][4 + t]
        }
        const int rk0 = rowk[kb * BSD + t], rk1 = rowk[kb * BSD + 4 + t];
        if (kb + 1 < N64 / BSD) {
          e_tile_update(M, kb + 1, af, rk0, rk1, g, t);
          wsync();
#pragma unroll
          for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int j = 0; j < BSD; j += 2) {
              const double2 v = *reinterpret_cast<const double2*>(M + mix(lane + 32 * r, 8 * (kb + 1) + j));
              x[r][j] = v.x;
              x[r][j + 1] = v.y;
            }
          e_panel_steps<0>((kb + 1) * BSD, x, kmask, pos, rec, rowk, lane, prow, TrailE{M, af, rk0, rk1, kb, g, t});
        } else {
#pragma unroll 1
          for (int j = 1; j < 8; ++j) e_tile_update(M, (kb + j) & 7, af, rk0, rk1, g, t);
        }
        wsync();
      }
    } else {
#pragma unroll 1
    for (int kb = 0; kb < N64 / BSD; ++kb) {
      // ---- the panel: rows lane, lane + 32 of column tile kb
      double x[2][BSD];
      int bs[2] = {-1, -1};
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int j = 0; j < BSD; j += 2) {
          const double2 v = *reinterpret_cast<const double2*>(M + mix(lane + 32 * r, 8 * kb + j));
          x[r][j] = v.x;
          x[r][j + 1] = v.y;
        }
      d_panel_steps<0, GJ_K2E_SROW != 0>(kb * BSD, x, kmask, pos, bs, rec, rowk, lane, prow);
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int j = 0; j < BSD; j += 2)
          *reinterpret_cast<double2*>(M + mix(lane + 32 * r, 8 * kb + j)) = make_double2(x[r][j], x[r][j + 1]);
      __syncwarp();
      // ---- X[:, ~panel] += (W - S) R, tile by tile on the FP64 tensor pipe
      double af[8][2];
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) {
        af[mt][0] = M[mix(8 * mt + g, 8 * kb + t)];       // A[g][t]
        af[mt][1] = M[mix(8 * mt + g, 8 * kb + 4 + t)];   // A[g][4 + t]
      }
      const int rk0 = rowk[kb * BSD + t], rk1 = rowk[kb * BSD + 4 + t];
#pragma unroll kK2eNtu
      for (int nt = 0; nt < 8; ++nt) {
        // determinant-only run: the compact D columns left of the panel are never read again
        if (nt == kb || (Xg == nullptr && nt < kb)) continue;
        const double b0 = M[mix(rk0, 8 * nt + g)];   // B[t][g]: pivot row of step t, block start
        const double b1 = M[mix(rk1, 8 * nt + g)];
        __syncwarp();                                  // every lane has its B before the tile is written
#if GJ_K2E_PHASED
        // all eight C fragments in flight: loads, then the k4 step 0 of every tile, then
        // step 1, then the stores (independent DMMAs back to back)
        double2 c[8];
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) c[mt] = *reinterpret_cast<const double2*>(M + mix(8 * mt + g, 8 * nt + 2 * t));
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) dmma884(c[mt].x, c[mt].y, af[mt][0], b0);
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) dmma884(c[mt].x, c[mt].y, af[mt][1], b1);
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) *reinterpret_cast<double2*>(M + mix(8 * mt + g, 8 * nt + 2 * t)) = c[mt];
#else
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
          double2* cp = reinterpret_cast<double2*>(M + mix(8 * mt + g, 8 * nt + 2 * t));
          double2 c = *cp;
          dmma884(c.x, c.y, af[mt][0], b0);
          dmma884(c.x, c.y, af[mt][1], b1);
          *cp = c;
        }
#endif
      }
      __syncwarp();
    }
    }   // LA

    // ---- a6: det / ipiv / singular flag from the record (steps lane, lane + 32)
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      posm[lane + 32 * r] = pos[r];
      double pk;
      int qk;
      rec_load(rec, lane + 32 * r, pk, qk);
      rpm[lane + 32 * r] = 1.0 / pk;
    }
    {
      unsigned fb0 = 0, fb1 = 0;
      int nswap = 0, nneg = 0;
      double lg = 0.0;
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int k = lane + 32 * r;
        double pk;
        int qk;
        rec_load(rec, k, pk, qk);
        const unsigned fb = __ballot_sync(0xffffffffu, fabs(pk) <= tau);
        if (r == 0) fb0 = fb; else fb1 = fb;
        nswap += __popc(__ballot_sync(0xffffffffu, qk != k));
        nneg += __popc(__ballot_sync(0xffffffffu, pk < 0.0));
        lg += log(fabs(pk));
        if (a.ipiv) a.ipiv[item * N64 + k] = qk + 1;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) lg += __shfl_xor_sync(0xffffffffu, lg, o);
      const int info = fb0 ? __ffs(fb0) : (fb1 ? 32 + __ffs(fb1) : 0);
      const int sgn = ((nswap ^ nneg) & 1) ? -1 : 1;
      if (lane == 0) {
        if (a.info) a.info[item] = info;
        if (a.logabsdet) a.logabsdet[item] = info ? -INFINITY : lg;
        if (a.sign) a.sign[item] = info ? 0 : (int8_t)sgn;
        if (a.det) static_cast<double*>(a.det)[item] = info ? 0.0 : (double)(sgn * exp(lg));
      }
    }
    __syncwarp();
    // ---- a7 + a8: Ainv[pos(i)][row(k)] = X[i][k] / p_pos(i) (+ 1 / p on the own entry)
    loaded = false;
    rm_next = 0.0;
    if (Xg != nullptr) {
      double* Xi = Xg + item * (N64 * N64);
      const int oc0 = rowk[lane], oc1 = rowk[lane + 32];
#if GJ_K2E_OVERLAP
      // the next matrix's rows stream in under this one's store: rows i0..i0+7 are loaded
      // while they are read out, and written once every lane has read them
      const int64_t nitem = item + gridDim.x;
      const bool pre = nitem < a.batch;
      const double* An = Ag + nitem * (N64 * N64);
#pragma unroll 1
      for (int i0 = 0; i0 < N64; i0 += 8) {
        double2 v[8];
        if (pre) {
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = __ldcs(reinterpret_cast<const double2*>(An + (i0 + u) * N64) + lane);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = i0 + u;
          const int ps = posm[i];
          const double rp = rpm[ps];
          double* orow = Xi + (int64_t)ps * N64;
          __stcs(orow + oc0, M[mix(i, lane)] * rp + (lane == ps ? rp : 0.0));
          __stcs(orow + oc1, M[mix(i, lane + 32)] * rp + (lane + 32 == ps ? rp : 0.0));
        }
        __syncwarp();
        if (pre) {
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            *reinterpret_cast<double2*>(M + mix(i0 + u, 2 * lane)) = v[u];
            rm_next = fmax(rm_next, fmax(fabs(v[u].x), fabs(v[u].y)));
          }
        }
      }
      loaded = pre;
#else
#pragma unroll 4
      for (int i = 0; i < N64; ++i) {
        const int ps = posm[i];
        const double rp = rpm[ps];
        double* orow = Xi + (int64_t)ps * N64;
        __stcs(orow + oc0, M[mix(i, lane)] * rp + (lane == ps ? rp : 0.0));
        __stcs(orow + oc1, M[mix(i, lane + 32)] * rp + (lane + 32 == ps ? rp : 0.0));
      }
#endif
    }
    __syncwarp();   // shared state is rewritten by the next matrix
  }
}


// ------------------------------------------------------------------ K2f: two warps per matrix
// K2e's layout and arithmetic with the panel chain and the trailing update on different warps
// of one CTA (64 threads per matrix, the same ~34 KB of shared memory): warp P factors panel
// kb + 1 while warp T applies block kb's update to the six other tiles — the update of tile
// kb + 1 comes first, and named barriers pass "panel kb stored" (P -> T) and "tile kb + 1
// updated" (T -> P).  Every output is bitwise K2e's (same operations in the same order per
// element); what changes is that the latency-bound chain and the DMMA work overlap, with two
// warps per matrix in flight on the SM instead of one.
__device__ __forceinline__ void nbar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void nbar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }
#ifndef GJ_K2F_WARPS
#define GJ_K2F_WARPS 2             // warps per matrix: panel + 1 or 2 trailing warps
#endif
constexpr int kFW = GJ_K2F_WARPS;
constexpr int BAR_PANEL = 1, BAR_TILE = 2;

// NTL tiles of the block update at once, phased for the trailing warp's ILP: every B, a warp
// barrier, every C fragment load, the k = 0..3 DMMAs, the k = 4..7 DMMAs, every store — so 8 x
// NTL independent accumulator chains are in flight instead of one tile's 8.
template <int NTL>
__device__ __forceinline__ void f_tiles_update(double* M, const int (&nts)[NTL], const double (&af)[8][2], int rk0,
                                               int rk1, int g, int t) {
  double b0[NTL], b1[NTL];
#pragma unroll
  for (int u = 0; u < NTL; ++u) {
    b0[u] = M[mix(rk0, 8 * nts[u] + g)];
    b1[u] = M[mix(rk1, 8 * nts[u] + g)];
  }
  wsync();   // every lane has its B (pivot rows are rows of the tiles) before any tile is written
  double2 c[NTL][8];
#pragma unroll
  for (int u = 0; u < NTL; ++u)
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) c[u][mt] = *reinterpret_cast<const double2*>(M + mix(8 * mt + g, 8 * nts[u] + 2 * t));
#pragma unroll
  for (int u = 0; u < NTL; ++u)
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) dmma884(c[u][mt].x, c[u][mt].y, af[mt][0], b0[u]);
#pragma unroll
  for (int u = 0; u < NTL; ++u)
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) dmma884(c[u][mt].x, c[u][mt].y, af[mt][1], b1[u]);
#pragma unroll
  for (int u = 0; u < NTL; ++u)
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) *reinterpret_cast<double2*>(M + mix(8 * mt + g, 8 * nts[u] + 2 * t)) = c[u][mt];
}

__global__ void __launch_bounds__(32 * kFW, 6) gj_batched64f_kernel(BatchedArgs a) {
  extern __shared__ __align__(16) unsigned char smem_e[];
  double* M = reinterpret_cast<double*>(smem_e + SmemE::M);
  unsigned char* rec = smem_e + SmemE::REC;
  int* rowk = reinterpret_cast<int*>(smem_e + SmemE::ROW);
  int* posm = reinterpret_cast<int*>(smem_e + SmemE::POS);
  double* rpm = reinterpret_cast<double*>(smem_e + SmemE::RP);
  double* prow = reinterpret_cast<double*>(smem_e + SmemE::PROW);
  double* rmx = rpm;   // [2] per-warp max |a_ij| (rpm is free until the epilogue)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const double* __restrict__ Ag = static_cast<const double*>(a.A);
  double* __restrict__ Xg = static_cast<double*>(a.Ainv);
  const int r0 = warp * 32;   // warps 0 and 1: their half of the rows for the load / store
  const bool io = warp < 2;

  bool loaded = false;
  double rm_next = 0.0;
  for (int64_t item = blockIdx.x; item < a.batch; item += gridDim.x) {
    const double* Ai = Ag + item * (N64 * N64);
    if (item + gridDim.x < a.batch && threadIdx.x == 0) bulk_prefetch_l2(Ag + (item + gridDim.x) * (N64 * N64), N64 * N64 * 8);
    // ---- a1: this warp's 32 rows -> shared memory, max |a_ij|
    double rm = rm_next;
#pragma unroll 2
    for (int i0 = r0; i0 < (loaded || !io ? r0 : r0 + 32); i0 += 8) {
      double2 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldcs(reinterpret_cast<const double2*>(Ai + (i0 + u) * N64) + lane);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        *reinterpret_cast<double2*>(M + mix(i0 + u, 2 * lane)) = v[u];
        rm = fmax(rm, fmax(fabs(v[u].x), fabs(v[u].y)));
      }
    }
    {
      const unsigned long long rb = (unsigned long long)__double_as_longlong(rm);
      const uint32_t mh = __reduce_max_sync(0xffffffffu, (uint32_t)(rb >> 32));
      const uint32_t ml = __reduce_max_sync(0xffffffffu, (uint32_t)(rb >> 32) == mh ? (uint32_t)rb : 0u);
      if (lane == 0 && io) rmx[warp] = __longlong_as_double((long long)(((unsigned long long)mh << 32) | ml));
    }
    __syncthreads();   // the whole matrix and both maxima are in shared memory
    const double tau = a.tol * fmax(rmx[0], rmx[1]);
    uint32_t kmask[2] = {0xffffffffu, 0xffffffffu};
    int pos[2] = {lane, lane + 32};

    if (warp == 0) {
      // ------------------------------------------------------------ P: the panels
#pragma unroll 1
      for (int kb = 0; kb < N64 / BSD; ++kb) {
        if (kb > 0) nbar_sync(BAR_TILE, 64);   // tile kb has block kb - 1's update
        double x[2][BSD];
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int j = 0; j < BSD; j += 2) {
            const double2 v = *reinterpret_cast<const double2*>(M + mix(lane + 32 * r, 8 * kb + j));
            x[r][j] = v.x;
            x[r][j + 1] = v.y;
          }
        e_panel_steps<0>(kb * BSD, x, kmask, pos, rec, rowk, lane, prow, NoWork{});
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int j = 0; j < BSD; j += 2)
            *reinterpret_cast<double2*>(M + mix(lane + 32 * r, 8 * kb + j)) = make_double2(x[r][j], x[r][j + 1]);
        nbar_arrive(BAR_PANEL, 32 * kFW);    // panel kb (W - S) and its record are stored
      }
    } else {
      // ------------------------------------------------------------ T: the block updates
      // (T1 = warp 1 takes the look-ahead tile first; with three warps T2 = warp 2 takes the
      // larger half of the rest)
      const int tw = warp - 1;
#pragma unroll 1
      for (int kb = 0; kb < N64 / BSD; ++kb) {
        nbar_sync(BAR_PANEL, 32 * kFW);
        double af[8][2];
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
          af[mt][0] = M[mix(8 * mt + g, 8 * kb + t)];       // A[g][t]
          af[mt][1] = M[mix(8 * mt + g, 8 * kb + 4 + t)];   // A[g][4 + t]
        }
        const int rk0 = rowk[kb * BSD + t], rk1 = rowk[kb * BSD + 4 + t];
        if (tw == 0 && kb + 1 < N64 / BSD) {
          const int la[1] = {kb + 1};
          f_tiles_update<1>(M, la, af, rk0, rk1, g, t);
          wsync();
          nbar_arrive(BAR_TILE, 64);
        }
        if (Xg != nullptr) {
          // the six other tiles (and at the last block tile 0 too), two at a time
          if constexpr (kFW == 2) {
#pragma unroll 1
            for (int j = 2; j < 8; j += 2) {
              const int pr[2] = {(kb + j) & 7, (kb + j + 1) & 7};
              f_tiles_update<2>(M, pr, af, rk0, rk1, g, t);
            }
            if (kb + 1 == N64 / BSD) {
              const int z0[1] = {0};
              f_tiles_update<1>(M, z0, af, rk0, rk1, g, t);
            }
          } else {
            if (tw == 0) {
              const int pr[2] = {(kb + 2) & 7, (kb + 3) & 7};
              f_tiles_update<2>(M, pr, af, rk0, rk1, g, t);
              if (kb + 1 == N64 / BSD) {
                const int z0[1] = {0};
                f_tiles_update<1>(M, z0, af, rk0, rk1, g, t);
              }
            } else {
              const int p1[2] = {(kb + 4) & 7, (kb + 5) & 7};
              f_tiles_update<2>(M, p1, af, rk0, rk1, g, t);
              const int p2[2] = {(kb + 6) & 7, (kb + 7) & 7};
              f_tiles_update<2>(M, p2, af, rk0, rk1, g, t);
            }
          }
        } else {
          // determinant-only run: only the tiles right of the next panel
#pragma unroll 1
          for (int nt = kb + 2 + (kFW == 3 ? tw : 0); nt < 8; nt += kFW - 1) {
            const int one[1] = {nt};
            f_tiles_update<1>(M, one, af, rk0, rk1, g, t);
          }
        }
      }
    }
    __syncthreads();   // the elimination is complete

    // ---- a6 (warp P holds the positions): det / ipiv / singular flag from the record
    if (warp == 0) {
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        posm[lane + 32 * r] = pos[r];
        double pk;
        int qk;
        rec_load(rec, lane + 32 * r, pk, qk);
        rpm[lane + 32 * r] = 1.0 / pk;
      }
      unsigned fb0 = 0, fb1 = 0;
      int nswap = 0, nneg = 0;
      double lg = 0.0;
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int k = lane + 32 * r;
        double pk;
        int qk;
        rec_load(rec, k, pk, qk);
        const unsigned fb = __ballot_sync(0xffffffffu, fabs(pk) <= tau);
        if (r == 0) fb0 = fb; else fb1 = fb;
        nswap += __popc(__ballot_sync(0xffffffffu, qk != k));
        nneg += __popc(__ballot_sync(0xffffffffu, pk < 0.0));
        lg += log(fabs(pk));
        if (a.ipiv) a.ipiv[item * N64 + k] = qk + 1;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) lg += __shfl_xor_sync(0xffffffffu, lg, o);
      const int info = fb0 ? __ffs(fb0) : (fb1 ? 32 + __ffs(fb1) : 0);
      const int sgn = ((nswap ^ nneg) & 1) ? -1 : 1;
      if (lane == 0) {
        if (a.info) a.info[item] = info;
        if (a.logabsdet) a.logabsdet[item] = info ? -INFINITY : lg;
        if (a.sign) a.sign[item] = info ? 0 : (int8_t)sgn;
        if (a.det) static_cast<double*>(a.det)[item] = info ? 0.0 : (double)(sgn * exp(lg));
      }
    }
    __syncthreads();
    // ---- a7 + a8: Ainv[pos(i)][row(k)] = X[i][k] / p_pos(i) (+ 1 / p on the own entry); each
    // warp stores its half of the rows and loads the next matrix's same half under the store
    loaded = false;
    rm_next = 0.0;
    if (Xg != nullptr && io) {
      double* Xi = Xg + item * (N64 * N64);
      const int oc0 = rowk[lane], oc1 = rowk[lane + 32];
      const int64_t nitem = item + gridDim.x;
      const bool pre = nitem < a.batch;
      const double* An = Ag + nitem * (N64 * N64);
#pragma unroll 1
      for (int i0 = r0; i0 < r0 + 32; i0 += 8) {
        double2 v[8];
        if (pre) {
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = __ldcs(reinterpret_cast<const double2*>(An + (i0 + u) * N64) + lane);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = i0 + u;
          const int ps = posm[i];
          const double rp = rpm[ps];
          double* orow = Xi + (int64_t)ps * N64;
          __stcs(orow + oc0, M[mix(i, lane)] * rp + (lane == ps ? rp : 0.0));
          __stcs(orow + oc1, M[mix(i, lane + 32)] * rp + (lane + 32 == ps ? rp : 0.0));
        }
        __syncwarp();
        if (pre) {
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            *reinterpret_cast<double2*>(M + mix(i0 + u, 2 * lane)) = v[u];
            rm_next = fmax(rm_next, fmax(fabs(v[u].x), fabs(v[u].y)));
          }
        }
      }
      loaded = pre;
    }
    __syncthreads();   // shared state is rewritten by the next matrix
  }
}


// ------------------------------------------------------------------ K2g: register-resident trailing matrix
// K2f's block algorithm with the trailing matrix in REGISTERS: four trailing warps T0..T3 hold
// rows 16 w .. 16 w + 15 as m8n8k4 accumulator fragments (2 m-tiles x 8 n-tiles x 2 doubles =
// 32 doubles per lane), warp P factors the panels exactly as K2f's P does.  Per block kb:
//   P:  panel kb (PANEL[kb & 1], 64 x 8) -> e_panel_steps -> W - S back into PANEL[kb & 1],
//       the block's pivot-step map (bsmap) -> arrive "panel kb factored";
//   T:  publish the block's pivot rows from their fragments (block-start values) into
//       BROWS[kb & 1] -> T barrier -> A fragments and tile kb (W - S) from PANEL[kb & 1] ->
//       tile kb + 1 (two DMMAs per m-tile) -> PANEL[(kb + 1) & 1] -> arrive "tile kb + 1
//       updated" -> the six (seven at the last block) other tiles.
// Same operations in the same order per element as K2e / K2f (the two k = 0..3 / 4..7 DMMAs of
// a tile, the panel steps), so every output is bitwise theirs; what changes is that C never
// makes the shared-memory round trip (K2f: ~65% of the shared pipe) and the block update runs
// on four warps.  The matrix passes through shared memory (M) only at the load and the
// un-permuted store.
#ifndef GJ_K2G_MINB
#define GJ_K2G_MINB 3
#endif
constexpr int kGT = 4;                         // trailing warps
constexpr int kGThreads = 32 * (kGT + 1);
constexpr int BAR_G_PANEL = 1, BAR_G_TILE = 2, BAR_G_T = 3;
constexpr int BRS = N64 + 4;                   // BROWS row stride (doubles): B-fragment reads hit 2 wavefronts
struct SmemG {
  static constexpr int M = 0;                                // [64][64] working array (mix layout)
  static constexpr int REC = M + N64 * N64 * 8;              // [64] (p, q)
  static constexpr int ROW = REC + N64 * 16;                 // [64] row pivoted at step k
  static constexpr int POS = ROW + N64 * 4;                  // [64] final position of row i
  static constexpr int RP = POS + N64 * 4;                   // [64] 1 / p of step k
  static constexpr int PROW = RP + N64 * 8;                  // [2][8] pivot-row broadcast (P)
  static constexpr int PANEL = PROW + 2 * BSD * 8;           // [2][64][8] panel / look-ahead tile
  static constexpr int BROWS = PANEL + 2 * N64 * BSD * 8;    // [2][8][BRS] the block's pivot rows
  static constexpr int BSMAP = BROWS + 2 * BSD * BRS * 8;    // [2][64] int8: block step of row i, or -1
  static constexpr int BYTES = BSMAP + 2 * N64;
};
// PANEL element (row, col): 64-byte rows, 16-byte chunk index XOR ((row >> 1) & 3) — P's row
// reads (8 rows per LDS.128 phase) and T's fragment accesses both hit 8 distinct chunks
__device__ __forceinline__ int pidx(int row, int col) {
  return row * BSD + ((((col >> 1) ^ ((row >> 1) & 3))) << 1) + (col & 1);
}

// Block KB's update of tiles N0, N0 + 1 (skipping the panel, the look-ahead tile and, in the
// determinant-only run, every tile left of the next panel), then the next pair.
template <int KB, int N0>
__device__ __forceinline__ void g_tiles(double2 (&C)[2][8], const double (&af)[2][2], const double* BR, int g, int t,
                                        bool inv) {
  if constexpr (N0 < N64 / BSD) {
    constexpr bool u0 = N0 != KB && N0 != KB + 1, u1 = N0 + 1 != KB && N0 + 1 != KB + 1;
    const bool d0 = u0 && (inv || N0 > KB + 1), d1 = u1 && (inv || N0 + 1 > KB + 1);
    double b00 = 0.0, b01 = 0.0, b10 = 0.0, b11 = 0.0;
    if (d0) {
      b00 = BR[t * BRS + 8 * N0 + g];
      b01 = BR[(4 + t) * BRS + 8 * N0 + g];
    }
    if (d1) {
      b10 = BR[t * BRS + 8 * (N0 + 1) + g];
      b11 = BR[(4 + t) * BRS + 8 * (N0 + 1) + g];
    }
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      if (d0) dmma884(C[mt][N0].x, C[mt][N0].y, af[mt][0], b00);
      if (d1) dmma884(C[mt][N0 + 1].x, C[mt][N0 + 1].y, af[mt][0], b10);
    }
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      if (d0) dmma884(C[mt][N0].x, C[mt][N0].y, af[mt][1], b01);
      if (d1) dmma884(C[mt][N0 + 1].x, C[mt][N0 + 1].y, af[mt][1], b11);
    }
    g_tiles<KB, N0 + 2>(C, af, BR, g, t, inv);
  }
}

// One T warp's block kb (static), fragments C[mt][n] = rows 16 tw + 8 mt + g, cols 8 n + 2 t.
template <int KB>
__device__ __forceinline__ void g_block(double2 (&C)[2][8], double* panel, double* brows, const int8_t* bsmap,
                                        int tw, int g, int t, bool inv) {
  constexpr int NB = N64 / BSD;
  nbar_sync(BAR_G_PANEL, kGThreads);   // P: panel KB factored (W - S), its map stored
  const double* PB = panel + (KB & 1) * N64 * BSD;
  double* BR = brows + (KB & 1) * BSD * BRS;
  const int8_t* bm = bsmap + (KB & 1) * N64;
  // publish the block's pivot rows (their values at block start): the lanes holding one
#pragma unroll
  for (int mt = 0; mt < 2; ++mt) {
    const int s = bm[16 * tw + 8 * mt + g];
    double* dst = BR + (s < 0 ? 0 : s) * BRS + 2 * t;
#pragma unroll
    for (int n = 0; n < NB; ++n)
      if (n != KB && (inv || n > KB)) st2_if(s >= 0, dst + 8 * n, C[mt][n].x, C[mt][n].y);
  }
  nbar_sync(BAR_G_T, 32 * kGT);        // every pivot row of the block is published
  double af[2][2];
#pragma unroll
  for (int mt = 0; mt < 2; ++mt) {
    const int r = 16 * tw + 8 * mt + g;
    af[mt][0] = PB[pidx(r, t)];        // A[g][t]
    af[mt][1] = PB[pidx(r, 4 + t)];    // A[g][4 + t]
    C[mt][KB] = *reinterpret_cast<const double2*>(PB + pidx(r, 2 * t));   // the factored panel
  }
  if constexpr (KB + 1 < NB) {
    const double b0 = BR[t * BRS + 8 * (KB + 1) + g], b1 = BR[(4 + t) * BRS + 8 * (KB + 1) + g];
    double* PN = panel + ((KB + 1) & 1) * N64 * BSD;
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      dmma884(C[mt][KB + 1].x, C[mt][KB + 1].y, af[mt][0], b0);
      dmma884(C[mt][KB + 1].x, C[mt][KB + 1].y, af[mt][1], b1);
      *reinterpret_cast<double2*>(PN + pidx(16 * tw + 8 * mt + g, 2 * t)) = C[mt][KB + 1];
    }
    nbar_arrive(BAR_G_TILE, kGThreads);   // tile KB + 1 has block KB's update
  }
  // the other tiles, two at a time: their B, the k = 0..3 DMMAs, then k = 4..7
  g_tiles<KB, 0>(C, af, BR, g, t, inv);
}
template <int KB>
__device__ __forceinline__ void g_blocks(double2 (&C)[2][8], double* panel, double* brows, const int8_t* bsmap, int tw,
                                         int g, int t, bool inv) {
  if constexpr (KB < N64 / BSD) {
    g_block<KB>(C, panel, brows, bsmap, tw, g, t, inv);
    g_blocks<KB + 1>(C, panel, brows, bsmap, tw, g, t, inv);
  }
}

__global__ void __launch_bounds__(kGThreads, GJ_K2G_MINB) gj_batched64g_kernel(BatchedArgs a) {
  extern __shared__ __align__(16) unsigned char smem_g[];
  double* M = reinterpret_cast<double*>(smem_g + SmemG::M);
  unsigned char* rec = smem_g + SmemG::REC;
  int* rowk = reinterpret_cast<int*>(smem_g + SmemG::ROW);
  int* posm = reinterpret_cast<int*>(smem_g + SmemG::POS);
  double* rpm = reinterpret_cast<double*>(smem_g + SmemG::RP);
  double* prow = reinterpret_cast<double*>(smem_g + SmemG::PROW);
  double* panel = reinterpret_cast<double*>(smem_g + SmemG::PANEL);
  double* brows = reinterpret_cast<double*>(smem_g + SmemG::BROWS);
  int8_t* bsmap = reinterpret_cast<int8_t*>(smem_g + SmemG::BSMAP);
  double* rmx = rpm;   // [4] per-warp max |a_ij| (rpm is free until the epilogue)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const double* __restrict__ Ag = static_cast<const double*>(a.A);
  double* __restrict__ Xg = static_cast<double*>(a.Ainv);
  const bool inv = Xg != nullptr;
  const int r0 = warp * 16;   // warps 0..3: their quarter of the rows for the load / store
  const bool io = warp < 4;

  bool loaded = false;
  double rm_next = 0.0;
  for (int64_t item = blockIdx.x; item < a.batch; item += gridDim.x) {
    const double* Ai = Ag + item * (N64 * N64);
    if (item + gridDim.x < a.batch && threadIdx.x == 0) bulk_prefetch_l2(Ag + (item + gridDim.x) * (N64 * N64), N64 * N64 * 8);
    // ---- a1: this warp's 16 rows -> shared memory, max |a_ij|
    double rm = rm_next;
    if (!loaded && io) {
#pragma unroll
      for (int i0 = r0; i0 < r0 + 16; i0 += 8) {
        double2 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcs(reinterpret_cast<const double2*>(Ai + (i0 + u) * N64) + lane);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          *reinterpret_cast<double2*>(M + mix(i0 + u, 2 * lane)) = v[u];
          rm = fmax(rm, fmax(fabs(v[u].x), fabs(v[u].y)));
        }
      }
    }
    {
      const unsigned long long rb = (unsigned long long)__double_as_longlong(rm);
      const uint32_t mh = __reduce_max_sync(0xffffffffu, (uint32_t)(rb >> 32));
      const uint32_t ml = __reduce_max_sync(0xffffffffu, (uint32_t)(rb >> 32) == mh ? (uint32_t)rb : 0u);
      if (lane == 0 && io) rmx[warp] = __longlong_as_double((long long)(((unsigned long long)mh << 32) | ml));
    }
    __syncthreads();   // the whole matrix and the maxima are in shared memory
    const double tau = a.tol * fmax(fmax(rmx[0], rmx[1]), fmax(rmx[2], rmx[3]));
    uint32_t kmask[2] = {0xffffffffu, 0xffffffffu};
    int pos[2] = {lane, lane + 32};

    if (warp == 0) {
      // ------------------------------------------------------------ P: the panels
#pragma unroll 1
      for (int kb = 0; kb < N64 / BSD; ++kb) {
        double x[2][BSD];
        if (kb == 0) {
#pragma unroll
          for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int j = 0; j < BSD; j += 2) {
              const double2 v = *reinterpret_cast<const double2*>(M + mix(lane + 32 * r, j));
              x[r][j] = v.x;
              x[r][j + 1] = v.y;
            }
        } else {
          nbar_sync(BAR_G_TILE, kGThreads);   // tile kb has block kb - 1's update
          const double* PB = panel + (kb & 1) * N64 * BSD;
#pragma unroll
          for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int j = 0; j < BSD; j += 2) {
              const double2 v = *reinterpret_cast<const double2*>(PB + pidx(lane + 32 * r, j));
              x[r][j] = v.x;
              x[r][j + 1] = v.y;
            }
        }
        e_panel_steps<0>(kb * BSD, x, kmask, pos, rec, rowk, lane, prow, NoWork{});
        double* PB = panel + (kb & 1) * N64 * BSD;
        int8_t* bm = bsmap + (kb & 1) * N64;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
#pragma unroll
          for (int j = 0; j < BSD; j += 2)
            *reinterpret_cast<double2*>(PB + pidx(lane + 32 * r, j)) = make_double2(x[r][j], x[r][j + 1]);
          const int bs = pos[r] - kb * BSD;
          bm[lane + 32 * r] = (int8_t)((kmask[r] == 0u && bs >= 0 && bs < BSD) ? bs : -1);
        }
        nbar_arrive(BAR_G_PANEL, kGThreads);   // panel kb (W - S), its record and map are stored
      }
    } else {
      // ------------------------------------------------------------ T: the block updates
      const int tw = warp - 1;
      double2 C[2][8];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int n = 0; n < 8; ++n) C[mt][n] = *reinterpret_cast<const double2*>(M + mix(16 * tw + 8 * mt + g, 8 * n + 2 * t));
      g_blocks<0>(C, panel, brows, bsmap, tw, g, t, inv);
      if (inv) {
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int n = 0; n < 8; ++n) *reinterpret_cast<double2*>(M + mix(16 * tw + 8 * mt + g, 8 * n + 2 * t)) = C[mt][n];
      }
    }
    __syncthreads();   // the elimination is complete (M holds the compact result)

    // ---- a6 (warp P holds the positions): det / ipiv / singular flag from the record
    if (warp == 0) {
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        posm[lane + 32 * r] = pos[r];
        double pk;
        int qk;
        rec_load(rec, lane + 32 * r, pk, qk);
        rpm[lane + 32 * r] = 1.0 / pk;
      }
      unsigned fb0 = 0, fb1 = 0;
      int nswap = 0, nneg = 0;
      double lg = 0.0;
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int k = lane + 32 * r;
        double pk;
        int qk;
        rec_load(rec, k, pk, qk);
        const unsigned fb = __ballot_sync(0xffffffffu, fabs(pk) <= tau);
        if (r == 0) fb0 = fb; else fb1 = fb;
        nswap += __popc(__ballot_sync(0xffffffffu, qk != k));
        nneg += __popc(__ballot_sync(0xffffffffu, pk < 0.0));
        lg += log(fabs(pk));
        if (a.ipiv) a.ipiv[item * N64 + k] = qk + 1;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) lg += __shfl_xor_sync(0xffffffffu, lg, o);
      const int info = fb0 ? __ffs(fb0) : (fb1 ? 32 + __ffs(fb1) : 0);
      const int sgn = ((nswap ^ nneg) & 1) ? -1 : 1;
      if (lane == 0) {
        if (a.info) a.info[item] = info;
        if (a.logabsdet) a.logabsdet[item] = info ? -INFINITY : lg;
        if (a.sign) a.sign[item] = info ? 0 : (int8_t)sgn;
        if (a.det) static_cast<double*>(a.det)[item] = info ? 0.0 : (double)(sgn * exp(lg));
      }
    }
    __syncthreads();
    // ---- a7 + a8: Ainv[pos(i)][row(k)] = X[i][k] / p_pos(i) (+ 1 / p on the own entry); warps
    // 0..3 store their quarter of the rows and load the next matrix's same quarter under it
    loaded = false;
    rm_next = 0.0;
    if (inv && io) {
      double* Xi = Xg + item * (N64 * N64);
      const int oc0 = rowk[lane], oc1 = rowk[lane + 32];
      const int64_t nitem = item + gridDim.x;
      const bool pre = nitem < a.batch;
      const double* An = Ag + nitem * (N64 * N64);
#pragma unroll 1
      for (int i0 = r0; i0 < r0 + 16; i0 += 8) {
        double2 v[8];
        if (pre) {
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = __ldcs(reinterpret_cast<const double2*>(An + (i0 + u) * N64) + lane);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = i0 + u;
          const int ps = posm[i];
          const double rp = rpm[ps];
          double* orow = Xi + (int64_t)ps * N64;
          __stcs(orow + oc0, M[mix(i, lane)] * rp + (lane == ps ? rp : 0.0));
          __stcs(orow + oc1, M[mix(i, lane + 32)] * rp + (lane + 32 == ps ? rp : 0.0));
        }
        __syncwarp();
        if (pre) {
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            *reinterpret_cast<double2*>(M + mix(i0 + u, 2 * lane)) = v[u];
            rm_next = fmax(rm_next, fmax(fabs(v[u].x), fabs(v[u].y)));
          }
        }
      }
      loaded = pre;
    }
    __syncthreads();   // shared state is rewritten by the next matrix
  }
}

}  // namespace

cudaError_t launch_batched64e(const BatchedArgs& a, cudaStream_t s) {
  if (a.n != N64 || a.batch <= 0) return cudaErrorInvalidValue;
  // 16-byte vector loads / stores of A and the inverse (__ldcs double2): an 8-byte-aligned
  // batch (e.g. a 1-D buffer sliced at an odd element) goes to the generic K2 instead
  if ((reinterpret_cast<uintptr_t>(a.A) & 15) || (a.Ainv && (reinterpret_cast<uintptr_t>(a.Ainv) & 15)))
    return cudaErrorNotSupported;
  const int smem = SmemE::BYTES;
  static unsigned long long configured = 0;
  const unsigned long long dbit = device_bit();
  if (!(configured & dbit)) {
    for (auto kern : {gj_batched64e_kernel<true>, gj_batched64e_kernel<false>}) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e != cudaSuccess) return e;
    }
    cudaError_t e2 = cudaFuncSetAttribute(gj_batched64f_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e2 != cudaSuccess) return e2;
    configured |= dbit;
  }
  int per_sm = 0;
#if GJ_K2G
  if (true) {
    static unsigned long long configured_g = 0;
    if (!(configured_g & dbit)) {
      cudaError_t e = cudaFuncSetAttribute(gj_batched64g_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SmemG::BYTES);
      if (e != cudaSuccess) return e;
      configured_g |= dbit;
    }
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gj_batched64g_kernel, kGThreads, SmemG::BYTES);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
    const int64_t cap = (int64_t)device_sm_count() * per_sm;
    const int grid = (int)(a.batch < cap ? a.batch : cap);
    gj_batched64g_kernel<<<grid, kGThreads, SmemG::BYTES, s>>>(a);
    return cudaGetLastError();
  }
#endif
#if GJ_K2E_TWO_WARPS
  auto kern = gj_batched64f_kernel;
  const int threads = 32 * kFW;
#else
  auto kern = a.Ainv != nullptr ? gj_batched64e_kernel<GJ_K2E_LA != 0> : gj_batched64e_kernel<false>;
  const int threads = 32;
#endif
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const int64_t cap = (int64_t)device_sm_count() * per_sm;
  const int grid = (int)(a.batch < cap ? a.batch : cap);
  kern<<<grid, threads, smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace gj

