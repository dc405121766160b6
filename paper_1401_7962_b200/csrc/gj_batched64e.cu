// K2f — the C3 hot path (BASELINE configs[2]): batched Gauss–Jordan for fp64 n = 64, the
// matrix resident in SHARED MEMORY, two warps per matrix (a panel warp P and a trailing warp
// T), the blocked trailing update on the FP64 tensor pipe (DMMA, mma.sync m8n8k4 f64).
//
// The elimination (§2, Eqs. (14)-(15), L61-L72; Obs. 2-3 L59-L60; listing
// L150-L177) runs in blocks of BS pivot steps (BS = 8; 16 as a build option), the
// aggregation K1b uses:
//   P: the block's BS panel columns (rows lane, lane + 32) in registers, factored step by
//      step: max |x_ik| over the un-pivoted rows (fp64 keys: high word, then low word), ties
//      to the smallest physical position (reading G3), logical swaps, deferred normalisation,
//      the pivot row's own compact entry held as W - S = 0; the pivot row's panel values
//      travel through a small shared buffer (one writer, broadcast reads, buffered by step
//      parity) and 1/|p| starts from the winning key before the winner is known; W - S goes
//      back to shared memory with the block's record;
//   T: X[:, ~panel] += (W - S) R tile by tile (8 columns per tile): per tile the BS/4 B
//      fragments are read from the block's pivot rows (before the tile is written, so no copy
//      of R), then the eight m-tiles' C fragments go LDS.128 -> BS/4 DMMAs -> STS.128.
//      Panel kb + 1's tiles come first; named barriers pass "panel kb stored" (P -> T) and
//      "panel kb + 1 updated" (T -> P), so P factors panel kb + 1 while T updates the rest.
// Layout: row stride 64 doubles with the 16-byte chunk index XOR f(row), f = ((row & 1) << 2)
// | ((row >> 1) & 3) — the panel's column access (8 rows per LDS.128 phase) and the
// accumulator-fragment access (rows 2p, 2p + 1 x 4 lanes per phase) both hit 8 distinct
// chunks.  A matrix costs ~34 KB of shared memory and 64 threads, so six run per SM.
// BS = 16 halves the blocks (and T's C-fragment round trips through shared memory, the largest
// share of the shared pipe) but doubles the panel chain's work per step; measured slower
// (C3 11.6 vs 9.6 ms, profiles/r02_k2f_summary.md), so BS = 8.
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
#ifndef GJ_K2_BS
#define GJ_K2_BS 8
#endif
constexpr int BS = GJ_K2_BS;       // block size: pivot steps (panel columns) per block
constexpr int NB = N64 / BS;       // blocks
constexpr int TPB = BS / 8;        // 8-column tiles per panel
constexpr int KS = BS / 4;         // k4 steps of a tile update
static_assert(BS == 8 || BS == 16, "block size");
#ifndef GJ_K2_NTL
#define GJ_K2_NTL (BS == 8 ? 2 : 1)  // tiles per T phase (register budget)
#endif
constexpr int NTL = GJ_K2_NTL;
#ifndef GJ_K2_TW
#define GJ_K2_TW 1                 // trailing warps per matrix (2: T0 = look-ahead + a share, T1 = the rest)
#endif
constexpr int TW = GJ_K2_TW;
constexpr int kThreads = 32 * (1 + TW);
#ifndef GJ_K2_MINB
#define GJ_K2_MINB (TW == 1 ? 6 : 5)
#endif

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ double rcp64d(double p) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(p));
  double e = fma(-p, r, 1.0);
  r = fma(r, e, r);
  e = fma(-p, r, 1.0);
  return fma(r, e, r);
}
// Warp barrier with memory ordering among the lanes that ptxas does not turn into a
// divergence check + branch (as __syncwarp does): the panel step stays one basic block.
__device__ __forceinline__ void wsync() { asm volatile("bar.warp.sync 0xffffffff;" ::: "memory"); }
__device__ __forceinline__ void st2_if(bool p, double* addr, double a, double b) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %0, 0;\n\t@q st.shared.v2.f64 [%1], {%2, %3};\n}" ::"r"(p ? 1u : 0u),
               "r"((uint32_t)__cvta_generic_to_shared(addr)), "d"(a), "d"(b)
               : "memory");
}
__device__ __forceinline__ void nbar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void nbar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// P's pivot step S (static) at global step k on the panel rows lane and lane + 32.
template <int S>
__device__ __forceinline__ void panel_step(const int k, double (&x)[2][BS], uint32_t (&kmask)[2], int (&pos)[2],
                                           unsigned char* rec, int* rowk, int lane, double* prow) {
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
  // |p| is the winning key itself: 1/|p| starts before the winner is known
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
  // the pivot row's panel values: one writer (predicated stores), broadcast reads
  double* pr = prow + (S & 1) * BS;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const bool me = lane == src && slot == r;
#pragma unroll
    for (int j = 0; j < BS; j += 2) st2_if(me, pr + j, x[r][j], x[r][j + 1]);
  }
  wsync();
  double z[BS];
#pragma unroll
  for (int j = 0; j < BS; j += 2) {
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
    for (int j = 0; j < BS; ++j)
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
template <int S>
__device__ __forceinline__ void panel_steps(const int kb, double (&x)[2][BS], uint32_t (&kmask)[2], int (&pos)[2],
                                            unsigned char* rec, int* rowk, int lane, double* prow) {
  if constexpr (S < BS) {
    panel_step<S>(kb + S, x, kmask, pos, rec, rowk, lane, prow);
    panel_steps<S + 1>(kb, x, kmask, pos, rec, rowk, lane, prow);
  }
}

// Element (row, col) of the shared working array: row stride 64 doubles and the 16-byte
// chunk index XOR f(row), f = ((row & 1) << 2) | ((row >> 1) & 3): a bijection on 8
// consecutive rows (a column access of 8 rows per LDS.128 phase hits 8 distinct chunks) with
// f(2p) ^ f(2p + 1) = 4 (the two rows of an accumulator-fragment phase use the two halves of
// the 128-byte line), so both access patterns run at 4 wavefronts per 512 B.
__device__ __forceinline__ int mix(int row, int col) {
  const int f = ((row & 1) << 2) | ((row >> 1) & 3);
  return row * N64 + ((((col >> 1) ^ f)) << 1) + (col & 1);
}
struct SmemE {
  static constexpr int M = 0;                              // [64][64] the working array
  static constexpr int REC = M + N64 * N64 * 8;            // [64] (p, q)
  static constexpr int ROW = REC + N64 * 16;               // [64] row pivoted at step k
  static constexpr int POS = ROW + N64 * 4;                // [64] final position of row i
  static constexpr int RP = POS + N64 * 4;                 // [64] 1 / p of step k
  static constexpr int PROW = RP + N64 * 8;                // [2][BS] pivot-row broadcast
  static constexpr int BYTES = PROW + 2 * BS * 8;
};
constexpr int BAR_PANEL = 1, BAR_TILE = 2;

// NT tiles of block kb's update at once, phased for the trailing warp's ILP: every B, a warp
// barrier, every C fragment load, then the DMMAs k4 step by k4 step, then every store — so
// 8 x NT independent accumulator chains are in flight.
template <int NT>
__device__ __forceinline__ void tiles_update(double* M, const int (&nts)[NT], const double (&af)[8][KS],
                                             const int (&rk)[KS], int g, int gr, int t) {
  double b[NT][KS];
#pragma unroll
  for (int u = 0; u < NT; ++u)
#pragma unroll
    for (int k = 0; k < KS; ++k) b[u][k] = M[mix(rk[k], 8 * nts[u] + g)];   // B[4k + t][g]
  wsync();   // every lane has its B (pivot rows are rows of the tiles) before any tile is written
  double2 c[NT][8];
#pragma unroll
  for (int u = 0; u < NT; ++u)
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) c[u][mt] = *reinterpret_cast<const double2*>(M + mix(8 * mt + gr, 8 * nts[u] + 2 * t));
#pragma unroll
  for (int k = 0; k < KS; ++k)
#pragma unroll
    for (int u = 0; u < NT; ++u)
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) dmma884(c[u][mt].x, c[u][mt].y, af[mt][k], b[u][k]);
#pragma unroll
  for (int u = 0; u < NT; ++u)
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) *reinterpret_cast<double2*>(M + mix(8 * mt + gr, 8 * nts[u] + 2 * t)) = c[u][mt];
}

__global__ void __launch_bounds__(kThreads, GJ_K2_MINB) gj_batched64f_kernel(BatchedArgs a) {
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
  // T's fragment row of lane group g: 0, 1, 4, 5, 2, 3, 6, 7 (a row relabelling, free for A and
  // C): the four rows of a half-warp's 8-byte A-fragment load then sit in different chunk
  // pairs of the swizzled layout (ncu: these loads were 2-way bank-conflicted), while the
  // accumulator pairs (2p, 2p + 1) of a quarter-warp's 16-byte C access stay together
  const int gr = (g & 1) | ((g & 2) << 1) | ((g & 4) >> 1);
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
      for (int kb = 0; kb < NB; ++kb) {
        if (kb > 0) nbar_sync(BAR_TILE, 64);   // panel kb has block kb - 1's update (P + T0)
        double x[2][BS];
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int j = 0; j < BS; j += 2) {
            const double2 v = *reinterpret_cast<const double2*>(M + mix(lane + 32 * r, BS * kb + j));
            x[r][j] = v.x;
            x[r][j + 1] = v.y;
          }
        panel_steps<0>(kb * BS, x, kmask, pos, rec, rowk, lane, prow);
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int j = 0; j < BS; j += 2)
            *reinterpret_cast<double2*>(M + mix(lane + 32 * r, BS * kb + j)) = make_double2(x[r][j], x[r][j + 1]);
        nbar_arrive(BAR_PANEL, kThreads);   // panel kb (W - S) and its record are stored
      }
    } else {
      // ------------------------------------------------------------ T: the block updates
      const int tw = warp - 1;
#pragma unroll 1
      for (int kb = 0; kb < NB; ++kb) {
        nbar_sync(BAR_PANEL, kThreads);
        double af[8][KS];
#pragma unroll
        for (int mt = 0; mt < 8; ++mt)
#pragma unroll
          for (int k = 0; k < KS; ++k) af[mt][k] = M[mix(8 * mt + gr, BS * kb + 4 * k + t)];   // A[gr][4k + t]
        int rk[KS];
#pragma unroll
        for (int k = 0; k < KS; ++k) rk[k] = rowk[kb * BS + 4 * k + t];
        const int nt1 = (kb + 1) * TPB;   // first tile of panel kb + 1
        if (tw == 0 && kb + 1 < NB) {
          // panel kb + 1 first, then release P to factor it
#pragma unroll
          for (int u = 0; u < TPB; ++u) {
            const int la[1] = {nt1 + u};
            tiles_update<1>(M, la, af, rk, g, gr, t);
          }
          wsync();
          nbar_arrive(BAR_TILE, 64);
        }
        // the other tiles: every tile outside panels kb and kb + 1 (inverse; from the tile
        // after them on, wrapping), or only those right of panel kb + 1 (determinant only)
        const int first = (kb + (Xg != nullptr && kb + 1 == NB ? 1 : 2)) * TPB;
        const int cnt = Xg != nullptr ? 8 - TPB * (kb + 1 < NB ? 2 : 1) : (first < 8 ? 8 - first : 0);
        // with two trailing warps: T0 (which also took panel kb + 1) the first (cnt - 1) / 2
        const int h = TW == 2 ? (cnt - 1) / 2 : cnt;
        const int j0 = tw == 0 ? 0 : h, j1 = tw == 0 ? h : cnt;
#pragma unroll 1
        for (int j = j0; j < j1; j += NTL) {
          if (NTL == 2 && j + 1 < j1) {
            const int pr[2] = {(first + j) & 7, (first + j + 1) & 7};
            tiles_update<2>(M, pr, af, rk, g, gr, t);
          } else {
            const int one[1] = {(first + j) & 7};
            tiles_update<1>(M, one, af, rk, g, gr, t);
            if (NTL == 2) break;
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
    cudaError_t e = cudaFuncSetAttribute(gj_batched64f_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    configured |= dbit;
  }
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gj_batched64f_kernel, kThreads, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const int64_t cap = (int64_t)device_sm_count() * per_sm;
  const int grid = (int)(a.batch < cap ? a.batch : cap);
  gj_batched64f_kernel<<<grid, kThreads, smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace gj
