// K4b — the trailing update of the large-n path (a9; Eqs. (14)-(15) aggregated over a
// 128-column panel):
//     C[i][c] = (replace(i) ? 0 : C[i][c]) + sum_{s < 128} W[i][s] R[s][c]
// with W = X[:, P0 .. P0 + 128) (the factored panel, W - S convention), R = the panel's pivot
// rows taken before the update, C = X at every column outside the panel (and, in the det /
// solve modes, only right of the next panel), replace(i) = row i was pivoted in this panel.
//
// An FP64 tensor-core GEMM with K = 128 on sm_100a: tcgen05 has no f64 kind, so the MMA is
// the warp-level mma.sync.m16n8k16.f64 (SASS DMMA.8x8x4, the FP64 pipe's full rate).
// Round 1's kernel (gemm_update_kernel in gj_large.cu) pulled C synchronously into registers
// at every tile, fed A/B with cp.async + __syncthreads per 16-deep slab and ran at ~73% of
// the DMMA rate of its SMs.  This one is warp-specialised and persistent:
//   * one producer warp streams the operands with TMA (cp.async.bulk.tensor, 128-byte
//     swizzle, 16 x 64 fp64 boxes): the CTA's A block (64 rows x 128 = 64 KB) stays in
//     shared memory while the CTA walks its contiguous run of tiles along N, and the B block
//     of each 64-column tile (R^T, 64 KB) is double-buffered behind full / empty mbarriers;
//   * CW consumer warps own 64 x 64 tiles split into 32 x (64 / (CW / 2)) warp tiles; each
//     k16 step reads its fragments from one swizzled box (conflict-free 8-byte loads) and
//     issues the m16n8k16 MMAs; C of the NEXT tile is loaded from global memory into
//     registers while this one computes, and results are stored straight from registers —
//     no shared-memory round trip for C, no block-wide barrier anywhere in the loop.
// One CTA per SM (192 KB of shared memory), persistent over the tile grid in M-major order so
// each CTA reloads A about once.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

#include "gj_internal.h"
#include "gj_ptx.cuh"

namespace gj {
namespace {

using namespace ptx;
#ifdef GJ_TIMELINE
__device__ unsigned long long g_tlg[3][512];
#endif

#ifndef GJ_DGEMM_WM
#define GJ_DGEMM_WM 2
#endif
constexpr int WMW = GJ_DGEMM_WM;             // consumer warps along M (32 rows each)
constexpr int TM = 32 * WMW, TN = 64, TK = 128;   // tile and the panel width K
constexpr int KB = 16;                       // one TMA box = 16 doubles = 128 bytes wide
constexpr int NBOX = TK / KB;                // 8 boxes per operand block
constexpr int BOX_BYTES = 64 * KB * 8;       // 8 KB: a 64-row B box
constexpr int BLK_BYTES = NBOX * BOX_BYTES;  // 64 KB: one B block
constexpr int ABOX_BYTES = TM * KB * 8;      // a TM-row A box
constexpr int ABLK_BYTES = NBOX * ABOX_BYTES;

struct DSmem {
  static constexpr int A = 0;
  static constexpr int B = A + ABLK_BYTES;                // [2 stages]
  static constexpr int BAR = B + 2 * BLK_BYTES;           // a_full, a_empty, full[2], empty[2]
  static constexpr int META = BAR + 64;                   // [2] (tile, next tile) per B stage
  static constexpr int BYTES = META + 32 + 1024;          // + alignment slack
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

__device__ __forceinline__ void dmma16816(double (&c)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
      "{%12,%13,%14,%15}, {%0,%1,%2,%3};"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]), "d"(b[1]),
        "d"(b[2]), "d"(b[3]));
}

// (row, col) of a 64 x 16 fp64 box stored with the 128-byte TMA swizzle (16-byte chunk index
// XOR row mod 8): byte offset.  Lanes (g, t) reading (r0 + g, c0 + t) hit 32 distinct banks.
__device__ __forceinline__ uint32_t boxoff(int r, int c) {
  return (uint32_t)(r * 128 + ((((c >> 1) ^ (r & 7)) << 4) | ((c & 1) << 3)));
}
__device__ __forceinline__ double lds64(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}

__device__ __forceinline__ int real_col(const DgemmArgs& g, int nc) {
  const int c = g.c_base + nc;
  return (g.skip_hi > g.skip_lo && c >= g.skip_lo) ? c + (g.skip_hi - g.skip_lo) : c;
}

// Tile schedule: CTA b takes a contiguous range of the M-major tile order, so it reloads its A
// block about once.  The ranges are weighted (DgemmArgs::late_from / late_w): launched beside
// the panel kernel, the last CTAs of the grid wait for the panel kernel's SMs and get shorter
// ranges sized to the time left after it ends.  (Measured and dropped: a counter-based dynamic
// schedule and work stealing from the back of the ranges, meant to put the panel kernel's 16
// SMs to work once it ends — the A reloads they cost outweighed the gain: C4 40.8 / 44.4 ms
// against 40.6 ms static; tools/timeline_large.py.)

template <int CW>
__global__ void __launch_bounds__((CW + 1) * 32, 1) dgemm_tma_kernel(DgemmArgs g, const __grid_constant__ CUtensorMap ma,
                                                                     const __grid_constant__ CUtensorMap mb) {
  constexpr int WN = CW / WMW;            // warps along N
  constexpr int WTN = TN / WN;            // warp tile columns (32 for CW = 4, 16 for CW = 8)
  constexpr int NT = WTN / 8;             // n8 tiles per warp
  extern __shared__ __align__(1024) unsigned char dsm_raw[];
  unsigned char* sm = dsm_raw + ((1024u - (smem_u32(dsm_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + DSmem::BAR);
  uint64_t* a_full = bars + 0;
  uint64_t* a_empty = bars + 1;
  uint64_t* full = bars + 2;    // [2]
  uint64_t* empty = bars + 4;   // [2]
  const uint32_t sA = smem_u32(sm + DSmem::A), sB = smem_u32(sm + DSmem::B);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  const int ntm = (g.M + TM - 1) / TM, ntn = (g.N + TN - 1) / TN;
  const int64_t T = (int64_t)ntm * ntn;
  longlong2* meta = reinterpret_cast<longlong2*>(sm + DSmem::META);
  if (threadIdx.x == 0) {
    mbar_init(a_full, 1);
    mbar_init(a_empty, CW);
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    mbar_init(&empty[0], CW);
    mbar_init(&empty[1], CW);
    fence_mbar_init();
  }
  __syncthreads();
#ifdef GJ_TIMELINE
  const bool tl = g.N > TK && g.rep_lo % 128 == 0;   // trailing updates only: per panel
  if (threadIdx.x == 0 && tl) {
    atomicMin(&g_tlg[0][g.rep_lo / 128], gtime());
    atomicMax(&g_tlg[2][g.rep_lo / 128], gtime());
  }
#endif

  if (warp == CW) {
    // ---------------------------------------------------------------- producer
    if (lane == 0) {
      // the range as one chunk; the next tile is known one chunk ahead, so the consumers can
      // prefetch its C
      auto wcum = [&](int64_t b) -> int64_t {
        return b <= g.late_from ? b * 1024 : (int64_t)g.late_from * 1024 + (b - g.late_from) * g.late_w;
      };
      const int64_t wtot = wcum(gridDim.x);
      int64_t static_next = T * wcum(blockIdx.x) / wtot;
      const int64_t static_end = T * wcum(blockIdx.x + 1) / wtot;
      auto claim = [&](int64_t& a, int64_t& b) {
        a = static_next;
        b = static_end;
        static_next = static_end;
        if (a >= b) a = b = T;
      };
      int64_t ca, cb, na_, nb_;
      claim(ca, cb);
      if (ca < T) claim(na_, nb_); else na_ = nb_ = T;
      int cur_m = -1, nA = 0, it = 0;
      while (ca < T) {
        for (int64_t t = ca; t < cb; ++t, ++it) {
          const int m = (int)(t / ntn), n = (int)(t % ntn);
          const int st = it & 1;
          const int64_t nxt = t + 1 < cb ? t + 1 : (na_ < T ? na_ : -1);
          if (it >= 2) mbar_wait(&empty[st], ((it >> 1) - 1) & 1);
          meta[st] = make_longlong2(t, nxt);
          mbar_expect_tx(&full[st], BLK_BYTES);
          const int rc = real_col(g, n * TN);
          for (int j = 0; j < NBOX; ++j)
            tma_load_2d(sm + DSmem::B + st * BLK_BYTES + j * BOX_BYTES, &mb, KB * j, rc, &full[st]);
          if (m != cur_m) {
            // the consumers read this tile's meta once its B lands, release the old A, then wait
            if (nA > 0) mbar_wait(a_empty, (nA - 1) & 1);
            mbar_expect_tx(a_full, ABLK_BYTES);
            for (int j = 0; j < NBOX; ++j)
              tma_load_2d(sm + DSmem::A + j * ABOX_BYTES, &ma, g.a_col0 + KB * j, m * TM, a_full);
            cur_m = m;
            ++nA;
          }
        }
        ca = na_;
        cb = nb_;
        if (ca < T) claim(na_, nb_); else na_ = nb_ = T;
      }
      // end of work: a stage whose meta says so
      const int st = it & 1;
      if (it >= 2) mbar_wait(&empty[st], ((it >> 1) - 1) & 1);
      meta[st] = make_longlong2(-1, -1);
      mbar_arrive(&full[st]);
    }
    return;   // the producer has no part in the PDL wait: stream order is kept by the consumers
  }

  // ------------------------------------------------------------------ consumers
  const int wm = warp / WN, wn = warp % WN;
  const int gq = lane >> 2, tq = lane & 3;
  // Fragment row of lane group gq: rho(gq) = 0, 2, 4, 6, 1, 3, 5, 7.  An 8-byte fragment load
  // is served per half-warp (gq 0..3, 4..7); under the 128-byte swizzle (chunk ^ row mod 8)
  // rows r and r ^ 1 use the same two chunks, so the four rows of a half-warp must differ in
  // (r >> 1): with rho the A loads (and the B loads, whose rows gather_rows_T_kernel stores in
  // the same order) are conflict-free — ncu: half the shared wavefronts were bank conflicts.
  // A row permutation of the warp tile is free for A and C (rows are independent).
  const int gr = ((gq & 3) << 1) | (gq >> 2);
  double acc[2][NT][4], cpre[2][NT][4];
  int kpre[2][2];   // pivstep of the prefetched rows (replace test applied when C is consumed)

  // C of tile t into `dst` (no dependence on pivstep: the loads issue at once and land while
  // this tile computes; rows outside the matrix / columns outside the update read 0)
  auto load_c = [&](double (&dst)[2][NT][4], int (&kp)[2][2], int64_t t) {
    const int m = (int)(t / ntn), n = (int)(t % ntn);
    const int rc0 = real_col(g, n * TN);
    const int nlim = g.N - n * TN;   // valid compact columns in this tile
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = m * TM + wm * 32 + mt * 16 + gr + 8 * h;
        const bool in = r < g.M;
        kp[mt][h] = in ? __ldg(g.pivstep + r) : g.rep_lo;   // rows outside: "replaced" (0)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int cl = wn * WTN + nt * 8 + 2 * tq;
          double2 v = make_double2(0.0, 0.0);
          if (in && cl < nlim) v = __ldcs(reinterpret_cast<const double2*>(g.C + (int64_t)r * g.ldc + rc0 + cl));
          dst[mt][nt][2 * h] = v.x;
          dst[mt][nt][2 * h + 1] = v.y;
        }
      }
  };

  int cur_m = -1, nA = 0;
  bool have_pre = false;
  for (int it = 0;; ++it) {
    const int st = it & 1;
    mbar_wait(&full[st], (it >> 1) & 1);
    const longlong2 mt_ = meta[st];
    const int64_t t = mt_.x, tn = mt_.y;
    if (t < 0) break;
    const int m = (int)(t / ntn), n = (int)(t % ntn);
    if (m != cur_m) {
      __syncwarp();
      if (cur_m >= 0 && lane == 0) mbar_arrive(a_empty);   // done with the old A block
      mbar_wait(a_full, nA & 1);
      cur_m = m;
      ++nA;
    }
    if (!have_pre) load_c(cpre, kpre, t);
    // accumulators start from C, or from 0 for the rows this panel pivoted (the update replaces)
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const bool keep = !(kpre[mt][h] >= g.rep_lo && kpre[mt][h] < g.rep_hi);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          acc[mt][nt][2 * h] = keep ? cpre[mt][nt][2 * h] : 0.0;
          acc[mt][nt][2 * h + 1] = keep ? cpre[mt][nt][2 * h + 1] : 0.0;
        }
      }
    have_pre = tn >= 0;
    if (have_pre) load_c(cpre, kpre, tn);   // in flight while this tile computes
    const uint32_t aB = sA, bB = sB + st * BLK_BYTES;
#pragma unroll 2
    for (int j = 0; j < NBOX; ++j) {
      const uint32_t ab = aB + j * ABOX_BYTES, bb = bB + j * BOX_BYTES;
      double af[2][8], bf[NT][4];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          af[mt][2 * i] = lds64(ab + boxoff(wm * 32 + mt * 16 + gr, tq + 4 * i));
          af[mt][2 * i + 1] = lds64(ab + boxoff(wm * 32 + mt * 16 + gr + 8, tq + 4 * i));
        }
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int i = 0; i < 4; ++i) bf[nt][i] = lds64(bb + boxoff(wn * WTN + nt * 8 + gr, tq + 4 * i));
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) dmma16816(acc[mt][nt], af[mt], bf[nt]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    // results straight from registers
    const int rc0 = real_col(g, n * TN);
    const int nlim = g.N - n * TN;
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = m * TM + wm * 32 + mt * 16 + gr + 8 * h;
        if (r >= g.M) continue;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int cl = wn * WTN + nt * 8 + 2 * tq;
          if (cl < nlim)
            __stcs(reinterpret_cast<double2*>(g.C + (int64_t)r * g.ldc + rc0 + cl),
                   make_double2(acc[mt][nt][2 * h], acc[mt][nt][2 * h + 1]));
        }
      }
  }
#ifdef GJ_TIMELINE
  if (lane == 0 && tl) atomicMax(&g_tlg[1][g.rep_lo / 128], gtime());
#endif
  // launched as a programmatic dependent of the panel kernel: complete only after it
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

template <int CW>
cudaError_t launch_cw(const DgemmArgs& g, const CUtensorMap& ma, const CUtensorMap& mb, int grid_sms, bool pdl,
                      cudaStream_t s) {
  static_assert(CW % WMW == 0 && (TN / (CW / WMW)) % 8 == 0, "warp grid");
  auto kern = dgemm_tma_kernel<CW>;
  static unsigned long long configured = 0;
  const unsigned long long dbit = device_bit();
  if (!(configured & dbit)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, DSmem::BYTES);
    if (e != cudaSuccess) return e;
    configured |= dbit;
  }
  const int64_t tiles = (int64_t)((g.M + TM - 1) / TM) * ((g.N + TN - 1) / TN);
  const int sms = grid_sms > 0 ? grid_sms : device_sm_count();
  const int grid = (int)(tiles < sms ? tiles : sms);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3((CW + 1) * 32, 1, 1);
  cfg.dynamicSmemBytes = DSmem::BYTES;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, g, ma, mb);
}

}  // namespace

bool dgemm_tma_supported(const DgemmArgs& g) {
  return g.K == TK && (g.ldx % 2) == 0 && (g.ldc % 2) == 0 && (g.a_col0 % 2) == 0 &&
         (reinterpret_cast<uintptr_t>(g.X) & 15) == 0 && (reinterpret_cast<uintptr_t>(g.RT) & 15) == 0 &&
         (reinterpret_cast<uintptr_t>(g.C) & 15) == 0 && (g.c_base % 2) == 0 && (g.skip_lo % 2) == 0 &&
         (g.skip_hi % 2) == 0;
}

cudaError_t launch_dgemm_tma(const DgemmArgs& g, int grid_sms, bool pdl, cudaStream_t s) {
  if (g.M <= 0 || g.N <= 0) return cudaSuccess;
  if (!dgemm_tma_supported(g)) return cudaErrorNotSupported;
  CUtensorMap ma, mb;
  if (!make_tma_map_2d(&ma, true, g.X, (uint64_t)g.x_cols, (uint64_t)g.x_rows, (uint64_t)g.ldx * 8, KB, TM, 128))
    return cudaErrorNotSupported;
  if (!make_tma_map_2d(&mb, true, g.RT, TK, (uint64_t)g.rt_rows, TK * 8, KB, 64, 128)) return cudaErrorNotSupported;
  // 16 consumer warps (32 x 8 warp tiles: four warps per scheduler) for matrices up to
  // ~12K rows, 8 (32 x 16) above: measured (tools/time_large_lib.py, bitwise-equal outputs)
  // C4 n = 8192 38.1 -> 37.5 ms with 16, but n = 32768 2.23 -> 2.28 s with the weighted ranges
  // (and n = 16384 alike), so the size decides
  return g.M <= GJ_DGEMM_CW16_MAX_M ? launch_cw<16>(g, ma, mb, grid_sms, pdl, s) : launch_cw<8>(g, ma, mb, grid_sms, pdl, s);
}

}  // namespace gj

#ifdef GJ_TIMELINE
extern "C" int gj_debug_timeline_gemm(unsigned long long* out, int reset) {   // out: [3][512]
  if (cudaMemcpyFromSymbol(out, gj::g_tlg, sizeof(gj::g_tlg)) != cudaSuccess) return -1;
  if (reset) {
    static unsigned long long z[3][512];
    for (int i = 0; i < 512; ++i) z[0][i] = ~0ull;
    cudaMemcpyToSymbol(gj::g_tlg, z, sizeof(z));
  }
  return 0;
}
#endif
