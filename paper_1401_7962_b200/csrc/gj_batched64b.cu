// K2b — batched Gauss–Jordan inversion for fp64 n = 64 on sm_100a (BASELINE configs[2],
// C3): one matrix per CTA of two warps, COLUMN-SPLIT: warp w holds columns [32w, 32w+32)
// of rows q and q + 32 in lane q (two half rows per thread), so every shared-memory
// read of the trailing update feeds two rows (the unsplit one-row-per-thread K2 has
// every thread read every pivot row whole, which bounds it by shared-memory delivery).
//
// The elimination (§2, Eqs. (14)-(15), L61-L72; Obs. 2-3 L59-L60; listing
// L150-L177) is taken in blocks of BS = 8 steps, as K1b does (gj_batched.cu):
//   panel phase (owner warp = the warp holding the block's columns): per step the
//     max-|x_ik| pivot among the un-pivoted rows (ties to the smallest physical position,
//     reading G3; three redux.sync on the fp64 bit pattern), the pivot row's 8 panel
//     values by shuffle, the panel columns updated with the deferred-normalisation
//     multiplier x_ik / p; the compact D entry of the pivot row is held as 1 - 1 = 0
//     (W - S);
//   block end: the owner publishes W - S (64 rows x 8) and its part of the block's pivot
//     rows; the other warp publishes its part; both apply X[:, J'] += (W - S) R.
// Rows never move (logical swaps on positions); the un-permutation (L179-L198) happens in
// the un-permuted store, as in K1/K2.  The owner warp rotates its registers by BS per
// block (four blocks per half: back to the identity); positions are handed from warp 0
// to warp 1 at the half boundary and back at the end.
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

constexpr int NPB = 64;         // matrix order
constexpr int BSB = 8;          // block (panel) width
constexpr int HW = 32;          // columns per warp
constexpr int RWO = HW - BSB;   // owner's trailing columns
constexpr int kThreadsB = 64;

struct SmemB {
  static constexpr int STAGE = NPB * NPB * 8;                 // 4 TMA boxes [64 rows][128 B]
  static constexpr int W = 2 * NPB * BSB * 8;                 // [2][64 rows][BS] W - S
  static constexpr int RO = 2 * BSB * RWO * 8;                // [2][BS][RWO] owner part of pivot rows
  static constexpr int RT = 2 * BSB * HW * 8;                 // [2][BS][32] other part
  static constexpr int REC = NPB * 16;                        // [step] (p, q)
  static constexpr int BSM = 2 * HW * 2 * 4;                  // [2][lane][slot] block step of pivot
  static constexpr int POS = NPB * 4;                         // [row] position hand-over
  static constexpr int PERM = NPB * 4;
  static constexpr int EX = 64;
  static constexpr int TOTAL = STAGE + W + RO + RT + REC + BSM + POS + PERM + EX + 16;
};

// (row, column byte) inside the TMA stage: 4 regions of [64 rows][128 B], 128-byte swizzle
__device__ __forceinline__ uint32_t st_addr(int row, uint32_t cb) {
  return (cb >> 7) * (NPB * 128) + (uint32_t)row * 128u + ((cb & 127u) ^ ((uint32_t)(row & 7) << 4));
}

__device__ __forceinline__ double shfl_d(double v, int src) {
  const long long b = __double_as_longlong(v);
  const int lo = __shfl_sync(0xffffffffu, (int)(b & 0xffffffffll), src);
  const int hi = __shfl_sync(0xffffffffu, (int)(b >> 32), src);
  return __longlong_as_double(((long long)hi << 32) | (unsigned int)lo);
}

__device__ __forceinline__ double rcp64(double p) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(p));
  double e = fma(-p, r, 1.0);
  r = fma(r, e, r);
  e = fma(-p, r, 1.0);
  return fma(r, e, r);
}

// One panel step of the owner warp: s static, k = global step.
__device__ __forceinline__ void panel_step64(const int s, const int k, double (&x)[2][HW], uint32_t (&kmask)[2],
                                             int (&pos)[2], int (&bs)[2], unsigned char* rec, int lane) {
  // a2: (hi, lo) words of |x| among the un-pivoted rows; ties -> smallest position
  uint32_t hi[2], lo[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(x[r][s]);
    hi[r] = (uint32_t)(b >> 32) & 0x7fffffffu & kmask[r];
    lo[r] = (uint32_t)b & kmask[r];
  }
  const uint32_t mh = __reduce_max_sync(0xffffffffu, max(hi[0], hi[1]));
  uint32_t lm = 0;
#pragma unroll
  for (int r = 0; r < 2; ++r)
    if (hi[r] == mh) lm = max(lm, lo[r]);
  const uint32_t ml = __reduce_max_sync(0xffffffffu, lm);
  uint32_t c = 0xffffffu;
#pragma unroll
  for (int r = 0; r < 2; ++r)
    if (hi[r] == mh && lo[r] == ml && kmask[r] != 0u) c = min(c, (uint32_t)pos[r] << 6 | (uint32_t)lane << 1 | (uint32_t)r);
  const uint32_t win = __reduce_min_sync(0xffffffffu, c);
  const int q = (int)(win >> 6);
  const int src = (int)((win >> 1) & 31u);
  const bool slot1 = (win & 1u) != 0u;
  bool pv[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) pv[r] = pos[r] == q;
  double z[BSB];
#pragma unroll
  for (int j = 0; j < BSB; ++j) z[j] = shfl_d(slot1 ? x[1][j] : x[0][j], src);
  const double p = z[s];
  const double rp = rcp64(p);
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const double nf = pv[r] ? 0.0 : -(x[r][s] * rp);
#pragma unroll
    for (int j = 0; j < BSB; ++j)
      if (j != s) x[r][j] = fma(nf, z[j], x[r][j]);
    x[r][s] = nf;   // W - S
    kmask[r] = pv[r] ? 0u : kmask[r];
    bs[r] = pv[r] ? s : bs[r];
    pos[r] = (pos[r] == k) ? q : pos[r];
    pos[r] = pv[r] ? k : pos[r];
  }
  if (lane == 0) rec_store(rec, k, p, q);
}

struct MapsB {
  CUtensorMap a, x;
};

__global__ void __launch_bounds__(kThreadsB)
gj_batched64b_kernel(BatchedArgs a, const __grid_constant__ MapsB tm) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* stage = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  double* Wsm = reinterpret_cast<double*>(stage + SmemB::STAGE);
  double* Ro = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(Wsm) + SmemB::W);
  double* Rt = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(Ro) + SmemB::RO);
  unsigned char* rec = reinterpret_cast<unsigned char*>(Rt) + SmemB::RT;
  int* bsm = reinterpret_cast<int*>(rec + SmemB::REC);
  int* posx = bsm + 2 * HW * 2;
  int* perm = posx + NPB;
  uint32_t* ex = reinterpret_cast<uint32_t*>(perm + NPB);
  uint64_t* bar = reinterpret_cast<uint64_t*>(ex + 16);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;

  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();

  int it = 0;
  for (int64_t m = blockIdx.x; m < a.batch; m += gridDim.x, ++it) {
    // ---- a1: load (TMA, 4 boxes of 64 rows x 16 doubles) ----
    if (tid == 0) {
      bulk_wait_read0();   // the previous matrix's store has read the stage
      mbar_expect_tx(bar, SmemB::STAGE);
#pragma unroll
      for (int rg = 0; rg < 4; ++rg) tma_load_2d(stage + rg * NPB * 128, &tm.a, rg * 16, (int)(m * NPB), bar);
    }
    while (!mbar_try_wait(bar, it & 1)) {
    }
    __syncwarp();
    double x[2][HW];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int row = lane + 32 * r;
#pragma unroll
      for (int j = 0; j < HW; j += 2) {
        const double2 v = *reinterpret_cast<const double2*>(stage + st_addr(row, (uint32_t)(HW * warp + j) * 8u));
        x[r][j] = v.x;
        x[r][j + 1] = v.y;
      }
    }
    // zero threshold tau = tol * max|a_ij| (Obs. 2, reading G1)
    {
      double rm = 0.0;
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int j = 0; j < HW; ++j) rm = fmax(rm, fabs(x[r][j]));
      const unsigned long long rb = (unsigned long long)__double_as_longlong(rm);
      const uint32_t mh = __reduce_max_sync(0xffffffffu, (uint32_t)(rb >> 32));
      const uint32_t ml = __reduce_max_sync(0xffffffffu, (uint32_t)(rb >> 32) == mh ? (uint32_t)rb : 0u);
      if (lane == 0) {
        ex[warp * 2] = mh;
        ex[warp * 2 + 1] = ml;
      }
    }
    __syncthreads();   // also: the stage has been fully read
    double tau;
    {
      const unsigned long long w0 = ((unsigned long long)ex[0] << 32) | ex[1];
      const unsigned long long w1 = ((unsigned long long)ex[2] << 32) | ex[3];
      tau = a.tol * __longlong_as_double((long long)(w0 > w1 ? w0 : w1));
    }

    uint32_t kmask[2] = {0xffffffffu, 0xffffffffu};
    int pos[2] = {lane, lane + 32};
    int blk = 0;
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
      if (h == 1) {
        // hand the positions over from warp 0 (owner of steps 0..31) to warp 1
        if (warp == 0) {
          posx[lane] = pos[0];
          posx[lane + 32] = pos[1];
        }
        __syncthreads();
        if (warp == 1) {
          pos[0] = posx[lane];
          pos[1] = posx[lane + 32];
          kmask[0] = pos[0] < 32 ? 0u : 0xffffffffu;
          kmask[1] = pos[1] < 32 ? 0u : 0xffffffffu;
        }
      }
#pragma unroll 1
      for (int bb = 0; bb < HW / BSB; ++bb, ++blk) {
        const int kb = HW * h + BSB * bb;
        const int buf = blk & 1;
        double* W = Wsm + buf * NPB * BSB;
        double* RO_ = Ro + buf * BSB * RWO;
        double* RT_ = Rt + buf * BSB * HW;
        int* bsb = bsm + buf * HW * 2;
        if (warp == h) {
          // ---- owner: panel phase on registers 0..BS ----
          int bs[2] = {-1, -1};
#pragma unroll
          for (int s = 0; s < BSB; ++s) panel_step64(s, kb + s, x, kmask, pos, bs, rec, lane);
          // publish W - S, the pivot rows' owner part (registers BS..32), block steps
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            double2* wd = reinterpret_cast<double2*>(W + (lane + 32 * r) * BSB);
#pragma unroll
            for (int j = 0; j < BSB; j += 2) wd[j / 2] = make_double2(x[r][j], x[r][j + 1]);
            if (bs[r] >= 0) {
              double2* rd = reinterpret_cast<double2*>(RO_ + bs[r] * RWO);
#pragma unroll
              for (int j = 0; j < RWO; j += 2) rd[j / 2] = make_double2(x[r][BSB + j], x[r][BSB + j + 1]);
            }
            bsb[lane * 2 + r] = bs[r];
          }
          __syncthreads();   // (1)
          __syncthreads();   // (2): the other warp's part of the pivot rows
          // trailing update of registers BS..32, written BS to the left; W - S appended
          double w[2][BSB];
#pragma unroll
          for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int s = 0; s < BSB; ++s) w[r][s] = x[r][s];
#pragma unroll
          for (int s = 0; s < BSB; ++s) {
            const double2* rs = reinterpret_cast<const double2*>(RO_ + s * RWO);
#pragma unroll
            for (int j = 0; j < RWO; j += 2) {
              const double2 v = rs[j / 2];
#pragma unroll
              for (int r = 0; r < 2; ++r) {
                if (s + 1 < BSB) {
                  x[r][BSB + j] = fma(w[r][s], v.x, x[r][BSB + j]);
                  x[r][BSB + j + 1] = fma(w[r][s], v.y, x[r][BSB + j + 1]);
                } else {
                  x[r][j] = fma(w[r][s], v.x, x[r][BSB + j]);
                  x[r][j + 1] = fma(w[r][s], v.y, x[r][BSB + j + 1]);
                }
              }
            }
          }
#pragma unroll
          for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int s = 0; s < BSB; ++s) x[r][RWO + s] = w[r][s];
        } else {
          __syncthreads();   // (1): W - S, the owner part, block steps
          int bs[2];
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            bs[r] = bsb[lane * 2 + r];
            if (bs[r] >= 0) {
              double2* rd = reinterpret_cast<double2*>(RT_ + bs[r] * HW);
#pragma unroll
              for (int j = 0; j < HW; j += 2) rd[j / 2] = make_double2(x[r][j], x[r][j + 1]);
            }
          }
          __syncthreads();   // (2)
          double w[2][BSB];
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            const double2* wd = reinterpret_cast<const double2*>(W + (lane + 32 * r) * BSB);
#pragma unroll
            for (int j = 0; j < BSB; j += 2) {
              const double2 v = wd[j / 2];
              w[r][j] = v.x;
              w[r][j + 1] = v.y;
            }
          }
#pragma unroll
          for (int s = 0; s < BSB; ++s) {
            const double2* rs = reinterpret_cast<const double2*>(RT_ + s * HW);
#pragma unroll
            for (int j = 0; j < HW; j += 2) {
              const double2 v = rs[j / 2];
#pragma unroll
              for (int r = 0; r < 2; ++r) {
                x[r][j] = fma(w[r][s], v.x, x[r][j]);
                x[r][j + 1] = fma(w[r][s], v.y, x[r][j + 1]);
              }
            }
          }
        }
      }
    }
    // positions back to both warps (warp 1 holds the final ones: pos = the row's pivot step)
    if (warp == 1) {
      posx[lane] = pos[0];
      posx[lane + 32] = pos[1];
    }
    __syncthreads();
    pos[0] = posx[lane];
    pos[1] = posx[lane + 32];

    // ---- a6: det / ipiv / singular flag from the per-step record (warp 0) ----
    double myrp[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      double p_own;
      int q_own;
      rec_load(rec, pos[r], p_own, q_own);
      myrp[r] = rcp64(p_own);
      (void)q_own;
    }
    if (warp == 0) {
      unsigned fb[2];
      int nsw = 0, nng = 0;
      double lgl = 0.0;
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int k = lane + 32 * r;
        double p_k;
        int q_k;
        rec_load(rec, k, p_k, q_k);
        fb[r] = __ballot_sync(0xffffffffu, fabs(p_k) <= tau);
        nsw += __popc(__ballot_sync(0xffffffffu, q_k != k));
        nng += __popc(__ballot_sync(0xffffffffu, p_k < 0.0));
        lgl += log_abs(p_k);
        if (a.ipiv) a.ipiv[m * NPB + k] = q_k + 1;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) lgl += __shfl_xor_sync(0xffffffffu, lgl, o);
      if (lane == 0) {
        const int info = fb[0] ? __ffs(fb[0]) : (fb[1] ? 32 + __ffs(fb[1]) : 0);
        const int sgn = ((nsw ^ nng) & 1) ? -1 : 1;
        if (a.info) a.info[m] = info;
        if (a.logabsdet) a.logabsdet[m] = info ? -INFINITY : lgl;
        if (a.sign) a.sign[m] = info ? 0 : (int8_t)sgn;
        if (a.det) static_cast<double*>(a.det)[m] = info ? 0.0 : (double)(sgn * exp(lgl));
      }
    }
    // ---- a7 + a8: un-permuted store: Ainv[pos(row)][perm[c]] = X[row][c] / p(row) ----
    if (a.Ainv != nullptr) {
      if (warp == 0) {
        perm[pos[0]] = lane * 8;          // output column (bytes) of compact column pos[row]
        perm[pos[1]] = (lane + 32) * 8;
      }
      __syncthreads();
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int orow = pos[r];
#pragma unroll
        for (int j = 0; j < HW; j += 2) {
          const int2 cb = *reinterpret_cast<const int2*>(perm + HW * warp + j);
          *reinterpret_cast<double*>(stage + st_addr(orow, (uint32_t)cb.x)) = myrp[r] * x[r][j];
          *reinterpret_cast<double*>(stage + st_addr(orow, (uint32_t)cb.y)) = myrp[r] * x[r][j + 1];
        }
        // the row's own compact entry was held as W - 1: add the 1 back (owner of that column)
        if (pos[r] / HW == warp) {
          double* own = reinterpret_cast<double*>(stage + st_addr(orow, (uint32_t)((lane + 32 * r) * 8)));
          *own = *own + myrp[r];
        }
      }
      fence_async_smem();
      __syncthreads();
      if (tid == 0) {
#pragma unroll
        for (int rg = 0; rg < 4; ++rg) tma_store_2d(&tm.x, rg * 16, (int)(m * NPB), stage + rg * NPB * 128);
        bulk_commit();
      }
    }
    __syncthreads();
  }
  if (tid == 0) bulk_wait0();
}

}  // namespace

// fp64 n = 64 with 16-byte aligned buffers; returns cudaErrorNotSupported otherwise.
cudaError_t launch_batched64b(const BatchedArgs& a, cudaStream_t s) {
  if (a.n != NPB) return cudaErrorNotSupported;
  const bool aligned = (reinterpret_cast<uintptr_t>(a.A) % 16 == 0) &&
                       (a.Ainv == nullptr || reinterpret_cast<uintptr_t>(a.Ainv) % 16 == 0);
  const uint64_t rows = (uint64_t)a.batch * NPB;
  if (!aligned || rows >= (1ull << 31)) return cudaErrorNotSupported;
  MapsB maps;
  if (!make_tma_map_2d(&maps.a, true, a.A, NPB, rows, NPB * 8, 16, NPB, 128)) return cudaErrorNotSupported;
  if (a.Ainv != nullptr) {
    if (!make_tma_map_2d(&maps.x, true, a.Ainv, NPB, rows, NPB * 8, 16, NPB, 128)) return cudaErrorNotSupported;
  } else {
    maps.x = maps.a;
  }
  const size_t smem = (size_t)SmemB::TOTAL + 1024;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(gj_batched64b_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gj_batched64b_kernel, kThreadsB, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const int64_t cap = (int64_t)device_sm_count() * per_sm;
  const int grid = (int)(a.batch < cap ? a.batch : cap);
  gj_batched64b_kernel<<<grid, kThreadsB, smem, s>>>(a, maps);
  return cudaGetLastError();
}

}  // namespace gj
