// K2b — batched Gauss–Jordan inversion for fp64 n = 64 on sm_100a (BASELINE configs[2],
// C3): one matrix per CTA of two warps.  Lane q of each warp holds rows q and q + 32
// ("two half rows per thread": every shared-memory read of an update feeds two rows);
// the 64 columns are split in eight blocks of BS = 8, warp w holding the blocks j with
// j % 2 == w.
//
// The elimination (§2, Eqs. (14)-(15), L61-L72; Obs. 2-3 L59-L60; listing
// L150-L177) is taken block by block, as K1b does (gj_batched.cu):
//   factor(b)  (the warp owning block b): BS pivot steps on the block's columns — per step
//              the max-|x_ik| pivot among the un-pivoted rows (ties to the smallest physical
//              position, reading G3; three redux.sync on the fp64 bit pattern), the pivot
//              row's block values by shuffle, the block's columns updated with the
//              deferred-normalisation multiplier x_ik / p (the pivot row's own compact
//              entry held as 1 - 1 = 0: W - S);
//   E_b        every other column: X[:, c] += (W_b - S_b) R_b[c], R_b = the block's pivot
//              rows before the update.  A column's update needs only
//              that column's R values, so each warp publishes and reads only its own.
// Cross-warp look-ahead: the only data crossing warps is W_b (64 x 8) and the block's
// pivot record.  The owner of b publishes them and goes on with E_b on its own columns;
// the other warp (the owner of b+1) applies E_b to its next block first, factors b+1 at
// once, and applies E_b to its remaining columns afterwards — so the two warps' panel
// chains and updates overlap.  Producer/consumer named barriers (bar.arrive / bar.sync)
// per W buffer parity; rows never move (logical swaps on positions, replayed by the
// non-owner from the record); the un-permutation (L179-L198) happens in the store.
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
constexpr int BSB = 8;          // block width
constexpr int HW = 32;          // columns per warp
constexpr int RWO = HW - BSB;   // a warp's columns outside its front block
constexpr int kThreadsB = 64;

struct SmemB {
  static constexpr int STAGE = NPB * NPB * 8;                 // 4 TMA boxes [64 rows][128 B]
  static constexpr int W = 2 * NPB * BSB * 8;                 // [parity][64 rows][BS] W - S
  static constexpr int BSM = 2 * HW * 2 * 4;                  // [parity][lane][slot] block step of a pivot row
  static constexpr int RO = 2 * BSB * HW * 8;                 // [warp][BS][32] each warp's pivot-row values
  static constexpr int REC = NPB * 16;                        // [step] (p, q)
  static constexpr int POS = NPB * 4;
  static constexpr int PERM = NPB * 4;
  static constexpr int EX = 64;
  static constexpr int TOTAL = STAGE + W + BSM + RO + REC + POS + PERM + EX + 16;
};

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
// named barriers over both warps: the producer arrives, the consumer waits
__device__ __forceinline__ void nb_arrive(int id) { asm volatile("bar.arrive %0, 64;" ::"r"(id) : "memory"); }
__device__ __forceinline__ void nb_sync(int id) { asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory"); }
constexpr int kFull = 1, kEmpty = 3;   // + parity

// One pivot step s (static) of factor(b) at global step k on registers x[.][0..BS).
__device__ __forceinline__ void panel_step64(const int s, const int k, double (&x)[2][HW], uint32_t (&kmask)[2],
                                             int (&pos)[2], int (&bs)[2], unsigned char* rec, int lane) {
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
  double z[BSB];
#pragma unroll
  for (int j = 0; j < BSB; ++j) z[j] = shfl_d(slot1 ? x[1][j] : x[0][j], src);
  const double p = z[s];
  const double rp = rcp64(p);
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const bool pv = pos[r] == q;
    const double nf = pv ? 0.0 : -(x[r][s] * rp);
#pragma unroll
    for (int j = 0; j < BSB; ++j)
      if (j != s) x[r][j] = fma(nf, z[j], x[r][j]);
    x[r][s] = nf;   // W - S
    kmask[r] = pv ? 0u : kmask[r];
    bs[r] = pv ? s : bs[r];
    pos[r] = (pos[r] == k) ? q : pos[r];
    pos[r] = pv ? k : pos[r];
  }
  if (lane == 0) rec_store(rec, k, p, q);
}

// Publish this warp's values of the block's pivot rows, registers [J0, J0 + N) -> R[s][0..N).
template <int J0, int N>
__device__ __forceinline__ void publish_rows(const double (&x)[2][HW], const int (&bs)[2], double* R) {
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    if (bs[r] >= 0) {
      double2* d = reinterpret_cast<double2*>(R + bs[r] * HW);
#pragma unroll
      for (int j = 0; j < N; j += 2) d[j / 2] = make_double2(x[r][J0 + j], x[r][J0 + j + 1]);
    }
  }
}

// E_b on registers [J0, J0 + N): x[r][c] += sum_s w[r][s] R[s][c - J0]; SHIFT writes the
// result BS registers to the left (the owner's rotation after its own panel).
template <int J0, int N, bool SHIFT>
__device__ __forceinline__ void apply_update(double (&x)[2][HW], const double (&w)[2][BSB], const double* R) {
#pragma unroll
  for (int s = 0; s < BSB; ++s) {
    const double2* rs = reinterpret_cast<const double2*>(R + s * HW);
#pragma unroll
    for (int j = 0; j < N; j += 2) {
      const double2 v = rs[j / 2];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        if (SHIFT && s + 1 == BSB) {
          x[r][J0 + j - BSB] = fma(w[r][s], v.x, x[r][J0 + j]);
          x[r][J0 + j + 1 - BSB] = fma(w[r][s], v.y, x[r][J0 + j + 1]);
        } else {
          x[r][J0 + j] = fma(w[r][s], v.x, x[r][J0 + j]);
          x[r][J0 + j + 1] = fma(w[r][s], v.y, x[r][J0 + j + 1]);
        }
      }
    }
  }
}

__device__ __forceinline__ void load_w(double (&w)[2][BSB], const double* W, int lane) {
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
}

struct MapsB {
  CUtensorMap a, x;
};

__global__ void __launch_bounds__(kThreadsB)
gj_batched64b_kernel(BatchedArgs a, const __grid_constant__ MapsB tm) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* stage = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  double* Wsm = reinterpret_cast<double*>(stage + SmemB::STAGE);
  int* bsm = reinterpret_cast<int*>(reinterpret_cast<unsigned char*>(Wsm) + SmemB::W);
  double* Rsm = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(bsm) + SmemB::BSM);
  unsigned char* rec = reinterpret_cast<unsigned char*>(Rsm) + SmemB::RO;
  int* posx = reinterpret_cast<int*>(rec + SmemB::REC);
  int* perm = posx + NPB;
  uint32_t* ex = reinterpret_cast<uint32_t*>(perm + NPB);
  uint64_t* bar = reinterpret_cast<uint64_t*>(ex + 16);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  double* Rw = Rsm + warp * BSB * HW;   // this warp's pivot-row values

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
    // warp w: blocks w, w+2, w+4, w+6 -> registers [0,8), [8,16), [16,24), [24,32)
    double x[2][HW];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int row = lane + 32 * r;
#pragma unroll
      for (int j = 0; j < HW; j += 2) {
        const int col = BSB * (2 * (j / BSB) + warp) + j % BSB;
        const double2 v = *reinterpret_cast<const double2*>(stage + st_addr(row, (uint32_t)col * 8u));
        x[r][j] = v.x;
        x[r][j + 1] = v.y;
      }
    }
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
    bool pending = false;   // E_{b-1} still to be applied to registers [BS, 32)
#pragma unroll 1
    for (int b = 0; b < NPB / BSB; ++b) {
      const int par = b & 1;
      const int k0 = BSB * b;
      double* W = Wsm + par * NPB * BSB;
      int* bsb = bsm + par * HW * 2;
      if ((b & 1) == warp) {
        // ---------------- owner of block b: its front block has every earlier update
        int bs[2] = {-1, -1};
#pragma unroll
        for (int s = 0; s < BSB; ++s) panel_step64(s, k0 + s, x, kmask, pos, bs, rec, lane);
        if (b >= 2) nb_sync(kEmpty + par);   // the other warp is done with W_{b-2}
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          double2* wd = reinterpret_cast<double2*>(W + (lane + 32 * r) * BSB);
#pragma unroll
          for (int j = 0; j < BSB; j += 2) wd[j / 2] = make_double2(x[r][j], x[r][j + 1]);
          bsb[lane * 2 + r] = bs[r];
        }
        nb_arrive(kFull + par);             // W_b, the block steps and the record are out
        if (pending) {
          // E_{b-1} on the columns outside the new panel (values R from this warp's copy)
          double w[2][BSB];
          load_w(w, Wsm + (par ^ 1) * NPB * BSB, lane);
          apply_update<BSB, RWO, false>(x, w, Rw + BSB);
          __syncwarp();
          if (b + 1 < NPB / BSB) nb_arrive(kEmpty + (par ^ 1));   // done with W_{b-1} (reused at b+1)
        }
        // E_b on this warp's other columns, rotating the panel to the end
        __syncwarp();
        publish_rows<BSB, RWO>(x, bs, Rw);
        __syncwarp();
        double w[2][BSB];
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int s = 0; s < BSB; ++s) w[r][s] = x[r][s];
        apply_update<BSB, RWO, true>(x, w, Rw);
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int s = 0; s < BSB; ++s) x[r][RWO + s] = w[r][s];
        pending = false;
      } else {
        // ---------------- the other warp: wait for W_b, replay the block's swaps, apply
        // E_b to the front block now (look-ahead) and to the rest after its next panel
        nb_sync(kFull + par);
        int bs[2];
#pragma unroll
        for (int r = 0; r < 2; ++r) bs[r] = bsb[lane * 2 + r];
#pragma unroll
        for (int s = 0; s < BSB; ++s) {
          int q;
          double pdd;
          rec_load(rec, k0 + s, pdd, q);
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            pos[r] = (pos[r] == k0 + s) ? q : pos[r];
            if (bs[r] == s) {
              pos[r] = k0 + s;
              kmask[r] = 0u;
            }
          }
        }
        publish_rows<0, HW>(x, bs, Rw);
        __syncwarp();
        double w[2][BSB];
        load_w(w, W, lane);
        apply_update<0, BSB, false>(x, w, Rw);
        pending = true;
        if (b + 1 == NPB / BSB) {   // no next panel: the rest now
          apply_update<BSB, RWO, false>(x, w, Rw + BSB);
          pending = false;
        }
      }
    }
    __syncthreads();
    // positions: warp 1 owns the last block, both are consistent now
    double myrp[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      double p_own;
      int q_own;
      rec_load(rec, pos[r], p_own, q_own);
      myrp[r] = rcp64(p_own);
      (void)q_own;
    }
    // ---- a6: det / ipiv / singular flag from the per-step record (warp 0) ----
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
        for (int j = 0; j < HW; ++j) {
          const int c = BSB * (2 * (j / BSB) + warp) + j % BSB;   // compact column of register j
          *reinterpret_cast<double*>(stage + st_addr(orow, (uint32_t)perm[c])) = myrp[r] * x[r][j];
        }
        // the row's own compact entry was held as W - 1: add the 1 back (owner of that column)
        if ((pos[r] / BSB) % 2 == warp) {
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
  static unsigned long long configured = 0;
  const unsigned long long dbit = device_bit();
  if (!(configured & dbit)) {
    cudaError_t e = cudaFuncSetAttribute(gj_batched64b_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured |= dbit;
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
