// K4t — the large-n trailing update for fp32 on the 5th-generation tensor cores
// (tcgen05.mma kind::tf32, accumulator in TMEM): SURVEY.md §8f f1, the aggregated form of
// Eqs. (14)-(15) for a panel of K = 128 columns:
//     C[i][c] = (replace(i) ? 0 : C[i][c]) + sum_s W[i][s] R[s][c]
// with fp32 accuracy from three TF32 products (3xTF32): W = Wh + Wl, R = Rh + Rl with
// Wh, Rh exactly representable in TF32, and W R ~ Wh Rh + Wh Rl + Wl Rh (the dropped
// Wl Rl and the TF32 rounding of the low parts are ~2^-21 of |W||R|).
// The operands arrive split and K-major (Ah/Al: M x 128, Bh/Bl: N x 128; B is R
// transposed) — gj_large.cu's split / transposed-gather kernels write them per panel.
// One CTA per SM (persistent over 128 x 64 tiles): TMA loads the whole K = 128 of both
// operands (128-byte swizzle, 192 KB), one elected thread issues 48 tcgen05.mma
// (4 k-blocks x 4 k-steps x 3 products) into a 128-lane x 64-column fp32 TMEM
// accumulator, tcgen05.commit signals an mbarrier, and four warps read the accumulator
// back with tcgen05.ld (warp w <-> TMEM lanes 32w..32w+31 = tile rows) and update C.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

#include "gj_internal.h"
#include "gj_ptx.cuh"

namespace gj {
namespace tc {

using namespace ptx;

constexpr int TM = 128, TN = 64, TK = 128, KB = 32;
constexpr int A_BLK = TM * KB * 4;                  // 16 KB: one k-block of Ah (or Al)
constexpr int B_BLK = TN * KB * 4;                  // 8 KB
constexpr int SMEM = 2 * (TK / KB) * (A_BLK + B_BLK) + 1024 + 64;
constexpr int kThreads = 128;

// Shared-memory matrix descriptor: K-major, 128-byte swizzle, 8-row groups 1024 B apart.
__device__ __forceinline__ uint64_t desc_k_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3fff);   // start address (16-byte units)
  d |= (uint64_t)1 << 16;                   // leading byte offset (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;         // stride byte offset
  d |= (uint64_t)1 << 46;                   // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                   // SWIZZLE_128B
  return d;
}
// Instruction descriptor: D f32, A/B tf32, both K-major, N >> 3, M >> 4.
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TN >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t tmem, uint64_t ad, uint64_t bd, uint32_t acc) {
  asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p; }"
               ::"r"(tmem), "l"(ad), "l"(bd), "r"(kIdesc), "r"(acc));
}

struct Maps {
  CUtensorMap ah, al, bh, bl;
};

__global__ void __launch_bounds__(kThreads, 1) tc_update_kernel(const __grid_constant__ Maps mp, TcUpdateArgs g) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* sAh = base;
  unsigned char* sAl = sAh + (TK / KB) * A_BLK;
  unsigned char* sBh = sAl + (TK / KB) * A_BLK;
  unsigned char* sBl = sBh + (TK / KB) * B_BLK;
  __shared__ uint64_t bar_tma, bar_mma;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "n"(TN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    mbar_init(&bar_tma, 1);
    mbar_init(&bar_mma, 1);
    fence_mbar_init();
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;

  const int ntn = (g.N + TN - 1) / TN, ntm = (g.M + TM - 1) / TM;
  const int shift = g.skip_hi - g.skip_lo;
  int it = 0;
  for (int tile = blockIdx.x; tile < ntn * ntm; tile += gridDim.x, ++it) {
    const int m0 = (tile % ntm) * TM;
    const int nc0 = (tile / ntm) * TN;                    // compact column of the tile
    const int n0 = nc0 + (nc0 >= g.skip_lo ? shift : 0);  // real column
    const int nlim = n0 + (g.N - nc0);
    if (tid == 0) {
      mbar_expect_tx(&bar_tma, 2 * (TK / KB) * (A_BLK + B_BLK));
#pragma unroll
      for (int kb = 0; kb < TK / KB; ++kb) {
        tma_load_2d(sAh + kb * A_BLK, &mp.ah, kb * KB, m0, &bar_tma);
        tma_load_2d(sAl + kb * A_BLK, &mp.al, kb * KB, m0, &bar_tma);
        tma_load_2d(sBh + kb * B_BLK, &mp.bh, kb * KB, n0, &bar_tma);
        tma_load_2d(sBl + kb * B_BLK, &mp.bl, kb * KB, n0, &bar_tma);
      }
    }
    while (!mbar_try_wait(&bar_tma, it & 1)) {
    }
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      uint32_t acc = 0;
#pragma unroll
      for (int kb = 0; kb < TK / KB; ++kb) {
#pragma unroll
        for (int kk = 0; kk < KB / 8; ++kk) {
          const uint64_t ah = desc_k_sw128(smem_u32(sAh + kb * A_BLK) + kk * 32);
          const uint64_t al = desc_k_sw128(smem_u32(sAl + kb * A_BLK) + kk * 32);
          const uint64_t bh = desc_k_sw128(smem_u32(sBh + kb * B_BLK) + kk * 32);
          const uint64_t bl = desc_k_sw128(smem_u32(sBl + kb * B_BLK) + kk * 32);
          mma_tf32(tmem, al, bh, acc);   // small products first
          acc = 1;
          mma_tf32(tmem, ah, bl, 1);
          mma_tf32(tmem, ah, bh, 1);
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar_mma))
                   : "memory");
    }
    while (!mbar_try_wait(&bar_mma, it & 1)) {
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
    // epilogue: warp w reads tile rows 32w..32w+31 (TMEM lanes), 64 columns
    const int r = m0 + warp * 32 + lane;
    bool keep = r < g.M;
    if (keep) {
      const int ps = g.pivstep[r];
      keep = !(ps >= g.rep_lo && ps < g.rep_hi);
    }
#pragma unroll
    for (int c = 0; c < TN; c += 16) {
      uint32_t v[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
            "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      if (r < g.M) {
        float* crow = g.C + (int64_t)r * g.ldc + n0 + c;
#pragma unroll
        for (int j = 0; j < 16; j += 4) {
          if (n0 + c + j + 3 < nlim) {
            float4 o = keep ? *reinterpret_cast<const float4*>(crow + j) : make_float4(0.f, 0.f, 0.f, 0.f);
            o.x += __uint_as_float(v[j]);
            o.y += __uint_as_float(v[j + 1]);
            o.z += __uint_as_float(v[j + 2]);
            o.w += __uint_as_float(v[j + 3]);
            *reinterpret_cast<float4*>(crow + j) = o;
          } else {
            for (int u = 0; u < 4; ++u)
              if (n0 + c + j + u < nlim) crow[j + u] = (keep ? crow[j + u] : 0.f) + __uint_as_float(v[j + u]);
          }
        }
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();   // TMEM read and smem consumed before the next tile's loads / MMAs
    asm volatile("tcgen05.fence::after_thread_sync;");
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TN));
  // launched as a programmatic dependent of the panel kernel: complete only after it
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

}  // namespace tc

cudaError_t launch_tc_update(const TcUpdateArgs& g, int grid_sms, bool pdl, cudaStream_t s) {
  using namespace tc;
  if (g.M <= 0 || g.N <= 0) return cudaSuccess;
  Maps mp;
  const uint64_t K = 128;
  if (!make_tma_map_2d(&mp.ah, false, g.Ah, K, (uint64_t)g.M, K * 4, KB, TM, 128) ||
      !make_tma_map_2d(&mp.al, false, g.Al, K, (uint64_t)g.M, K * 4, KB, TM, 128) ||
      !make_tma_map_2d(&mp.bh, false, g.Bh, K, (uint64_t)g.Nrows, K * 4, KB, TN, 128) ||
      !make_tma_map_2d(&mp.bl, false, g.Bl, K, (uint64_t)g.Nrows, K * 4, KB, TN, 128))
    return cudaErrorInvalidValue;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(tc_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int tiles = ((g.N + TN - 1) / TN) * ((g.M + TM - 1) / TM);
  const int sms = grid_sms > 0 ? grid_sms : device_sm_count();
  const int grid = tiles < sms ? tiles : sms;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, tc_update_kernel, mp, g);
}

}  // namespace gj
