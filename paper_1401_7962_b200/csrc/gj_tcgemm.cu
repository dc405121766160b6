// K4t — the large-n trailing update for fp32 on the 5th-generation tensor cores
// (tcgen05.mma kind::tf32, accumulator in TMEM): SURVEY.md §8f f1, the aggregated form of
// Eqs. (14)-(15) for a panel of K = 128 columns:
//     C[i][c] = (replace(i) ? 0 : C[i][c]) + sum_s W[i][s] R[s][c]
// with fp32 accuracy from three TF32 products (3xTF32): W = Wh + Wl, R = Rh + Rl with
// Wh, Rh exactly representable in TF32, and W R ~ Wh Rh + Wh Rl + Wl Rh (the dropped
// Wl Rl and the TF32 rounding of the low parts are ~2^-21 of |W||R|).
// The operands arrive split and K-major (Ah/Al: M x 128, Bh/Bl: N x 128; B is R
// transposed) — gj_large.cu's split / transposed-gather kernels write them per panel.
// One CTA per SM, warp-specialised: warp 4 issues the TMA loads (the row block's Ah/Al,
// 128 KB, resident for a whole work unit; B tiles of 128 x 32 through two 32 KB stages),
// one thread of warp 5 issues 48 tcgen05.mma per tile (4 k-blocks x 4 k-steps x 3
// products) into one of two 128-lane x 32-column fp32 TMEM accumulators and signals
// mbarriers with tcgen05.commit, and warps 0-3 read the accumulator back with tcgen05.ld
// (warp w <-> TMEM lanes 32w..32w+31 = tile rows) and update C while the next tile's
// MMAs run.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

#include "gj_internal.h"
#include "gj_ptx.cuh"

namespace gj {
namespace tc {

using namespace ptx;

constexpr int TM = 128, TN = 32, TK = 128, KB = 32, NKB = TK / KB;
constexpr int A_BLK = TM * KB * 4;                  // 16 KB: one k-block of Ah (or Al)
constexpr int B_BLK = TN * KB * 4;                  // 4 KB
constexpr int B_STAGE = 2 * NKB * B_BLK;            // Bh + Bl of one column tile: 32 KB
constexpr int SMEM = 2 * NKB * A_BLK + 2 * B_STAGE + 1024;
constexpr int kEpiWarps = 8;                        // warps 0-7: epilogue (lane quarter w % 4, column half w / 4)
constexpr int kPW = kEpiWarps, kMW = kEpiWarps + 1; // producer warp, MMA warp
constexpr int kThreads = (kEpiWarps + 2) * 32;
constexpr int EC = TN / 2;                          // columns per epilogue thread

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
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
__device__ __forceinline__ void arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

struct Maps {
  CUtensorMap ah, al, bh, bl;
};

// Work unit = (row block, contiguous range of column tiles): A of the row block stays in
// shared memory for the whole unit; B tiles stream through two stages; the accumulator is
// double-buffered in TMEM so the epilogue of tile t overlaps the MMAs of tile t+1.
__global__ void __launch_bounds__(kThreads, 1) tc_update_kernel(const __grid_constant__ Maps mp, TcUpdateArgs g) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* sAh = base;
  unsigned char* sAl = sAh + NKB * A_BLK;
  unsigned char* sB = sAl + NKB * A_BLK;   // [stage][h/l][kb][TN x KB]
  __shared__ uint64_t a_full, a_empty, b_full[2], b_empty[2], t_full[2], t_empty[2];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == kMW) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "n"(2 * TN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == kPW * 32) {
    mbar_init(&a_full, 1);
    mbar_init(&a_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&b_full[i], 1);
      mbar_init(&b_empty[i], 1);
      mbar_init(&t_full[i], 1);
      mbar_init(&t_empty[i], kEpiWarps);
    }
    fence_mbar_init();
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;

  const int ntn = (g.N + TN - 1) / TN, ntm = (g.M + TM - 1) / TM;
  const int shift = g.skip_hi - g.skip_lo;
  // units: each row block's column tiles split into `cpr` contiguous parts
  const int cpr = gridDim.x >= ntm ? (int)gridDim.x / ntm : 1;
  const int nunits = ntm * cpr;
  auto unit_range = [&](int u, int& rb, int& t0, int& t1) {
    rb = u / cpr;
    const int part = u % cpr;
    t0 = (int)((int64_t)ntn * part / cpr);
    t1 = (int)((int64_t)ntn * (part + 1) / cpr);
  };
  auto real_col = [&](int ct) {
    const int nc0 = ct * TN;
    return nc0 + (nc0 >= g.skip_lo ? shift : 0);
  };

  if (warp == kPW) {
    // ---------------- TMA producer
    if (lane == 0) {
      int ua = 0, tb = 0;
      for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++ua) {
        int rb, t0, t1;
        unit_range(u, rb, t0, t1);
        wait(&a_empty, (ua & 1) ^ 1);
        mbar_expect_tx(&a_full, 2 * NKB * A_BLK);
        for (int kb = 0; kb < NKB; ++kb) {
          tma_load_2d(sAh + kb * A_BLK, &mp.ah, kb * KB, rb * TM, &a_full);
          tma_load_2d(sAl + kb * A_BLK, &mp.al, kb * KB, rb * TM, &a_full);
        }
        for (int t = t0; t < t1; ++t, ++tb) {
          const int st = tb & 1;
          wait(&b_empty[st], ((tb >> 1) & 1) ^ 1);
          unsigned char* sb = sB + st * B_STAGE;
          mbar_expect_tx(&b_full[st], B_STAGE);
          const int n0 = real_col(t);
          for (int kb = 0; kb < NKB; ++kb) {
            tma_load_2d(sb + kb * B_BLK, &mp.bh, kb * KB, n0, &b_full[st]);
            tma_load_2d(sb + (NKB + kb) * B_BLK, &mp.bl, kb * KB, n0, &b_full[st]);
          }
        }
      }
    }
  } else if (warp == kMW) {
    // ---------------- MMA issuer (one thread)
    if (lane == 0) {
      int ua = 0, tb = 0;
      for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++ua) {
        int rb, t0, t1;
        unit_range(u, rb, t0, t1);
        wait(&a_full, ua & 1);
        for (int t = t0; t < t1; ++t, ++tb) {
          const int st = tb & 1, ac = tb & 1;
          wait(&b_full[st], (tb >> 1) & 1);
          wait(&t_empty[ac], ((tb >> 1) & 1) ^ 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t d = tmem + (uint32_t)(ac * TN);
          const uint32_t sb = smem_u32(sB + st * B_STAGE);
          uint32_t acc = 0;
#pragma unroll
          for (int kb = 0; kb < NKB; ++kb) {
#pragma unroll
            for (int kk = 0; kk < KB / 8; ++kk) {
              const uint64_t ah = desc_k_sw128(smem_u32(sAh + kb * A_BLK) + kk * 32);
              const uint64_t al = desc_k_sw128(smem_u32(sAl + kb * A_BLK) + kk * 32);
              const uint64_t bh = desc_k_sw128(sb + kb * B_BLK + kk * 32);
              const uint64_t bl = desc_k_sw128(sb + (NKB + kb) * B_BLK + kk * 32);
              mma_tf32(d, al, bh, acc);   // the small products first
              acc = 1;
              mma_tf32(d, ah, bl, 1);
              mma_tf32(d, ah, bh, 1);
            }
          }
          mma_commit(&b_empty[st]);   // the B stage may be refilled
          mma_commit(&t_full[ac]);    // the accumulator is ready
        }
        mma_commit(&a_empty);         // A of this unit no longer read
      }
    }
  } else {
    // ---------------- epilogue: warp w <-> TMEM lanes (rows) 32(w%4).., columns 16(w/4)..
    const int quarter = warp & 3, half = warp >> 2;
    int tb = 0;
    for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
      int rb, t0, t1;
      unit_range(u, rb, t0, t1);
      const int r = rb * TM + quarter * 32 + lane;
      bool keep = r < g.M;
      if (keep) {
        const int ps = g.pivstep[r];
        keep = !(ps >= g.rep_lo && ps < g.rep_hi);
      }
      for (int t = t0; t < t1; ++t, ++tb) {
        const int ac = tb & 1;
        const int n0 = real_col(t) + half * EC;
        const int nlim = real_col(t) + (g.N - t * TN);
        float* crow = g.C + (int64_t)r * g.ldc + n0;
        const bool full = r < g.M && n0 + EC <= nlim;
        // C of this tile while the MMAs run
        float4 cv[EC / 4];
#pragma unroll
        for (int j = 0; j < EC / 4; ++j)
          cv[j] = (full && keep) ? *reinterpret_cast<const float4*>(crow + 4 * j) : make_float4(0.f, 0.f, 0.f, 0.f);
        wait(&t_full[ac], (tb >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        uint32_t v[EC];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(ac * TN + half * EC)));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) arrive(&t_empty[ac]);   // the TMEM buffer may be overwritten
        if (full) {
#pragma unroll
          for (int j = 0; j < EC / 4; ++j) {
            float4 o = cv[j];
            o.x += __uint_as_float(v[4 * j]);
            o.y += __uint_as_float(v[4 * j + 1]);
            o.z += __uint_as_float(v[4 * j + 2]);
            o.w += __uint_as_float(v[4 * j + 3]);
            *reinterpret_cast<float4*>(crow + 4 * j) = o;
          }
        } else if (r < g.M) {
          for (int q = 0; q < EC; ++q)
            if (n0 + q < nlim) crow[q] = (keep ? crow[q] : 0.f) + __uint_as_float(v[q]);
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == kMW) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(2 * TN));
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
  static unsigned long long configured = 0;
  const unsigned long long dbit = device_bit();
  if (!(configured & dbit)) {
    cudaError_t e = cudaFuncSetAttribute(tc_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return e;
    configured |= dbit;
  }
  const int ntm = (g.M + TM - 1) / TM, ntn = (g.N + TN - 1) / TN;
  const int sms = grid_sms > 0 ? grid_sms : device_sm_count();
  // units of (row block, column range): as many as SMs when there are fewer row blocks
  const int cpr = ntm >= sms ? 1 : (sms / ntm < ntn ? sms / ntm : ntn);
  const int units = ntm * cpr;
  const int grid = units < sms ? units : sms;
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
