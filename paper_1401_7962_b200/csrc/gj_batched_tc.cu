// K1t — batched Gauss–Jordan for fp32 n = 32 with the blocked trailing update on the
// 5th-generation tensor cores (tcgen05.mma kind::tf32, 3xTF32, accumulator in TMEM).
//
// The elimination is K1b's (gj_batched.cu): blocks of BS = 4 pivot steps; inside a block
// each step updates only the block's panel columns (the pivot search of Obs. 3, PAPER.md
// L60, ties to the smallest physical position — reading G3 —, logical swaps, deferred
// normalisation, compact storage, the pivot row's own entry held as W - S = 0); after the
// block every row takes the block's BS rank-1 updates at once (the aggregation of
// Eqs. (14)-(15), L61-L72):   x_i[j] += sum_s (W - S)_is R_s[j]   for j outside the panel.
// Here that update is ONE matrix product per block for the 4 matrices of a CTA:
//     D (128 x 32) += A (128 x 16) * B (16 x 32)
// D = the four 32 x 32 matrices stacked (TMEM lane = matrix row, column = matrix column;
// the matrices live in TMEM for the whole elimination), A = blockdiag(W_0 - S_0, ...,
// W_3 - S_3) (row 32m + i holds matrix m's panel values in K columns 4m..4m+3, zeros
// elsewhere; A lives in TMEM too, next to D, so a CTA needs only ~29 KB of shared memory
// and seven CTAs share an SM), B = the four matrices' block pivot rows (K row 4m + s =
// matrix m's step-s pivot row, its panel columns zeroed; shared memory, K-major).  fp32 accuracy from three TF32 products
// (Al Bh + Ah Bl + Ah Bh; x = hi + lo, both rounded to TF32).
// Status: correct (tests/test_gpu_k1t.py) but not faster than K1b on C2 (4.3 vs 3.5 ms): the
// tensor cores remove the trailing FMAs, which were a quarter of K1b's instructions; the
// per-step pivot chain and the per-block TMEM / barrier / MMA round trip remain, with one
// matrix per warp instead of K1b's two.  Opt-in with GJ_K1_TC=1.  One warp per matrix, lane =
// row: the panel columns come out of TMEM with tcgen05.ld, the pivot search is a
// full-warp redux, and the panel goes back with tcgen05.st before the MMA.
// A singular or non-finite item must not leak into its neighbours through the shared
// product (0 * Inf = NaN): the B operand is sanitised and a zero pivot uses 1/p = 0.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "gj_internal.h"
#include "gj_ptx.cuh"
#include "gj_rowops.cuh"

namespace gj {
namespace {

using namespace ptx;
using namespace rowops;

constexpr int TW = 4;                 // warps per CTA
#ifndef GJ_TC_MH
#define GJ_TC_MH 1
#endif
constexpr int MH = GJ_TC_MH;          // matrices per warp (lane = one row of each)
constexpr int MPC = TW * MH;          // matrices per CTA task
#ifndef GJ_TC_BS
#define GJ_TC_BS 4
#endif
constexpr int TBS = GJ_TC_BS;         // block size (pivot steps per MMA)
constexpr int TK = MPC * TBS;         // K of the block product (16 or 32)
static_assert(TK <= 32, "one 128-byte K row");
constexpr int TN = 32 * MH;           // N of the block product (a warp's matrices side by side)
constexpr int STAGE_B = MPC * 32 * 128;   // one task: MPC matrices, rows of 128 B (TMA, 128-byte swizzle)
constexpr int BOP_B = TN * 128;           // B operand: TN rows (N) x 128 B (K-major)
// TMEM columns: D [0, TN) (matrix (w, h) in lanes 32w.., columns 32h..); A hi [TN, TN + TK),
// A lo [TN + TK, TN + 2 TK)
constexpr int TM_NEED = TN + 2 * TK;
constexpr int TM_COLS = TM_NEED <= 32 ? 32 : TM_NEED <= 64 ? 64 : TM_NEED <= 128 ? 128 : 256;
struct TcSmem {
  static constexpr int STAGE = 0;
  static constexpr int BH = STAGE + STAGE_B;
  static constexpr int BL = BH + BOP_B;
  static constexpr int RS = BL + BOP_B;                  // [MPC][TBS][32] fp32 pivot rows (transpose staging)
  static constexpr int PERM = RS;                        // [MPC][32] int — aliases RS (blocks done)
  static constexpr int REC = RS + MPC * TBS * 32 * 4;    // [MPC][32] (p, q)
  static constexpr int BAR = REC + MPC * 32 * 8;         // load, mma mbarriers; TMEM base
  static constexpr int BYTES = BAR + 32;
};

__device__ __forceinline__ uint32_t swz128(int row, int colf) {   // byte offset of (row, fp32 col)
  return (uint32_t)(row * 128 + ((((colf * 4) >> 4) ^ (row & 7)) << 4) + ((colf * 4) & 15));
}
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3fff);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// x = hi + lo, both rounded to TF32 (10 explicit mantissa bits; the tensor core ignores the
// low 13 bits of an fp32 operand, so rounding them ourselves halves the representation
// error): |x - hi - lo| <= 2^-22 |x|
__device__ __forceinline__ float round_tf32(float x) { return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u); }
__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
  hi = round_tf32(x);
  lo = round_tf32(x - hi);
}

__device__ __forceinline__ void tm_ld4(uint32_t addr, float (&v)[4]) {
  uint32_t r0, r1, r2, r3;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  v[0] = __uint_as_float(r0); v[1] = __uint_as_float(r1); v[2] = __uint_as_float(r2); v[3] = __uint_as_float(r3);
}
__device__ __forceinline__ void tm_st4(uint32_t addr, const float (&v)[4]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};"
               ::"r"(addr), "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
                 "r"(__float_as_uint(v[3])) : "memory");
}
__device__ __forceinline__ void tm_ld8(uint32_t addr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = __uint_as_float(r[j]);
}
__device__ __forceinline__ void tm_st8(uint32_t addr, const float (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
               ::"r"(addr), "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
                 "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
                 "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])) : "memory");
}
template <int N>
__device__ __forceinline__ void tm_ldp(uint32_t addr, float (&v)[N]) {
  if constexpr (N == 4) tm_ld4(addr, v); else tm_ld8(addr, v);
}
template <int N>
__device__ __forceinline__ void tm_stp(uint32_t addr, const float (&v)[N]) {
  if constexpr (N == 4) tm_st4(addr, v); else tm_st8(addr, v);
}
__device__ __forceinline__ void tm_ld32(uint32_t addr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
}
__device__ __forceinline__ void tm_st32(uint32_t addr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
      "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
      ::"r"(addr), "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
        "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])),
        "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])),
        "r"(__float_as_uint(v[11])), "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])),
        "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15])), "r"(__float_as_uint(v[16])),
        "r"(__float_as_uint(v[17])), "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])),
        "r"(__float_as_uint(v[20])), "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])),
        "r"(__float_as_uint(v[23])), "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])),
        "r"(__float_as_uint(v[26])), "r"(__float_as_uint(v[27])), "r"(__float_as_uint(v[28])),
        "r"(__float_as_uint(v[29])), "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31]))
      : "memory");
}

// One panel step S (static) at global step k for each of the lane's MH matrices (full-warp
// reductions per matrix; the MH chains are independent and interleave).
template <int S>
__device__ __forceinline__ void tc_panel_step(const int k, float (&P)[MH][TBS], uint32_t (&kmask)[MH],
                                              int (&pos)[MH], int (&bs)[MH], unsigned char* rec, int mm0, int lane) {
  uint32_t key[MH], m[MH], win[MH];
#pragma unroll
  for (int h = 0; h < MH; ++h) {
    key[h] = __float_as_uint(P[h][S]) & 0x7fffffffu & kmask[h];
    m[h] = __reduce_max_sync(0xffffffffu, key[h]);
  }
#pragma unroll
  for (int h = 0; h < MH; ++h) {
    const uint32_t c = (key[h] == m[h] && kmask[h] != 0u) ? ((uint32_t)pos[h] << 5 | (uint32_t)lane) : 0xffffffffu;
    win[h] = __reduce_min_sync(0xffffffffu, c);
  }
#pragma unroll
  for (int h = 0; h < MH; ++h) {
    const int q = (int)(win[h] >> 5), src = (int)(win[h] & 31u);
    const bool pv = lane == src;
    float z[TBS];
#pragma unroll
    for (int j = 0; j < TBS; ++j) z[j] = __shfl_sync(0xffffffffu, P[h][j], src);
    const float p = z[S];
    // 1/p (0 for a zero pivot: a singular item stays finite, so it cannot poison the
    // neighbours' products); Eq. (15)'s multiplier with the deferred pivot-row scale
    const float rp = p != 0.0f ? rcp(p) : 0.0f;
    const float nf = pv ? 0.0f : -(P[h][S] * rp);
#pragma unroll
    for (int j = 0; j < TBS; ++j)
      if (j != S) P[h][j] = fmaf(nf, z[j], P[h][j]);
    P[h][S] = nf;   // compact D entry; 0 on the pivot row (W - S: its 1 is held as 0)
    kmask[h] = pv ? 0u : kmask[h];
    bs[h] = pv ? S : bs[h];
    pos[h] = (pos[h] == k) ? q : pos[h];   // a3: the listing's swap of positions k and q (L156-L162)
    pos[h] = pv ? k : pos[h];
    if (lane == 0) rec_store(rec + (mm0 + h) * 32 * 8, k, p, q);
  }
}
template <int S>
__device__ __forceinline__ void tc_panel_steps(const int kb, float (&P)[MH][TBS], uint32_t (&kmask)[MH],
                                               int (&pos)[MH], int (&bs)[MH], unsigned char* rec, int mm0, int lane) {
  if constexpr (S < TBS) {
    tc_panel_step<S>(kb + S, P, kmask, pos, bs, rec, mm0, lane);
    tc_panel_steps<S + 1>(kb, P, kmask, pos, bs, rec, mm0, lane);
  }
}

// D f32, A/B tf32, A from TMEM, B K-major: N = TN, M = 128
constexpr uint32_t kIdescT = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);

__global__ void __launch_bounds__(TW * 32) gj_tc32_kernel(BatchedArgs a, const __grid_constant__ CUtensorMap tma_a,
                                                          const __grid_constant__ CUtensorMap tma_x) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sb = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* stage = sb + TcSmem::STAGE;
  unsigned char* bH = sb + TcSmem::BH;
  unsigned char* bL = sb + TcSmem::BL;
  float* rs = reinterpret_cast<float*>(sb + TcSmem::RS);
  unsigned char* rec = sb + TcSmem::REC;
  int* perm = reinterpret_cast<int*>(sb + TcSmem::PERM);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sb + TcSmem::BAR);   // [0] load, [1] mma
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sb + TcSmem::BAR + 16);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int mm0 = warp * MH;   // the warp's first matrix within the task

  for (int e = tid; e < 2 * BOP_B / 16; e += TW * 32) reinterpret_cast<uint4*>(bH)[e] = make_uint4(0u, 0u, 0u, 0u);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "n"(TM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;
  const uint32_t tm_row = tmem + ((uint32_t)(warp * 32) << 16);   // this warp's lanes, column 0
  // A operand in TMEM (block-diagonal): zero once; a row's nonzero K columns are rewritten
  // every block
  {
    float zz[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int c = 0; c < 2 * TK; c += 4) tm_st4(tm_row + (uint32_t)(TN + c), zz);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }

  const int64_t ntasks = (a.batch + MPC - 1) / MPC;
  int it = 0, mph = 0;
  if (tid == 0 && (int64_t)blockIdx.x < ntasks) {
    mbar_expect_tx(&bars[0], STAGE_B);
    tma_load_2d(stage, &tma_a, 0, (int)(blockIdx.x * MPC * 32), &bars[0]);
  }
  for (int64_t task = blockIdx.x; task < ntasks; task += gridDim.x, ++it) {
    const int64_t nxt = task + gridDim.x;
    if (tid == 0 && nxt < ntasks) bulk_prefetch_l2(static_cast<const float*>(a.A) + nxt * MPC * 32 * 32, STAGE_B);
    while (!mbar_try_wait(&bars[0], it & 1)) {
    }
    // ---- a1: the lane's rows (one per matrix) into TMEM
    uint32_t kmask[MH];
    int pos[MH];
    float tau[MH];
    bool item_ok[MH];
#pragma unroll
    for (int h = 0; h < MH; ++h) {
      const int srow = (mm0 + h) * 32 + lane;
      item_ok[h] = task * MPC + mm0 + h < a.batch;
      float x[32];
#pragma unroll
      for (int j = 0; j < 32; j += 4) {
        const float4 v = *reinterpret_cast<const float4*>(stage + swz128(srow, j));
        x[j] = v.x; x[j + 1] = v.y; x[j + 2] = v.z; x[j + 3] = v.w;
      }
      if (!item_ok[h]) {   // padding matrices: the identity (finite, harmless in the shared products)
#pragma unroll
        for (int j = 0; j < 32; ++j) x[j] = lane == j ? 1.0f : 0.0f;
      }
      float rowmax = 0.0f;
#pragma unroll
      for (int j = 0; j < 32; ++j) rowmax = fmaxf(rowmax, fabsf(x[j]));
      const double smax = (double)__uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(rowmax)));
      tau[h] = round_down_to(a.tol * smax, 0.0f);
      tm_st32(tm_row + (uint32_t)(32 * h), x);
      kmask[h] = 0x7fffffffu;
      pos[h] = lane;
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");

#pragma unroll 1
    for (int kb = 0; kb < 32; kb += TBS) {
      // ---- the block's panel columns out of TMEM; BS pivot steps on them
      float P[MH][TBS];
#pragma unroll
      for (int h = 0; h < MH; ++h) tm_ldp<TBS>(tm_row + (uint32_t)(32 * h + kb), P[h]);
      int bs[MH];
#pragma unroll
      for (int h = 0; h < MH; ++h) bs[h] = -1;
      tc_panel_steps<0>(kb, P, kmask, pos, bs, rec, mm0, lane);
      // the block's pivot rows as they were at the block's start -> transpose staging
#pragma unroll
      for (int h = 0; h < MH; ++h) {
        float y[32];
        tm_ld32(tm_row + (uint32_t)(32 * h), y);
        if (bs[h] >= 0) {
          float* dst = rs + ((mm0 + h) * TBS + bs[h]) * 32;
#pragma unroll
          for (int j = 0; j < 32; j += 4) *reinterpret_cast<float4*>(dst + j) = make_float4(y[j], y[j + 1], y[j + 2], y[j + 3]);
        }
        tm_stp<TBS>(tm_row + (uint32_t)(32 * h + kb), P[h]);   // the panel's compact values (W - S)
        // A operand (TMEM): row = this lane, K columns TBS (mm0 + h) .. (hi / lo)
        float hh[TBS], ll[TBS];
#pragma unroll
        for (int s2 = 0; s2 < TBS; ++s2) split_tf32(P[h][s2], hh[s2], ll[s2]);
        tm_stp<TBS>(tm_row + (uint32_t)(TN + TBS * (mm0 + h)), hh);
        tm_stp<TBS>(tm_row + (uint32_t)(TN + TK + TBS * (mm0 + h)), ll);
      }
      __syncwarp();
      // B operand (K-major): row 32 h + j (N) holds, in K columns TBS (mm0 + h) + s, column j
      // of step s's pivot row of matrix (warp, h); lane j gathers its column
#pragma unroll
      for (int h = 0; h < MH; ++h) {
        float hh[TBS], ll[TBS];
#pragma unroll
        for (int s2 = 0; s2 < TBS; ++s2) {
          float v = rs[((mm0 + h) * TBS + s2) * 32 + lane];
          // the panel's own columns take no product term; and no Inf / NaN may enter the
          // shared product (0 * Inf would reach the other matrices)
          v = (lane >= kb && lane < kb + TBS) || !(fabsf(v) <= 3.0e38f) ? 0.0f : v;
          split_tf32(v, hh[s2], ll[s2]);
        }
#pragma unroll
        for (int c = 0; c < TBS; c += 4) {
          *reinterpret_cast<float4*>(bH + swz128(32 * h + lane, TBS * (mm0 + h) + c)) = make_float4(hh[c], hh[c + 1], hh[c + 2], hh[c + 3]);
          *reinterpret_cast<float4*>(bL + swz128(32 * h + lane, TBS * (mm0 + h) + c)) = make_float4(ll[c], ll[c + 1], ll[c + 2], ll[c + 3]);
        }
      }
      fence_async_smem();
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncthreads();
      if (tid == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
        for (int kk = 0; kk < TK / 8; ++kk) {
          const uint32_t ah = tmem + (uint32_t)(TN + 8 * kk), al = tmem + (uint32_t)(TN + TK + 8 * kk);
          const uint64_t bh = desc_sw128(smem_u32(bH) + kk * 32), bl = desc_sw128(smem_u32(bL) + kk * 32);
          asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;" ::"r"(tmem), "r"(al), "l"(bh), "r"(kIdescT));
          asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;" ::"r"(tmem), "r"(ah), "l"(bl), "r"(kIdescT));
          asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;" ::"r"(tmem), "r"(ah), "l"(bh), "r"(kIdescT));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bars[1]))
                     : "memory");
      }
      while (!mbar_try_wait(&bars[1], mph & 1)) {
      }
      ++mph;
      asm volatile("tcgen05.fence::after_thread_sync;");
    }

    // ---- a6 + a7 + a8 per matrix
#pragma unroll
    for (int h = 0; h < MH; ++h) {
      const int mm = mm0 + h;
      const int64_t item = task * MPC + mm;
      unsigned char* rec_m = rec + mm * 32 * 8;
      int* perm_m = perm + mm * 32;
      float xr[32];
      tm_ld32(tm_row + (uint32_t)(32 * h), xr);
      float p_own, p_k;
      int q_own, q_k;
      rec_load(rec_m, pos[h], p_own, q_own);
      rec_load(rec_m, lane, p_k, q_k);
      (void)q_own;
      const float myrp = rcp(p_own);
      const unsigned fb = __ballot_sync(0xffffffffu, fabsf(p_k) <= tau[h]);
      const int info = fb ? __ffs(fb) : 0;
      const int nswap = __popc(__ballot_sync(0xffffffffu, q_k != lane));
      const int nneg = __popc(__ballot_sync(0xffffffffu, p_k < 0.0f));
      double lg = log_abs(p_k);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) lg += __shfl_xor_sync(0xffffffffu, lg, o);
      const int sgn = ((nswap ^ nneg) & 1) ? -1 : 1;
      if (item_ok[h]) {
        if (a.ipiv) a.ipiv[item * 32 + lane] = q_k + 1;
        if (lane == 0) {
          if (a.info) a.info[item] = info;
          if (a.logabsdet) a.logabsdet[item] = info ? -INFINITY : lg;
          if (a.sign) a.sign[item] = info ? 0 : (int8_t)sgn;
          if (a.det) static_cast<float*>(a.det)[item] = info ? 0.0f : (float)(sgn * exp(lg));
        }
      }
      // A^-1[k][perm[k']] = X[perm[k]][k'] / p through the stage (un-permutation, L179-L198)
      if (a.Ainv != nullptr) {
        perm_m[pos[h]] = lane;   // perm[k] = the row pivoted at step k = output column of compact column k
        __syncwarp();
        const int orow = mm * 32 + pos[h];
#pragma unroll
        for (int kp = 0; kp < 32; ++kp) *reinterpret_cast<float*>(stage + swz128(orow, perm_m[kp])) = myrp * xr[kp];
        float* own = reinterpret_cast<float*>(stage + swz128(orow, lane));
        *own = *own + myrp;   // the row's own compact entry was held as W - 1: add the 1 back
      }
    }
    if (a.Ainv != nullptr) fence_async_smem();
    __syncthreads();   // every warp's rows are in the stage
    if (tid == 0) {
      if (a.Ainv != nullptr) {
        tma_store_2d(&tma_x, 0, (int)(task * MPC * 32), stage);
        bulk_commit();
        bulk_wait_read0();   // the store has read the stage
      }
      if (nxt < ntasks) {
        mbar_expect_tx(&bars[0], STAGE_B);
        tma_load_2d(stage, &tma_a, 0, (int)(nxt * MPC * 32), &bars[0]);
      }
    }
  }
  if (tid == 0) bulk_wait0();
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TM_COLS));
}

}  // namespace

cudaError_t launch_tc32(const BatchedArgs& a, cudaStream_t s) {
  if (a.n != 32 || a.batch <= 0) return cudaErrorInvalidValue;
  if ((reinterpret_cast<uintptr_t>(a.A) & 15) || (a.Ainv && (reinterpret_cast<uintptr_t>(a.Ainv) & 15)))
    return cudaErrorNotSupported;
  if (a.batch * 32 >= (int64_t(1) << 31)) return cudaErrorNotSupported;
  CUtensorMap ta, tx;
  const uint64_t rows = (uint64_t)a.batch * 32;
  if (!make_tma_map_2d(&ta, false, a.A, 32, rows, 128, 32, MPC * 32, 128)) return cudaErrorNotSupported;
  if (a.Ainv != nullptr) {
    if (!make_tma_map_2d(&tx, false, a.Ainv, 32, rows, 128, 32, MPC * 32, 128)) return cudaErrorNotSupported;
  } else {
    tx = ta;
  }
  const int smem = TcSmem::BYTES + 1024;
  static unsigned long long configured = 0;
  const unsigned long long dbit = device_bit();
  if (!(configured & dbit)) {
    cudaError_t e = cudaFuncSetAttribute(gj_tc32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    // all of the unified L1 as shared memory: several 62 KB CTAs per SM (without a
    // preference the occupancy calculation settles for one)
    e = cudaFuncSetAttribute(gj_tc32_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    configured |= dbit;
  }
  // resident CTAs per SM from the shared memory they need (the occupancy calculator answers
  // 1 for a kernel that allocates tensor memory; each CTA here takes 32 of the 512 columns)
  int smem_sm = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaError_t e = cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  if (e != cudaSuccess) return e;
  int per_sm = smem_sm / (smem + 1024);
  if (per_sm > 512 / TM_COLS) per_sm = 512 / TM_COLS;   // tensor-memory columns
  if (per_sm < 1) per_sm = 1;
  if (getenv("GJ_TC_DEBUG")) fprintf(stderr, "tc32: smem %d per_sm %d\n", smem, per_sm);
  const int64_t ntasks = (a.batch + MPC - 1) / MPC;
  const int64_t cap = (int64_t)device_sm_count() * per_sm;
  const int grid = (int)(ntasks < cap ? ntasks : cap);
  gj_tc32_kernel<<<grid, TW * 32, smem, s>>>(a, ta, tx);
  return cudaGetLastError();
}

}  // namespace gj
