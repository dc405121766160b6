// Large-n blocked Gauss–Jordan (gj_invert for n > 64) on sm_100a — the aggregated form
// of the per-step rank-1 updates of Eqs. (14)-(15):
//
//   for each panel P of b = 128 columns:
//     for each leaf L of W columns inside P (W = 32, 16, 8, 4 for n <= 8192 / 16384 / 32768 / 65536):
//       K3  leaf factorisation: W pivot steps (a2-a5) over ALL n rows but only the W leaf
//           columns, by one thread-block cluster of 16 CTAs x 512 threads (every thread
//           holds its rows' W values in registers; per step a warp redux argmax, a CTA
//           winner among the warp winners, and one cp.async.bulk DSMEM copy of the CTA
//           winner into every CTA of the cluster, completing on that CTA's mbarrier — no
//           cluster barrier per step);
//       the rest of P's columns right of L:  X[:,T] += (W_L - S_L) R_L  (inside K3)
//     K4  trailing update of all columns outside P:  X[:,~P] += (W_P - S_P) R_P
//   K5  un-permutation: Ainv[k][j] = X[perm[k]][step(j)]       (listing L179-L198)
//   K6  log|det|, sign, singular flag, ipiv from the per-step record (Eq. (13), Obs. 2)
//
// Here W_L is the leaf's compact D columns (normalised), R_L = X[pivot rows of L, T] taken
// before the update, and S_L selects the pivot rows: for a pivot row the update REPLACES
// the old values (X_s <- (W R)_s), for every other row it adds.  Derivation: the block's
// row operation is E = I + (S - C) A11^-1 S^T and its compact D columns are
// W = E S = S + (S - C) A11^-1, so E v = v + (W - S) v[S].
//
// K4 is an FP64 tensor-core GEMM: mma.sync.m16n8k16.f64 (SASS DMMA; tcgen05 has no f64
// kind on sm_100a), 128x64 CTA tiles, 4 warps of 64x32, cp.async double-buffered K slabs,
// persistent grid, launched with programmatic stream serialisation so that the next
// panel's K3 runs beside it (look-ahead).  Pivoting is logical (rows never move); ties go to the smallest
// physical position of the listing's swapped array (reading G3), so ipiv equals
// LAPACK getrf's.  n is padded to a multiple of 32 with an identity block.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "gj_internal.h"
#include "gj_ptx.cuh"

namespace gj {
#ifdef GJ_TIMELINE
__device__ unsigned long long g_tl[2][512];
#endif
namespace large {

using namespace ptx;

// ============================================================================ small kernels
__global__ void init_perm_kernel(int n, int* pos, int* pivstep) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    pos[i] = i;
    pivstep[i] = -1;
  }
}

// X (npad x npad, ld npad) = blockdiag(A, I) and max |a_ij| (the bit pattern of a non-negative
// double, atomicMax on u64 is monotone; fmax: a NaN never wins) in one pass over A: one row of
// X per CTA iteration (coalesced)
__global__ void copy_pad_absmax_kernel(const double* __restrict__ A, int64_t lda, int n, double* __restrict__ X,
                                       int npad, unsigned long long* out) {
  double m = 0.0;
  for (int i = blockIdx.x; i < npad; i += gridDim.x) {
    const double* a = A + (int64_t)i * lda;
    double* x = X + (int64_t)i * npad;
    if (i < n) {
#pragma unroll 4
      for (int j = threadIdx.x; j < n; j += blockDim.x) {
        const double v = __ldcs(a + j);
        m = fmax(m, fabs(v));
        x[j] = v;
      }
      for (int j = n + threadIdx.x; j < npad; j += blockDim.x) x[j] = 0.0;
    } else {
      for (int j = threadIdx.x; j < npad; j += blockDim.x) x[j] = i == j ? 1.0 : 0.0;
    }
  }
  unsigned long long b = (unsigned long long)__double_as_longlong(m);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long ob = __shfl_xor_sync(0xffffffffu, b, o);
    b = ob > b ? ob : b;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(out, b);
}

// max |a_ij| as the bit pattern of a non-negative double (atomicMax on u64 is monotone)
__global__ void absmax_kernel(const double* __restrict__ A, int64_t lda, int n, unsigned long long* out) {
  double m = 0.0;
  const int64_t tot = (int64_t)n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / n), j = (int)(e - (int64_t)i * n);
    m = fmax(m, fabs(A[(int64_t)i * lda + j]));
  }
  unsigned long long b = (unsigned long long)__double_as_longlong(m);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long ob = __shfl_xor_sync(0xffffffffu, b, o);
    b = ob > b ? ob : b;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(out, b);
}

// R[s][c] = X[rows[s]][c] for s < w, c in [c_lo, c_hi) (R has leading dimension npad;
// c_lo, c_hi even)
__global__ void gather_rows_kernel(const double* __restrict__ X, int64_t ld, const int* __restrict__ rows, int w,
                                   double* __restrict__ R, int c_lo, int c_hi) {
  const int s = blockIdx.y;
  if (s >= w) return;
  const double2* src = reinterpret_cast<const double2*>(X + (int64_t)rows[s] * ld + c_lo);
  double2* dst = reinterpret_cast<double2*>(R + (int64_t)s * ld + c_lo);
  const int m = (c_hi - c_lo) / 2;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) dst[j] = src[j];
}

// RT[rt(c)][s] = X[rows[s]][c] for s < 128, c < ncols (the pivot rows transposed, K-major, for
// K4b's B operand), with column c of each aligned group of 8 stored at position
// rt(c) = (c & ~7) | rho(c & 7), rho = 0, 2, 4, 6, 1, 3, 5, 7: K4b's lane group g reads
// position rho(g) of its 8-row group, which keeps its fragment loads conflict-free
// (gj_dgemm.cu); 32 x 32 tiles through shared memory, grid (ceil(ncols / 32), 4), block (32, 8)
__global__ void gather_rows_T_kernel(const double* __restrict__ X, int64_t ld, const int* __restrict__ rows, int ncols,
                                     double* __restrict__ RT) {
  __shared__ double tile[32][33];
  const int c0 = blockIdx.x * 32, s0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int c = c0 + threadIdx.x;
    tile[i][threadIdx.x] = c < ncols ? X[(int64_t)rows[s0 + i] * ld + c] : 0.0;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int c = c0 + i;
    const int rc = (c & ~7) | (((c & 3) << 1) | ((c >> 2) & 1));
    if (c < ncols) RT[(int64_t)rc * 128 + s0 + threadIdx.x] = tile[threadIdx.x][i];
  }
}

// Ainv[k][j] = X[perm[k]][pivstep[j]]  (k, j < n); perm[k] = row pivoted at step k
__global__ void unpermute_kernel(const double* __restrict__ X, int npad, const int* __restrict__ rec_row,
                                 const int* __restrict__ pivstep, int n, double* __restrict__ Y, int64_t ldy) {
  for (int k = blockIdx.y; k < n; k += gridDim.y) {   // gridDim.y <= 65535 < GJ_LARGE_MAX_N
    const double* src = X + (int64_t)rec_row[k] * npad;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
      Y[(int64_t)k * ldy + j] = src[pivstep[j]];
  }
}

// unpermute_kernel with the source row staged in shared memory (npad doubles): the row is read
// once, coalesced, and the column gather runs out of shared memory
constexpr int kUnpermSmemMaxN = 26624;   // 208 KB
__global__ void __launch_bounds__(512) unpermute_smem_kernel(const double* __restrict__ X, int npad,
                                                             const int* __restrict__ rec_row,
                                                             const int* __restrict__ pivstep, int n,
                                                             double* __restrict__ Y, int64_t ldy) {
  extern __shared__ double srow[];
  for (int k = blockIdx.x; k < n; k += gridDim.x) {
    const double2* src = reinterpret_cast<const double2*>(X + (int64_t)rec_row[k] * npad);
    for (int j = threadIdx.x; j < npad / 2; j += blockDim.x) reinterpret_cast<double2*>(srow)[j] = __ldcs(src + j);
    __syncthreads();
    double* y = Y + (int64_t)k * ldy;
    for (int j = threadIdx.x; j < n; j += blockDim.x) __stcs(y + j, srow[__ldg(pivstep + j)]);
    __syncthreads();
  }
}

// log|det|, sign, singular flag and ipiv from the per-step record (Eq. (13), Obs. 2, G4)
__global__ void finalize_kernel(int n, const double* __restrict__ rec_p, const int* __restrict__ rec_q, double tol,
                                const unsigned long long* smax_bits, int32_t* ipiv, double* logabsdet, int8_t* sign,
                                double* det, int32_t* info) {
  __shared__ double s_lg[32];
  __shared__ int s_first[32], s_par[32];
  const double tau = tol * __longlong_as_double((long long)*smax_bits);
  double lg = 0.0;
  int first = 0x7fffffff, par = 0;
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const double p = rec_p[k];
    const int q = rec_q[k];
    if (ipiv) ipiv[k] = q + 1;
    lg += log(fabs(p));
    par ^= (q != k) ^ (p < 0.0);
    if (fabs(p) <= tau && k < first) first = k;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lg += __shfl_xor_sync(0xffffffffu, lg, o);
    first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
    par ^= __shfl_xor_sync(0xffffffffu, par, o);
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { s_lg[w] = lg; s_first[w] = first; s_par[w] = par; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double L = 0.0;
    int F = 0x7fffffff, Pp = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) { L += s_lg[i]; F = min(F, s_first[i]); Pp ^= s_par[i]; }
    const int inf = F == 0x7fffffff ? 0 : F + 1;
    if (info) *info = inf;
    if (logabsdet) *logabsdet = inf ? -INFINITY : L;
    if (sign) *sign = inf ? 0 : (Pp ? -1 : 1);
    if (det) *det = inf ? 0.0 : (Pp ? -exp(L) : exp(L));
  }
}

// ============================================================================ K3: leaf
// Cluster helpers
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_size() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t map_remote(uint32_t laddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(laddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_remote_v4(uint32_t raddr, uint4 v) {
  asm volatile("st.shared::cluster.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(raddr), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

struct LeafArgs {
  void* X;           // npad rows of T, leading dimension ld (all columns, or one rank's local columns)
  int64_t ld;        // row stride of X (elements)
  int npad;          // padded order (rows)
  int c0;            // first column of the panel in X
  int k0;            // global step of the panel's first column
  int pw;            // panel width (a multiple of the leaf width W)
  int* pos;          // [npad] physical position of each row
  int* pivstep;      // [npad] step at which the row was pivot, -1 if not yet
  double* rec_p;     // [npad] pivot value per step
  int* rec_q;        // [npad] pivot's physical position per step
  int* rec_row;      // [npad] pivot row per step
  void* Wout;        // if non-null: the factored panel (T), npad x pw (ld pw), written at the end
};

constexpr int kLeafThreads = 512;

// Candidate key: |p| as (hi, lo) words, position, row.
struct Cand {
  uint32_t hi, lo, pos, row;
};
__device__ __forceinline__ bool better(const Cand& a, const Cand& b) {   // a strictly preferred to b
  if (a.hi != b.hi) return a.hi > b.hi;
  if (a.lo != b.lo) return a.lo > b.lo;
  return a.pos < b.pos;
}

__device__ __forceinline__ void st_async_v4(uint32_t raddr, uint4 v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(raddr),
               "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_all(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// Index of the preferred candidate among the lanes with `ok` (all lanes get it): larger
// |p| (high word, then low word), ties to the smallest position.  Fast path: a unique
// high-word maximum decides without the other two reductions.
__device__ __forceinline__ int warp_pick(const Cand& c, bool ok) {
  const bool h = ok && c.pos != 0xffffffffu;
  const uint32_t H = __reduce_max_sync(0xffffffffu, h ? c.hi : 0u);
  const unsigned bh = __ballot_sync(0xffffffffu, h && c.hi == H);
  if (__popc(bh) == 1) return __ffs(bh) - 1;
  if (bh == 0) return 0;   // no candidate anywhere
  const uint32_t Lo = __reduce_max_sync(0xffffffffu, (h && c.hi == H) ? c.lo : 0u);
  const uint32_t P = __reduce_min_sync(0xffffffffu, (h && c.hi == H && c.lo == Lo) ? c.pos : 0xffffffffu);
  const unsigned bp = __ballot_sync(0xffffffffu, h && c.pos == P);
  return __ffs(bp) - 1;
}
// Bulk copy shared::cta -> shared::cluster, completing on the destination's mbarrier.
__device__ __forceinline__ void bulk_s2c(uint32_t dst, uint32_t src, uint32_t bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "r"(src), "r"(bytes), "r"(mbar)
               : "memory");
}
// 1/p: MUFU approximation + two Newton steps (exact for powers of two).
__device__ __forceinline__ double rcp_f64(double p) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(p));
  double e = fma(-p, r, 1.0);
  r = fma(r, e, r);
  e = fma(-p, r, 1.0);
  return fma(r, e, r);
}

__device__ __forceinline__ float rcp_t(float p) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(p));
  return fmaf(r, fmaf(-p, r, 1.0f), r);
}
__device__ __forceinline__ double rcp_t(double p) { return rcp_f64(p); }
// the candidate key of |v|: (hi, lo) words of the IEEE bit pattern (monotone for |v|)
__device__ __forceinline__ void abs_key(double v, uint32_t& hi, uint32_t& lo) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(v) & 0x7fffffffffffffffull;
  hi = (uint32_t)(u >> 32);
  lo = (uint32_t)u;
}
__device__ __forceinline__ void abs_key(float v, uint32_t& hi, uint32_t& lo) {
  hi = __float_as_uint(v) & 0x7fffffffu;
  lo = 0u;
}
// two consecutive elements as one vector access
template <typename T> struct Vec2;
template <> struct Vec2<double> { using type = double2; };
template <> struct Vec2<float> { using type = float2; };
template <typename T>
__device__ __forceinline__ void ld2(const T* p, T& a, T& b) {
  const typename Vec2<T>::type v = *reinterpret_cast<const typename Vec2<T>::type*>(p);
  a = v.x;
  b = v.y;
}
template <typename T>
__device__ __forceinline__ void st2(T* p, T a, T b) {
  typename Vec2<T>::type v;
  v.x = a;
  v.y = b;
  *reinterpret_cast<typename Vec2<T>::type*>(p) = v;
}

// Rotated leaf update (pivot column in register PC; the second step of a pair shifts the
// registers two to the left and appends the two new D columns, as in K1).
template <typename T, int W, int PC, bool SECOND>
__device__ __forceinline__ void leaf_update(T (&x)[W], const T* y, T nf, T dcol) {
  if constexpr (!SECOND) {
#pragma unroll
    for (int j = 1; j < W; ++j) x[j] = fma(nf, y[j], x[j]);
    x[0] = dcol;
  } else {
    const T c0 = fma(nf, y[0], x[0]);
#pragma unroll
    for (int j = 0; j + 2 < W; ++j) x[j] = fma(nf, y[j + 2], x[j + 2]);
    x[W - 2] = c0;
    x[W - 1] = dcol;
  }
}

// Row stride (elements) of the leaf's pivot rows Rs in shared memory: the B-fragment loads of
// leaf_update_mma (lanes (g, t) read Rs[t][c + g]) then hit distinct banks per half-warp (fp64)
// or per warp (fp32)
template <typename T>
constexpr int rs_ld() {
  return sizeof(T) == 8 ? 132 : 136;
}

__device__ __forceinline__ void dmma884_leaf(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// The leaf's update of the panel's other columns for one warp's 32 rows [r0, r0 + 32) (the
// aggregated Eqs. (14)-(15) within a panel, as in K4b):
//     X[i][P0 + c] = (rep_i ? 0 : X[i][P0 + c]) + sum_s x_i[s] Rs[s][c]
// for c in [0, pw) outside the leaf's columns [off, off + W), rep_i = row i was pivoted in this
// leaf.  FP64 m8n8k4 MMAs (fp32 data converted exactly, accumulated in fp64): A = the rows'
// leaf columns (just written back to X by this warp), B = the leaf's pivot rows (Rs), C = X,
// NCH 8-column tiles at a time.  Why: as per-thread FMAs every Rs element was a broadcast
// shared load feeding two FMAs, and these updates took more of the panel kernel than its
// pivot steps (232 against 168 us per n = 8192 panel, fp64; tools/leaf_prof.sh).
template <typename T, int W>
__device__ __forceinline__ void leaf_update_mma(T* X, int64_t ld, int npad, int P0, int pw, int off, int r0,
                                                bool rep_mine, const T* Rs, int lane) {
  constexpr int RSLD = rs_ld<T>();
  constexpr int NCH = 8;    // 8-column tiles per pass (one pass covers 64 columns)
  constexpr int KS = W / 4; // k4 steps
  const int g = lane >> 2, t = lane & 3;
  const int ntiles = pw / 8;
  const int lt0 = (off + 7) / 8, lt1 = (off + W) / 8;   // tiles wholly inside the leaf
#pragma unroll 1
  for (int mt = 0; mt < 4; ++mt) {
    const int row = r0 + 8 * mt + g;
    const bool ok = row < npad;
    const bool rep = __shfl_sync(0xffffffffu, rep_mine, 8 * mt + g);
    T* cr = X + (int64_t)(ok ? row : 0) * ld + P0;
#pragma unroll 1
    for (int nt0 = 0; nt0 < ntiles; nt0 += NCH) {
      // A (the row's leaf columns k = 4 kk + t) and C of every tile of the pass: all loads
      // issue together, one memory latency per pass
      double av[KS];
#pragma unroll
      for (int kk = 0; kk < KS; ++kk) av[kk] = ok ? (double)cr[off + 4 * kk + t] : 0.0;
      double c[NCH][2];
      bool act[NCH], wr[NCH];
#pragma unroll
      for (int u = 0; u < NCH; ++u) {
        const int nt = nt0 + u, col = 8 * nt + 2 * t;
        act[u] = nt < ntiles && !(nt >= lt0 && nt < lt1);
        wr[u] = act[u] && ok && !(col >= off && col < off + W);   // W = 4: the leaf's half of a tile
        T v0 = T(0), v1 = T(0);
        if (wr[u] && !rep) ld2(cr + col, v0, v1);
        c[u][0] = (double)v0;
        c[u][1] = (double)v1;
      }
#pragma unroll
      for (int kk = 0; kk < KS; ++kk)
#pragma unroll
        for (int u = 0; u < NCH; ++u)
          if (act[u]) dmma884_leaf(c[u][0], c[u][1], av[kk], (double)Rs[(4 * kk + t) * RSLD + 8 * (nt0 + u) + g]);
#pragma unroll
      for (int u = 0; u < NCH; ++u)
        if (wr[u]) st2(cr + 8 * (nt0 + u) + 2 * t, (T)c[u][0], (T)c[u][1]);
    }
  }
}

// Shared-memory layout of the leaf kernel (bytes); T elements
template <typename T, int W>
struct LeafSmem {
  static constexpr int KEYT = 16 / (int)sizeof(T);        // the 16-byte key in T units
  static constexpr int EXW = W + KEYT;                    // entry: key + W row values (T units)
  static constexpr int RS = 0;                            // [W][rs_ld] pivot rows of a leaf (panel columns)
  static constexpr int PROW = RS + W * rs_ld<T>() * (int)sizeof(T);   // [W] pivot row ids of the current leaf
  // [2][kLeafThreads/32][EXW] warp winners, double-buffered by step parity: the bulk copies
  // of step k read their source asynchronously, and only the wait of step k+1 proves (via
  // the peers' step-(k+1) entries) that every peer has received — so the copy has read —
  // this CTA's step-k entry; step k+2 may then rewrite the buffer
  static constexpr int WSLOT = (PROW + W * 4 + 15) / 16 * 16;
  static constexpr int EXCH = WSLOT + 2 * (kLeafThreads / 32) * EXW * (int)sizeof(T);   // [2][CL][EXW]
  static int bytes(int cl) { return EXCH + 2 * cl * EXW * (int)sizeof(T) + 2 * 8 + 64; }
};

// K3 as one launch per PANEL: the panel's leaves one after another, each followed by its
// update of the panel's other columns for this CTA's rows (X[i, T] += (W_i - S_i) R_L[T]
// with the leaf's pivot rows R_L staged in shared memory).  The kernel releases its
// programmatic dependents at once, so the trailing GEMM of the previous panel (launched
// right after it with programmatic stream serialisation) runs on the other SMs while
// this panel is factored (look-ahead).
#ifdef GJ_LEAF_PROF
// diagnostic build only (tools/leaf_prof.sh): per-phase cycle sums of the leaf step, thread 0 of CTA 0
__device__ unsigned long long g_leaf_prof[8];
#define LEAF_T(i)                                                        \
  do {                                                                   \
    if (tid == 0 && rank == 0) {                                         \
      const long long t_ = clock64();                                    \
      if ((i) > 0) atomicAdd(&g_leaf_prof[(i)], (unsigned long long)(t_ - t_prev)); \
      t_prev = t_;                                                       \
    }                                                                    \
  } while (0)
#else
#define LEAF_T(i) do { } while (0)
#endif

template <typename T, int W, int RPT>
__global__ void __launch_bounds__(kLeafThreads, 1) leaf_kernel(LeafArgs a) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#ifdef GJ_LEAF_PROF
  const long long tk0 = clock64();
#endif
#ifdef GJ_TIMELINE
  if (threadIdx.x == 0 && blockIdx.x == 0 && a.c0 % 128 == 0) g_tl[0][a.c0 / 128] = gtime();
#endif
  using LS = LeafSmem<T, W>;
  constexpr int EXW = LS::EXW;
  constexpr int KEYT = LS::KEYT;
  T* const X = static_cast<T*>(a.X);
  extern __shared__ __align__(16) unsigned char smem[];
  T* Rs = reinterpret_cast<T*>(smem + LS::RS);
  int* prow = reinterpret_cast<int*>(smem + LS::PROW);
  T* wslot = reinterpret_cast<T*>(smem + LS::WSLOT);
  T* exch = reinterpret_cast<T*>(smem + LS::EXCH);

  const uint32_t rank = cluster_rank();
  const uint32_t CL = cluster_size();
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + LS::EXCH + 2 * CL * EXW * (int)sizeof(T));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int npad = a.npad, P0 = a.c0, pw = a.pw;
  const int64_t ld = a.ld;
  const uint32_t entry_bytes = (uint32_t)(CL * EXW * (int)sizeof(T));

  T x[RPT][W];
  int pos[RPT], pst[RPT], rowid[RPT];
  bool valid[RPT];
  T myrp[RPT];
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const int r = (int)(rank * (kLeafThreads * RPT)) + i * kLeafThreads + tid;
    rowid[i] = r;
    valid[i] = r < npad;
    pos[i] = valid[i] ? a.pos[r] : 0x7fffffff;
    pst[i] = valid[i] ? a.pivstep[r] : 0;
  }
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
    mbar_expect_tx(&bars[0], entry_bytes);   // steps 0, 2, 4, ...
    mbar_expect_tx(&bars[1], entry_bytes);   // steps 1, 3, 5, ...
  }
  __syncthreads();
  cluster_sync_all();   // every CTA resident and its barriers armed before any remote store

  for (int off = 0, leaf = 0; off < pw; off += W, ++leaf) {
    const int c0 = P0 + off;       // column of the leaf in X
    const int s0 = a.k0 + off;     // global step of the leaf's first column
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      myrp[i] = T(1);
      if (valid[i]) {
        const T* src = X + (int64_t)rowid[i] * ld + c0;
#pragma unroll
        for (int j = 0; j < W; j += 2) ld2(src + j, x[i][j], x[i][j + 1]);
      } else {
#pragma unroll
        for (int j = 0; j < W; ++j) x[i][j] = T(0);
      }
    }
    auto step = [&](int kk, auto pc_tag, auto second_tag) {
      constexpr int PC = decltype(pc_tag)::value;
      constexpr bool SECOND = decltype(second_tag)::value;
#ifdef GJ_LEAF_PROF
      long long t_prev = 0;
#endif
      LEAF_T(0);
      const int kg = s0 + kk;
      const int gk = leaf * W + kk;   // step count within this launch: mbarrier phase
      const int b = gk & 1;
      // ---- a2: this thread's best candidate among its un-pivoted rows
      Cand best{0u, 0u, 0xffffffffu, 0u};
      int bi = -1;
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        if (valid[i] && pst[i] < 0) {
          uint32_t kh, kl;
          abs_key(x[i][PC], kh, kl);
          const Cand c{kh, kl, (uint32_t)pos[i], (uint32_t)rowid[i]};
          if (bi < 0 || better(c, best)) { best = c; bi = i; }
        }
      }
      const bool has = bi >= 0;
      const uint32_t mh = __reduce_max_sync(0xffffffffu, has ? best.hi : 0u);
      const uint32_t ml = __reduce_max_sync(0xffffffffu, (has && best.hi == mh) ? best.lo : 0u);
      const uint32_t pw_ = __reduce_min_sync(0xffffffffu, (has && best.hi == mh && best.lo == ml) ? best.pos : 0xffffffffu);
      // the warp winner writes its KEY into the warp's slot; only the CTA winner (picked by
      // every warp from the keys after the barrier) writes its row values — one lane's
      // 16-byte stores cost the shared pipe the same as a full warp's, so 16 warps writing
      // whole rows every step was the largest part of the step
      LEAF_T(1);
      const bool wwin = has && best.pos == pw_;
      T* const wsb = wslot + b * (kLeafThreads / 32) * EXW;
      if (lane == 0 && pw_ == 0xffffffffu) reinterpret_cast<uint4*>(wsb + warp * EXW)[0] = make_uint4(0u, 0u, 0xffffffffu, 0u);
      if (wwin) reinterpret_cast<uint4*>(wsb + warp * EXW)[0] = make_uint4(best.hi, best.lo, best.pos, best.row);
      __syncthreads();
      LEAF_T(2);
      // ---- CTA winner (every warp picks it redundantly); its lane writes the row; warp d
      // then ships the entry to CTA d with one bulk DSMEM copy completing on the
      // destination's mbarrier — the CL copies issue in parallel from CL warps (a bulk copy
      // takes warp-uniform operands, so one warp issuing all of them would serialise them)
      {
        constexpr int nw = kLeafThreads / 32;
        Cand c{0u, 0u, 0xffffffffu, 0u};
        if (lane < nw) {
          const uint4 k4 = reinterpret_cast<const uint4*>(wsb + lane * EXW)[0];
          c = Cand{k4.x, k4.y, k4.z, k4.w};
        }
        const int src_warp = warp_pick(c, lane < nw);
        if (warp == src_warp && wwin) {
#pragma unroll
          for (int i = 0; i < RPT; ++i) {
            if (bi == i) {
              T* slot = wsb + warp * EXW;
#pragma unroll
              for (int j = 0; j < W; j += 2) st2(slot + KEYT + j, x[i][j], x[i][j + 1]);
            }
          }
          fence_async_smem();
        }
        __syncthreads();
        const uint32_t src = smem_u32(wsb + src_warp * EXW);
        const uint32_t ldst = smem_u32(exch + (size_t)(b * CL + rank) * EXW);
        for (uint32_t d = (uint32_t)warp; d < CL; d += nw)
          if (lane == 0)
            bulk_s2c(map_remote(ldst, d), src, (uint32_t)(EXW * (int)sizeof(T)), map_remote(smem_u32(&bars[b]), d));
      }
      LEAF_T(3);
      // ---- all: wait for the CL entries of this step, pick the cluster winner
      mbar_wait_all(&bars[b], (uint32_t)((gk >> 1) & 1));
      LEAF_T(4);
      if (tid == 0) mbar_expect_tx(&bars[b], entry_bytes);   // arm the barrier for step gk + 2
      const T* ex0 = exch + (size_t)(b * CL) * EXW;
      Cand cc{0u, 0u, 0xffffffffu, 0u};
      if (lane < (int)CL) {
        const uint4 k4 = *reinterpret_cast<const uint4*>(ex0 + (size_t)lane * EXW);
        cc = Cand{k4.x, k4.y, k4.z, k4.w};
      }
      const int wr = warp_pick(cc, lane < (int)CL);
      const Cand wc = [&] {
        const uint4 k4 = *reinterpret_cast<const uint4*>(ex0 + (size_t)wr * EXW);
        return Cand{k4.x, k4.y, k4.z, k4.w};
      }();
      const T* y = ex0 + (size_t)wr * EXW + KEYT;
      const T p = y[PC];
      const int q = (int)wc.pos;
      if (tid == 0) {
        prow[kk] = (int)wc.row;
        if (rank == 0) {
          a.rec_p[kg] = (double)p;
          a.rec_q[kg] = q;
          a.rec_row[kg] = (int)wc.row;
        }
      }
      const T rp = rcp_t(p);
      LEAF_T(5);
      // ---- a3 + a5
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const bool is_piv = valid[i] && pst[i] < 0 && pos[i] == q;
        if (pos[i] == kg) pos[i] = q;
        if (is_piv) {
          pos[i] = kg;
          pst[i] = kg;
          myrp[i] = rp;
        }
        const T nf = is_piv ? T(0) : -(x[i][PC] * rp);
        const T dcol = is_piv ? T(1) : nf;
        leaf_update<T, W, PC, SECOND>(x[i], y, nf, dcol);
      }
      LEAF_T(6);
    };
#pragma unroll 1
    for (int kk = 0; kk < W; kk += 2) {
      step(kk, std::integral_constant<int, 0>{}, std::integral_constant<bool, false>{});
      step(kk + 1, std::integral_constant<int, 1>{}, std::integral_constant<bool, true>{});
    }
    // deferred normalisation of this leaf's pivot rows; write back the leaf columns (W)
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const T sc = (pst[i] >= s0 && pst[i] < s0 + W) ? myrp[i] : T(1);
#pragma unroll
      for (int j = 0; j < W; ++j) x[i][j] *= sc;
      if (!valid[i]) continue;
      T* dst = X + (int64_t)rowid[i] * ld + c0;
#pragma unroll
      for (int j = 0; j < W; j += 2) st2(dst + j, x[i][j], x[i][j + 1]);
    }
    if (pw > W) {
#ifdef GJ_LEAF_PROF
      const long long tu0 = clock64();
#endif
      // the leaf's transformation on the panel's other columns (left: D columns of earlier
      // leaves, right: columns still to be factored), for this CTA's rows
      cluster_sync_all();   // every CTA's earlier updates of the pivot rows are visible
      const int half = pw / 2;
      for (int e = tid; e < W * half; e += kLeafThreads) {
        const int sidx = e / half, cc2 = e - sidx * half;
        T u0, u1;
        ld2(X + (int64_t)prow[sidx] * ld + P0 + 2 * cc2, u0, u1);
        st2(Rs + sidx * rs_ld<T>() + 2 * cc2, u0, u1);
      }
      cluster_sync_all();   // every CTA has its copy before any CTA rewrites a pivot row
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const int r0 = (int)(rank * (kLeafThreads * RPT)) + i * kLeafThreads + warp * 32;
        if (r0 >= npad) continue;   // warp-uniform
        const bool rep = valid[i] && pst[i] >= s0 && pst[i] < s0 + W;   // pivot row of this leaf: replaced
        leaf_update_mma<T, W>(X, ld, npad, P0, pw, c0 - P0, r0, rep, Rs, lane);
      }
      __syncthreads();   // Rs / prow are rewritten by the next leaf
#ifdef GJ_LEAF_PROF
      if (tid == 0 && rank == 0) atomicAdd(&g_leaf_prof[7], (unsigned long long)(clock64() - tu0));
#endif
    }
  }
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    if (!valid[i]) continue;
    a.pos[rowid[i]] = pos[i];
    a.pivstep[rowid[i]] = pst[i];
    if (a.Wout != nullptr) {   // this thread wrote every final panel value of its rows itself
      const T* src = X + (int64_t)rowid[i] * ld + P0;
      T* dst = static_cast<T*>(a.Wout) + (int64_t)rowid[i] * pw;
      for (int j = 0; j < pw; j += 2) {
        T u0, u1;
        ld2(src + j, u0, u1);
        st2(dst + j, u0, u1);
      }
    }
  }
  cluster_sync_all();   // no CTA leaves while a peer's bulk copy may still target it
#ifdef GJ_LEAF_PROF
  if (threadIdx.x == 0 && cluster_rank() == 0) atomicAdd(&g_leaf_prof[0], (unsigned long long)(clock64() - tk0));
#endif
#ifdef GJ_TIMELINE
  if (threadIdx.x == 0 && blockIdx.x == 0 && a.c0 % 128 == 0) g_tl[1][a.c0 / 128] = gtime();
#endif
}

// ============================================================================ K4: GEMM update
// C[i][c] = (replace(i) ? 0 : C[i][c]) + sum_s A[i][s] * B[s][c]
//   A: M x K (ld lda)  = X[:, leaf/panel columns]
//   B: K x N (ld ldb)  = gathered pivot rows R
//   C: M x N (ld ldc)  = X[:, target columns], updated in place
//   replace(i) = pivstep[i] in [rep_lo, rep_hi)
constexpr int BM = 128, BN = 64, BK = 16;   // 2 CTAs per SM: one streams C while the other computes
constexpr int AST = BK + 4;    // A smem row stride (doubles): conflict-free fragment loads
constexpr int BST = BN + 4;    // B smem row stride
#ifndef GJ_GEMM_WARPS
#define GJ_GEMM_WARPS 4
#endif
constexpr int kGemmWarps = GJ_GEMM_WARPS;          // 4: warp tiles 64 x 32; 8: 32 x 32 (build option)
constexpr int kGemmThreads = 32 * kGemmWarps;
constexpr int WTM = kGemmWarps == 4 ? 64 : 32;    // warp tile rows
constexpr int MT = WTM / 16;                      // m16 tiles per warp
#ifndef GJ_GEMM_NST
#define GJ_GEMM_NST 2
#endif
constexpr int GEMM_NST = GJ_GEMM_NST;   // cp.async stages (build option, A/B)
constexpr int GEMM_SMEM = GEMM_NST * (BM * AST + BK * BST) * (int)sizeof(double);

struct GemmArgs {
  const double* A;
  int64_t lda;
  const double* B;
  int64_t ldb;
  double* C;
  int64_t ldc;
  int M, N, K;          // N counts the updated columns (the skipped range excluded)
  const int* pivstep;
  int rep_lo, rep_hi;
  int skip_lo, skip_hi; // B / C columns [skip_lo, skip_hi) are not part of the update (128-aligned)
};

__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g, bool pred) {
  const int sz = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(saddr), "l"(g), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void dmma16816(double (&c)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
      "{%12,%13,%14,%15}, {%0,%1,%2,%3};"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]), "d"(b[1]),
        "d"(b[2]), "d"(b[3]));
}

__global__ void __launch_bounds__(kGemmThreads, 2) gemm_update_kernel(GemmArgs g) {
  extern __shared__ __align__(16) double gsm[];
  double* As = gsm;                       // [GEMM_NST][BM][AST]
  double* Bs = gsm + GEMM_NST * BM * AST; // [GEMM_NST][BK][BST]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;       // (kGemmWarps/2) x 2 warps, warp tile WTM x 32
  const int gq = lane >> 2, tq = lane & 3;
  const int ntn = (g.N + BN - 1) / BN, ntm = (g.M + BM - 1) / BM;
  const int shift = g.skip_hi - g.skip_lo;
  // persistent: tiles in column-major order of the tile grid (consecutive CTAs share B)
  for (int tile = blockIdx.x; tile < ntn * ntm; tile += gridDim.x) {
  const int m0 = (tile % ntm) * BM;
  const int nc0 = (tile / ntm) * BN;                       // compact column of the tile
  const int n0 = nc0 + (nc0 >= g.skip_lo ? shift : 0);     // real column
  const int nlim = n0 + (g.N - nc0);                        // real column bound of this tile

  auto load_stage = [&](int st, int k0) {
    // A: BM x BK doubles in 16-byte chunks (BK/2 per row); B: BK x BN (BN/2 per row)
#pragma unroll
    for (int u = 0; u < BM * BK / 2 / kGemmThreads; ++u) {
      const int c = tid + u * kGemmThreads;
      const int r = c / (BK / 2), kc = (c % (BK / 2)) * 2;
      const int gr = m0 + r;
      const bool ok = gr < g.M && k0 + kc < g.K;
      cp_async16(smem_u32(As + st * BM * AST + r * AST + kc), g.A + (ok ? (int64_t)gr * g.lda + k0 + kc : 0), ok);
    }
#pragma unroll
    for (int u = 0; u < BK * BN / 2 / kGemmThreads; ++u) {
      const int c = tid + u * kGemmThreads;
      const int r = c / (BN / 2), nc = (c % (BN / 2)) * 2;
      const int gc = n0 + nc;
      const bool ok = gc < nlim && k0 + r < g.K;
      cp_async16(smem_u32(Bs + st * BK * BST + r * BST + nc), g.B + (ok ? (int64_t)(k0 + r) * g.ldb + gc : 0), ok);
    }
  };

  // accumulators initialised from C (0 for the rows the update replaces)
  double acc[MT][4][4];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = m0 + wm * WTM + mt * 16 + gq + 8 * h;
      bool keep = r < g.M;
      if (keep) {
        const int ps = g.pivstep[r];
        keep = !(ps >= g.rep_lo && ps < g.rep_hi);
      }
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const int c = n0 + wn * 32 + nt * 8 + 2 * tq;
        double2 v = make_double2(0.0, 0.0);
        if (keep && c < nlim) v = *reinterpret_cast<const double2*>(g.C + (int64_t)r * g.ldc + c);
        acc[mt][nt][2 * h] = v.x;
        acc[mt][nt][2 * h + 1] = v.y;
      }
    }
  }

  const int nk = (g.K + BK - 1) / BK;   // K % 16 == 8 (8-wide leaves): zero-filled tail
#pragma unroll
  for (int st = 0; st < GEMM_NST - 1; ++st) {
    if (st < nk) load_stage(st, st * BK);
    cp_async_commit();
  }
  for (int kb = 0; kb < nk; ++kb) {
    if (kb + GEMM_NST - 1 < nk) load_stage((kb + GEMM_NST - 1) % GEMM_NST, (kb + GEMM_NST - 1) * BK);
    cp_async_commit();
    cp_async_wait<GEMM_NST - 1>();
    __syncthreads();
    const int cs = kb % GEMM_NST;
    const double* as = As + cs * BM * AST + (wm * WTM) * AST;
    const double* bs = Bs + cs * BK * BST + wn * 32;
    // m16n8k16 (8 DMMA.8x8x4 in SASS); measured faster here than k-outer m8n8k4 issue
#pragma unroll
    for (int k16 = 0; k16 < BK; k16 += 16) {
      double bf[4][4];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int i = 0; i < 4; ++i) bf[nt][i] = bs[(k16 + tq + 4 * i) * BST + nt * 8 + gq];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        double af[8];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          af[2 * i] = as[(mt * 16 + gq) * AST + k16 + tq + 4 * i];
          af[2 * i + 1] = as[(mt * 16 + gq + 8) * AST + k16 + tq + 4 * i];
        }
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma16816(acc[mt][nt], af, bf[nt]);
      }
    }
    __syncthreads();
  }

#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = m0 + wm * WTM + mt * 16 + gq + 8 * h;
      if (r >= g.M) continue;
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const int c = n0 + wn * 32 + nt * 8 + 2 * tq;
        if (c < nlim)
          *reinterpret_cast<double2*>(g.C + (int64_t)r * g.ldc + c) = make_double2(acc[mt][nt][2 * h], acc[mt][nt][2 * h + 1]);
      }
    }
  __syncthreads();   // the next tile's first cp.async overwrites stage 0
  }
  // launched as a programmatic dependent of the panel kernel: complete only after it
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// ============================================================================ host driver
struct Workspace {
  double* X;        // npad^2
  double* R;        // PANEL x npad
  double* rec_p;    // npad
  int* rec_q;       // npad
  int* rec_row;     // npad
  int* pos;         // npad
  int* pivstep;     // npad
  unsigned long long* smax;   // 1
};

constexpr int PANEL = 128;

static int pad_to(int n, int m) { return (n + m - 1) / m * m; }

size_t workspace_bytes(int n) {
  const int npad = pad_to(n, 32);
  size_t b = 0;
  b += (size_t)npad * npad * 8;
  b += (size_t)PANEL * npad * 8;
  b += (size_t)npad * 8;
  b += (size_t)npad * 4 * 4;
  b += 256;
  return b + 1024;
}

static Workspace carve(void* ws, int npad) {
  Workspace w;
  char* p = static_cast<char*>(ws);
  auto take = [&](size_t bytes) {
    char* r = p;
    p += (bytes + 255) / 256 * 256;
    return r;
  };
  w.X = reinterpret_cast<double*>(take((size_t)npad * npad * 8));
  w.R = reinterpret_cast<double*>(take((size_t)PANEL * npad * 8));
  w.rec_p = reinterpret_cast<double*>(take((size_t)npad * 8));
  w.rec_q = reinterpret_cast<int*>(take((size_t)npad * 4));
  w.rec_row = reinterpret_cast<int*>(take((size_t)npad * 4));
  w.pos = reinterpret_cast<int*>(take((size_t)npad * 4));
  w.pivstep = reinterpret_cast<int*>(take((size_t)npad * 4));
  w.smax = reinterpret_cast<unsigned long long*>(take(8));
  return w;
}

template <int W, int RPT, typename T = double>
static cudaError_t launch_leaf(const LeafArgs& la, int cl, cudaStream_t s) {
  const size_t smem = (size_t)LeafSmem<T, W>::bytes(cl);
  static unsigned long long configured = 0;
  const unsigned long long dbit = device_bit();
  if (!(configured & dbit)) {
    cudaFuncSetAttribute(leaf_kernel<T, W, RPT>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(leaf_kernel<T, W, RPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    configured |= dbit;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cl, 1, 1);
  cfg.blockDim = dim3(kLeafThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, leaf_kernel<T, W, RPT>, la);
}

// grid_sms: SMs the persistent grid may use; pdl: launch as a programmatic dependent of the
// preceding kernel in the stream (it may start once that kernel has released it).
static cudaError_t launch_gemm(const GemmArgs& g, cudaStream_t s, int grid_sms = 0, bool pdl = false) {
  if (g.M <= 0 || g.N <= 0 || g.K <= 0) return cudaSuccess;
  static int per_sm = 0;
  static unsigned long long configured = 0;
  const unsigned long long dbit = device_bit();
  if (!(configured & dbit)) {
    cudaError_t e = cudaFuncSetAttribute(gemm_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, GEMM_SMEM);
    if (e != cudaSuccess) return e;
    configured |= dbit;
  }
  if (per_sm == 0) {
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gemm_update_kernel, kGemmThreads, GEMM_SMEM);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
  }
  const int tiles = ((g.N + BN - 1) / BN) * ((g.M + BM - 1) / BM);
  const int sms = grid_sms > 0 ? grid_sms : device_sm_count();
  const int grid = tiles < sms * per_sm ? tiles : sms * per_sm;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(kGemmThreads, 1, 1);
  cfg.dynamicSmemBytes = GEMM_SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, gemm_update_kernel, g);
}

// Leaf configuration: cluster size and rows per thread, leaf width W.
struct LeafCfg {
  int cl, rpt, w;
};
static bool leaf_cfg(int npad, LeafCfg* c) {
  // rows per cluster = cl * 512 * rpt; registers hold rpt * w doubles per thread
  if (npad <= 16 * kLeafThreads) { *c = {16, 1, 32}; return true; }
  if (npad <= 16 * kLeafThreads * 2) { *c = {16, 2, 16}; return true; }
  if (npad <= 16 * kLeafThreads * 4) { *c = {16, 4, 8}; return true; }
  if (npad <= 16 * kLeafThreads * 8) { *c = {16, 8, 4}; return true; }
  return false;
}

// K4b launched beside the panel kernel: the whole grid, its last `cl` CTAs (resident only once
// the panel kernel's SMs are free) weighted by the share of the update left when it ends.
// The panel kernel's time relative to the update's (ncols columns) is modelled from
// tools/timeline_large.py measurements on B200 (leaf / update on the other SMs: 308 / 581 us
// at n = 8192, 528 / 2334 at 16384, 1365 / 9386 at 32768: the ratio falls as ~npad^-0.935,
// the update grows as npad * ncols).  0.9 keeps a margin below the measured cliff (n = 8192:
// weights 400..450 measure alike, 500 costs 3%: the late CTAs then finish last).  A wrong
// weight only moves time between CTAs: the tiles and their arithmetic are the same.
#ifndef GJ_DGEMM_LATE_W
#define GJ_DGEMM_LATE_W -1
#endif
static void late_ranges(DgemmArgs& d, int sms, int cl, int npad) {
  d.late_from = sms - cl;
  if (GJ_DGEMM_LATE_W >= 0) {   // A/B builds
    d.late_w = GJ_DGEMM_LATE_W;
    return;
  }
  const double ncols = d.N > 0 ? (double)d.N : 1.0;
  const double leaf_over_update = 0.53 * (8192.0 / ncols) * pow(npad / 8192.0, 0.065);
  const double w = 1024.0 * 0.9 * (1.0 - leaf_over_update);
  d.late_w = w > 0.0 ? (int)w : 0;
}

// Diagnostic builds only (-DGJ_DEBUG_SYNC: synchronise and check after every launch;
// -DGJ_LARGE_NO_PDL: no overlap of the trailing update with the next panel).
static constexpr bool debug_sync() {
#ifdef GJ_DEBUG_SYNC
  return true;
#else
  return false;
#endif
}
static constexpr bool no_pdl() {
#ifdef GJ_LARGE_NO_PDL
  return true;
#else
  return false;
#endif
}
#define GJ_DBG(name)                                                                        \
  do {                                                                                      \
    if (debug_sync()) {                                                                     \
      cudaError_t de = cudaStreamSynchronize(s);                                            \
      if (de != cudaSuccess) {                                                              \
        fprintf(stderr, "gjinv large: %s failed: %s\n", name, cudaGetErrorString(de));      \
        return de;                                                                          \
      }                                                                                     \
    }                                                                                       \
  } while (0)

}  // namespace large

// ============================================================================ fp32 (f1)
// The same blocked Gauss-Jordan in fp32: the panel kernel instantiated for
// float, the trailing update on tcgen05 TF32 tensor cores with a 3xTF32 split
// (gj_tcgemm.cu).  npad is a multiple of 128 (whole tensor-core tiles of K = 128).
namespace f32 {
constexpr int PANEL = large::PANEL;

__global__ void copy_pad_f32(const float* __restrict__ A, int64_t lda, int n, float* __restrict__ X, int npad,
                             unsigned long long* smax) {
  float m = 0.0f;
  const int64_t tot = (int64_t)npad * npad;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / npad), j = (int)(e - (int64_t)i * npad);
    float v;
    if (i < n && j < n) {
      v = A[(int64_t)i * lda + j];
      m = fmaxf(m, fabsf(v));
    } else {
      v = (i == j) ? 1.0f : 0.0f;
    }
    X[e] = v;
  }
  unsigned long long b = (unsigned long long)__double_as_longlong((double)m);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long ob = __shfl_xor_sync(0xffffffffu, b, o);
    b = ob > b ? ob : b;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(smax, b);
}

// x = hi + lo, both rounded to TF32 (10 explicit mantissa bits; the tensor core ignores the
// low 13 bits of an fp32 operand, so rounding them here halves the representation error):
// |x - hi - lo| <= 2^-22 |x|
__device__ __forceinline__ float round_tf32(float x) { return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u); }
__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
  hi = round_tf32(x);
  lo = round_tf32(x - hi);
}

// Ah/Al (npad x 128) = split X[:, P0 .. P0 + 128)  (X rows of stride ld)
__global__ void split_panel_f32(const float* __restrict__ X, int64_t ld, int npad, int P0, float* __restrict__ Ah,
                                float* __restrict__ Al) {
  const int64_t tot = (int64_t)npad * PANEL;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / PANEL), k = (int)(e - (int64_t)i * PANEL);
    float h, l;
    split_tf32(X[(int64_t)i * ld + P0 + k], h, l);
    Ah[e] = h;
    Al[e] = l;
  }
}

// Bh/Bl (ncols x 128): B[c][s] = split X[rows[s]][c]  (R transposed, through a 32 x 32
// tile; one block column per 32 columns of X, rows of stride ld)
__global__ void gather_split_T_f32(const float* __restrict__ X, int64_t ld, const int* __restrict__ rows,
                                   float* __restrict__ Bh, float* __restrict__ Bl) {
  __shared__ float t[32][33];
  const int c0 = blockIdx.x * 32, s0 = blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;   // 32 x 8
  for (int j = ty; j < 32; j += 8) t[j][tx] = X[(int64_t)rows[s0 + j] * ld + c0 + tx];
  __syncthreads();
  for (int j = ty; j < 32; j += 8) {
    float h, l;
    split_tf32(t[tx][j], h, l);
    Bh[(int64_t)(c0 + j) * PANEL + s0 + tx] = h;
    Bl[(int64_t)(c0 + j) * PANEL + s0 + tx] = l;
  }
}

__global__ void unpermute_f32(const float* __restrict__ X, int npad, const int* __restrict__ rec_row,
                              const int* __restrict__ pivstep, int n, float* __restrict__ Y, int64_t ldy) {
  for (int k = blockIdx.y; k < n; k += gridDim.y) {
    const float* src = X + (int64_t)rec_row[k] * npad;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
      Y[(int64_t)k * ldy + j] = src[pivstep[j]];
  }
}

__global__ void finalize_det_f32(const double* logabsdet, const int8_t* sign, float* det) {
  *det = *sign == 0 ? 0.0f : (float)((double)*sign * exp(*logabsdet));
}

struct Workspace {
  float *X, *Ah, *Al, *Bh, *Bl;
  double* rec_p;
  int *rec_q, *rec_row, *pos, *pivstep;
  unsigned long long* smax;
  double* lg;
  int8_t* sg;
};
static int pad128(int n) { return (n + 127) / 128 * 128; }
static size_t bytes(int n) {
  const size_t np = (size_t)pad128(n);
  return np * np * 4 + 4 * np * PANEL * 4 + np * 8 + 4 * np * 4 + 64 + 16 * 256 + 1024;
}
static Workspace carve(void* ws, int npad) {
  Workspace w;
  char* p = static_cast<char*>(ws);
  auto take = [&](size_t b) {
    char* r = p;
    p += (b + 255) / 256 * 256;
    return r;
  };
  w.X = reinterpret_cast<float*>(take((size_t)npad * npad * 4));
  w.Ah = reinterpret_cast<float*>(take((size_t)npad * PANEL * 4));
  w.Al = reinterpret_cast<float*>(take((size_t)npad * PANEL * 4));
  w.Bh = reinterpret_cast<float*>(take((size_t)npad * PANEL * 4));
  w.Bl = reinterpret_cast<float*>(take((size_t)npad * PANEL * 4));
  w.rec_p = reinterpret_cast<double*>(take((size_t)npad * 8));
  w.rec_q = reinterpret_cast<int*>(take((size_t)npad * 4));
  w.rec_row = reinterpret_cast<int*>(take((size_t)npad * 4));
  w.pos = reinterpret_cast<int*>(take((size_t)npad * 4));
  w.pivstep = reinterpret_cast<int*>(take((size_t)npad * 4));
  w.smax = reinterpret_cast<unsigned long long*>(take(8));
  w.lg = reinterpret_cast<double*>(take(8));
  w.sg = reinterpret_cast<int8_t*>(take(8));
  return w;
}
}  // namespace f32

size_t large_workspace_size_f32(int n) { return f32::bytes(n); }

cudaError_t invert_large_f32(int n, const float* A, int64_t lda, float* Ainv, int64_t ldainv, int32_t* ipiv,
                             double* logabsdet, int8_t* sign, float* det, int32_t* info, double tol, void* ws_ptr,
                             cudaStream_t s) {
  using large::LeafCfg;
  using large::LeafArgs;
  using large::leaf_cfg;
  using large::launch_leaf;
  using large::debug_sync;
  constexpr int PANEL = f32::PANEL;
  const int npad = f32::pad128(n);
  LeafCfg lc;
  if (!leaf_cfg(npad, &lc)) return cudaErrorInvalidValue;
  f32::Workspace w = f32::carve(ws_ptr, npad);
  cudaError_t e;
  const int sms = device_sm_count();
  large::init_perm_kernel<<<(npad + 255) / 256, 256, 0, s>>>(npad, w.pos, w.pivstep);
  cudaMemsetAsync(w.smax, 0, 8, s);
  f32::copy_pad_f32<<<sms * 8, 256, 0, s>>>(A, lda, n, w.X, npad, w.smax);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const int det_only = Ainv == nullptr ? 1 : 0;   // gj_det: columns right of the panel only
  auto factor_panel = [&](int P0) -> cudaError_t {
    LeafArgs la{w.X, npad, npad, P0, P0, PANEL, w.pos, w.pivstep, w.rec_p, w.rec_q, w.rec_row, nullptr};
    if (lc.w == 32) return launch_leaf<32, 1, float>(la, lc.cl, s);
    if (lc.w == 16) return launch_leaf<16, 2, float>(la, lc.cl, s);
    if (lc.w == 8) return launch_leaf<8, 4, float>(la, lc.cl, s);
    return launch_leaf<4, 8, float>(la, lc.cl, s);
  };
  if ((e = factor_panel(0)) != cudaSuccess) return e;
  for (int P0 = 0; P0 < npad; P0 += PANEL) {
    const int P1 = P0 + PANEL;
    const bool nxt = P1 < npad;
    f32::split_panel_f32<<<sms * 4, 256, 0, s>>>(w.X, npad, npad, P0, w.Ah, w.Al);
    f32::gather_split_T_f32<<<dim3(npad / 32, PANEL / 32), dim3(32, 8), 0, s>>>(w.X, npad, w.rec_row + P0, w.Bh, w.Bl);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if (nxt) {
      TcUpdateArgs ga{w.Ah, w.Al, w.Bh, w.Bl, w.X, npad, npad, PANEL, npad, w.pivstep, P0, P0 + PANEL, 0, P1};
      if ((e = launch_tc_update(ga, 0, false, s)) != cudaSuccess) return e;
      if ((e = factor_panel(P1)) != cudaSuccess) return e;
    }
    const int pw1 = nxt ? PANEL : 0;
    TcUpdateArgs gb{w.Ah, w.Al, w.Bh, w.Bl, w.X, npad, npad, npad - PANEL - pw1, npad, w.pivstep, P0, P0 + PANEL,
                    P0, P1 + pw1};
    if (det_only) {
      gb.N = npad - P1 - pw1;
      gb.skip_lo = 0;
      gb.skip_hi = P1 + pw1;
    }
    const bool pdl = nxt && !large::no_pdl();
    if ((e = launch_tc_update(gb, pdl ? sms - lc.cl : 0, pdl, s)) != cudaSuccess) return e;
    GJ_DBG("f32 panel");
  }
  if (Ainv != nullptr)
    f32::unpermute_f32<<<dim3((n + 255) / 256, n < 65535 ? n : 65535), 256, 0, s>>>(w.X, npad, w.rec_row, w.pivstep, n, Ainv, ldainv);
  large::finalize_kernel<<<1, 1024, 0, s>>>(n, w.rec_p, w.rec_q, tol, w.smax, ipiv, logabsdet ? logabsdet : w.lg,
                                     sign ? sign : w.sg, nullptr, info);
  if (det != nullptr)
    f32::finalize_det_f32<<<1, 1, 0, s>>>(logabsdet ? logabsdet : w.lg, sign ? sign : w.sg, det);
  return cudaGetLastError();
}

// Large-n solve in fp32 (f4): invert_large_f32's panels on the working array [A | B]
// (npad x (npad + mpad)), each trailing tcgen05 update restricted to the columns right of
// the next panel (as gj_det) — the rest of A and all of B.
namespace f32 {
static int solve_mpad(int m) { return (m + 31) / 32 * 32; }
static size_t solve_bytes(int n, int m) {
  const size_t np = (size_t)pad128(n), ld = np + (size_t)solve_mpad(m);
  return np * ld * 4 + 2 * np * PANEL * 4 + 2 * ld * PANEL * 4 + np * 8 + 4 * np * 4 + 64 + 16 * 256 + 1024;
}
__global__ void copy_pad_solve_f32(const float* __restrict__ A, int64_t lda, const float* __restrict__ B, int64_t ldb,
                                   int n, int m, float* __restrict__ X, int npad, int ld, unsigned long long* smax) {
  float mx = 0.0f;
  const int64_t tot = (int64_t)npad * ld;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / ld), j = (int)(e - (int64_t)i * ld);
    float v;
    if (j < npad) {
      if (i < n && j < n) {
        v = A[(int64_t)i * lda + j];
        mx = fmaxf(mx, fabsf(v));
      } else {
        v = (i == j) ? 1.0f : 0.0f;
      }
    } else {
      const int c = j - npad;
      v = (i < n && c < m) ? B[(int64_t)i * ldb + c] : 0.0f;
    }
    X[e] = v;
  }
  unsigned long long b = (unsigned long long)__double_as_longlong((double)mx);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long ob = __shfl_xor_sync(0xffffffffu, b, o);
    b = ob > b ? ob : b;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(smax, b);
}
__global__ void solve_gather_f32(const float* __restrict__ X, int ld, int npad, const int* __restrict__ rec_row, int n,
                                 int m, float* __restrict__ Xs, int64_t ldx) {
  for (int k = blockIdx.y; k < n; k += gridDim.y) {
    const float* src = X + (int64_t)rec_row[k] * ld + npad;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) Xs[(int64_t)k * ldx + j] = src[j];
  }
}
}  // namespace f32

size_t large_solve_workspace_size_f32(int n, int m) { return f32::solve_bytes(n, m); }

cudaError_t solve_large_f32(int n, int m, const float* A, int64_t lda, const float* B, int64_t ldb, float* Xs,
                            int64_t ldx, int32_t* ipiv, double* logabsdet, int8_t* sign, int32_t* info, double tol,
                            void* ws_ptr, cudaStream_t s) {
  using large::LeafCfg;
  using large::LeafArgs;
  using large::leaf_cfg;
  using large::launch_leaf;
  using large::debug_sync;
  constexpr int PANEL = f32::PANEL;
  const int npad = f32::pad128(n);
  const int ld = npad + f32::solve_mpad(m);
  LeafCfg lc;
  if (!leaf_cfg(npad, &lc)) return cudaErrorInvalidValue;
  f32::Workspace w;
  {
    char* p = static_cast<char*>(ws_ptr);
    auto take = [&](size_t b) {
      char* r = p;
      p += (b + 255) / 256 * 256;
      return r;
    };
    w.X = reinterpret_cast<float*>(take((size_t)npad * ld * 4));
    w.Ah = reinterpret_cast<float*>(take((size_t)npad * PANEL * 4));
    w.Al = reinterpret_cast<float*>(take((size_t)npad * PANEL * 4));
    w.Bh = reinterpret_cast<float*>(take((size_t)ld * PANEL * 4));
    w.Bl = reinterpret_cast<float*>(take((size_t)ld * PANEL * 4));
    w.rec_p = reinterpret_cast<double*>(take((size_t)npad * 8));
    w.rec_q = reinterpret_cast<int*>(take((size_t)npad * 4));
    w.rec_row = reinterpret_cast<int*>(take((size_t)npad * 4));
    w.pos = reinterpret_cast<int*>(take((size_t)npad * 4));
    w.pivstep = reinterpret_cast<int*>(take((size_t)npad * 4));
    w.smax = reinterpret_cast<unsigned long long*>(take(8));
    w.lg = reinterpret_cast<double*>(take(8));
    w.sg = reinterpret_cast<int8_t*>(take(8));
  }
  cudaError_t e;
  const int sms = device_sm_count();
  large::init_perm_kernel<<<(npad + 255) / 256, 256, 0, s>>>(npad, w.pos, w.pivstep);
  cudaMemsetAsync(w.smax, 0, 8, s);
  f32::copy_pad_solve_f32<<<sms * 8, 256, 0, s>>>(A, lda, B, ldb, n, m, w.X, npad, ld, w.smax);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  auto factor_panel = [&](int P0) -> cudaError_t {
    LeafArgs la{w.X, ld, npad, P0, P0, PANEL, w.pos, w.pivstep, w.rec_p, w.rec_q, w.rec_row, nullptr};
    if (lc.w == 32) return launch_leaf<32, 1, float>(la, lc.cl, s);
    if (lc.w == 16) return launch_leaf<16, 2, float>(la, lc.cl, s);
    if (lc.w == 8) return launch_leaf<8, 4, float>(la, lc.cl, s);
    return launch_leaf<4, 8, float>(la, lc.cl, s);
  };
  if ((e = factor_panel(0)) != cudaSuccess) return e;
  for (int P0 = 0; P0 < npad; P0 += PANEL) {
    const int P1 = P0 + PANEL;
    const bool nxt = P1 < npad;
    f32::split_panel_f32<<<sms * 4, 256, 0, s>>>(w.X, ld, npad, P0, w.Ah, w.Al);
    f32::gather_split_T_f32<<<dim3(ld / 32, PANEL / 32), dim3(32, 8), 0, s>>>(w.X, ld, w.rec_row + P0, w.Bh, w.Bl);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if (nxt) {
      TcUpdateArgs ga{w.Ah, w.Al, w.Bh, w.Bl, w.X, ld, npad, PANEL, ld, w.pivstep, P0, P0 + PANEL, 0, P1};
      if ((e = launch_tc_update(ga, 0, false, s)) != cudaSuccess) return e;
      if ((e = factor_panel(P1)) != cudaSuccess) return e;
    }
    const int pw1 = nxt ? PANEL : 0;
    TcUpdateArgs gb{w.Ah, w.Al, w.Bh, w.Bl, w.X, ld, npad, ld - P1 - pw1, ld, w.pivstep, P0, P0 + PANEL, 0, P1 + pw1};
    const bool pdl = nxt && !large::no_pdl();
    if ((e = launch_tc_update(gb, pdl ? sms - lc.cl : 0, pdl, s)) != cudaSuccess) return e;
  }
  f32::solve_gather_f32<<<dim3((m + 127) / 128, n < 65535 ? n : 65535), 128, 0, s>>>(w.X, ld, npad, w.rec_row, n, m, Xs, ldx);
  large::finalize_kernel<<<1, 1024, 0, s>>>(n, w.rec_p, w.rec_q, tol, w.smax, ipiv, logabsdet ? logabsdet : w.lg,
                                     sign ? sign : w.sg, nullptr, info);
  return cudaGetLastError();
}

size_t large_workspace_size(int n) { return large::workspace_bytes(n); }

// Single fp64 matrix, n > 64.  All work on `s`; returns cudaSuccess or the error.
cudaError_t invert_large_f64(int n, const double* A, int64_t lda, double* Ainv, int64_t ldainv, int32_t* ipiv,
                             double* logabsdet, int8_t* sign, double* det, int32_t* info, double tol, void* ws_ptr,
                             cudaStream_t s) {
  using namespace large;
  const int npad = pad_to(n, 32);
  LeafCfg lc;
  if (!leaf_cfg(npad, &lc)) return cudaErrorInvalidValue;
  Workspace w = carve(ws_ptr, npad);
  cudaError_t e;
  const int sms = device_sm_count();
  init_perm_kernel<<<(npad + 255) / 256, 256, 0, s>>>(npad, w.pos, w.pivstep);
  cudaMemsetAsync(w.smax, 0, 8, s);
  copy_pad_absmax_kernel<<<sms * 8, 256, 0, s>>>(A, lda, n, w.X, npad, w.smax);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  GJ_DBG("setup");

  // determinant only (Ainv == NULL, gj_det): the pivots need every column right of the
  // current panel, never the compact D columns on the left — about half the work (the
  // panel itself is factored whole: its compact columns W drive the update)
  const int det_only = Ainv == nullptr ? 1 : 0;
  // Look-ahead over panels: panel k+1 is updated by panel k first and factored by the
  // cluster kernel while the rest of panel k's update runs on the other SMs.
  auto factor_panel = [&](int P0, int pw) -> cudaError_t {
    LeafArgs la{w.X, npad, npad, P0, P0, pw, w.pos, w.pivstep, w.rec_p, w.rec_q, w.rec_row, nullptr};
    if (lc.w == 32) return launch_leaf<32, 1>(la, lc.cl, s);
    if (lc.w == 16) return launch_leaf<16, 2>(la, lc.cl, s);
    if (lc.w == 8) return launch_leaf<8, 4>(la, lc.cl, s);
    return launch_leaf<4, 8>(la, lc.cl, s);
  };
  auto width = [&](int P0) { return (npad - P0) < PANEL ? (npad - P0) : PANEL; };
  if ((e = factor_panel(0, width(0))) != cudaSuccess) return e;
  GJ_DBG("panel 0");
  for (int P0 = 0; P0 < npad; P0 += PANEL) {
    const int pw = width(P0);
    const int P1 = P0 + pw;
    const int pw1 = P1 < npad ? width(P1) : 0;
    // K4b (TMA-fed DMMA GEMM) takes full 128-column panels; a narrower last panel uses K4
    DgemmArgs d{w.X, npad, npad, npad, P0, w.R, npad, w.X, npad, npad, 0, pw, 0, 0, 0, w.pivstep, P0, P0 + pw};
    const bool tma_gemm = pw == PANEL && dgemm_tma_supported(d);
    if (tma_gemm)
      gather_rows_T_kernel<<<dim3((npad + 31) / 32, PANEL / 32), dim3(32, 8), 0, s>>>(w.X, npad, w.rec_row + P0, npad, w.R);
    else
      gather_rows_kernel<<<dim3((npad / 2 + 255) / 256, pw), 256, 0, s>>>(w.X, npad, w.rec_row + P0, pw, w.R, 0, npad);
    if (pw1 > 0) {
      if (tma_gemm) {
        DgemmArgs da = d;
        da.N = pw1;
        da.c_base = P1;
        if ((e = launch_dgemm_tma(da, 0, false, s)) != cudaSuccess) return e;
      } else {
        GemmArgs ga{w.X + P0, npad, w.R + P1, npad, w.X + P1, npad, npad, pw1, pw, w.pivstep, P0, P0 + pw, 0, 0};
        if ((e = launch_gemm(ga, s)) != cudaSuccess) return e;
      }
      GJ_DBG("look-ahead gemm");
      if ((e = factor_panel(P1, pw1)) != cudaSuccess) return e;
    }
    // every column outside panels k and k+1 (the D columns on the left included)
    const int grid_sms = pw1 > 0 ? sms - lc.cl : 0;
    const bool pdl = pw1 > 0 && !debug_sync();
    if (tma_gemm) {
      DgemmArgs db = d;
      db.N = npad - pw - pw1;
      db.c_base = 0;
      db.skip_lo = P0;
      db.skip_hi = P1 + pw1;
      if (det_only) {   // only the columns right of panel k+1
        db.N = npad - P1 - pw1;
        db.skip_lo = 0;
      }
      if (pdl) late_ranges(db, sms, lc.cl, npad);
      if ((e = launch_dgemm_tma(db, pdl ? sms : 0, pdl, s)) != cudaSuccess) return e;
    } else {
      GemmArgs gb{w.X + P0, npad, w.R, npad, w.X, npad, npad, npad - pw - pw1, pw, w.pivstep, P0, P0 + pw, P0, P1 + pw1};
      if (det_only) {   // only the columns right of panel k+1
        gb.N = npad - P1 - pw1;
        gb.skip_lo = 0;
        gb.skip_hi = P1 + pw1;
      }
      if ((e = launch_gemm(gb, s, grid_sms, pdl)) != cudaSuccess) return e;
    }
    GJ_DBG("trailing gemm");
  }
  if (Ainv != nullptr) {
    if (npad <= kUnpermSmemMaxN) {
      const int smem = npad * 8;
      static unsigned long long configured = 0;
      const unsigned long long dbit = device_bit();
      if (!(configured & dbit)) {
        if ((e = cudaFuncSetAttribute(unpermute_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      kUnpermSmemMaxN * 8)) != cudaSuccess)
          return e;
        configured |= dbit;
      }
      unpermute_smem_kernel<<<sms * (smem <= 72 * 1024 ? 3 : 1), 512, smem, s>>>(w.X, npad, w.rec_row, w.pivstep, n,
                                                                                  Ainv, ldainv);
    } else {
      unpermute_kernel<<<dim3((n + 255) / 256, n < 65535 ? n : 65535), 256, 0, s>>>(w.X, npad, w.rec_row, w.pivstep, n,
                                                                                     Ainv, ldainv);
    }
  }
  finalize_kernel<<<1, 1024, 0, s>>>(n, w.rec_p, w.rec_q, tol, w.smax, ipiv, logabsdet, sign, det, info);
  return cudaGetLastError();
}

// ============================================================================ large-n solve (f4)
// X = A^-1 B for one fp64 matrix: the working array is [A | B] (npad x (npad + mpad)); the
// panels and pivots are gj_invert's, and — as in the determinant-only mode — the trailing
// update of panel k touches only the columns right of panel k+1: the rest of A and the
// right-hand sides (the compact D columns on the left are never needed).  The pivot rows
// end normalised, so the solution row k is the B part of the row pivoted at step k.
namespace large {
static int solve_ld(int npad, int m) { return npad + pad_to(m, 32); }
size_t solve_workspace_bytes(int n, int m) {
  const int npad = pad_to(n, 32), ld = solve_ld(npad, m);
  return (size_t)npad * ld * 8 + (size_t)PANEL * ld * 8 + (size_t)npad * 8 + (size_t)npad * 4 * 4 + 256 + 1024 +
         6 * 256;
}
// X[:, :npad] = blockdiag(A, I); X[:, npad:] = [B | 0; 0]
__global__ void copy_pad_solve_kernel(const double* __restrict__ A, int64_t lda, const double* __restrict__ B,
                                      int64_t ldb, int n, int m, double* __restrict__ X, int npad, int ld) {
  const int64_t tot = (int64_t)npad * ld;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / ld), j = (int)(e - (int64_t)i * ld);
    double v;
    if (j < npad) {
      v = (i < n && j < n) ? A[(int64_t)i * lda + j] : (i == j ? 1.0 : 0.0);
    } else {
      const int c = j - npad;
      v = (i < n && c < m) ? B[(int64_t)i * ldb + c] : 0.0;
    }
    X[e] = v;
  }
}
// Xs[k][j] = X[rec_row[k]][npad + j]
__global__ void solve_gather_kernel(const double* __restrict__ X, int ld, int npad, const int* __restrict__ rec_row,
                                    int n, int m, double* __restrict__ Xs, int64_t ldx) {
  for (int k = blockIdx.y; k < n; k += gridDim.y) {
    const double* src = X + (int64_t)rec_row[k] * ld + npad;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) Xs[(int64_t)k * ldx + j] = src[j];
  }
}
}  // namespace large

size_t large_solve_workspace_size(int n, int m) { return large::solve_workspace_bytes(n, m); }

cudaError_t solve_large_f64(int n, int m, const double* A, int64_t lda, const double* B, int64_t ldb, double* Xs,
                            int64_t ldx, int32_t* ipiv, double* logabsdet, int8_t* sign, int32_t* info, double tol,
                            void* ws_ptr, cudaStream_t s) {
  using namespace large;
  const int npad = pad_to(n, 32);
  const int ld = solve_ld(npad, m);
  LeafCfg lc;
  if (!leaf_cfg(npad, &lc)) return cudaErrorInvalidValue;
  Workspace w;
  {
    char* p = static_cast<char*>(ws_ptr);
    auto take = [&](size_t bytes) {
      char* r = p;
      p += (bytes + 255) / 256 * 256;
      return r;
    };
    w.X = reinterpret_cast<double*>(take((size_t)npad * ld * 8));
    w.R = reinterpret_cast<double*>(take((size_t)PANEL * ld * 8));
    w.rec_p = reinterpret_cast<double*>(take((size_t)npad * 8));
    w.rec_q = reinterpret_cast<int*>(take((size_t)npad * 4));
    w.rec_row = reinterpret_cast<int*>(take((size_t)npad * 4));
    w.pos = reinterpret_cast<int*>(take((size_t)npad * 4));
    w.pivstep = reinterpret_cast<int*>(take((size_t)npad * 4));
    w.smax = reinterpret_cast<unsigned long long*>(take(8));
  }
  cudaError_t e;
  const int sms = device_sm_count();
  init_perm_kernel<<<(npad + 255) / 256, 256, 0, s>>>(npad, w.pos, w.pivstep);
  copy_pad_solve_kernel<<<sms * 8, 256, 0, s>>>(A, lda, B, ldb, n, m, w.X, npad, ld);
  cudaMemsetAsync(w.smax, 0, 8, s);
  absmax_kernel<<<sms * 8, 256, 0, s>>>(A, lda, n, w.smax);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  auto factor_panel = [&](int P0, int pw) -> cudaError_t {
    LeafArgs la{w.X, ld, npad, P0, P0, pw, w.pos, w.pivstep, w.rec_p, w.rec_q, w.rec_row, nullptr};
    if (lc.w == 32) return launch_leaf<32, 1>(la, lc.cl, s);
    if (lc.w == 16) return launch_leaf<16, 2>(la, lc.cl, s);
    if (lc.w == 8) return launch_leaf<8, 4>(la, lc.cl, s);
    return launch_leaf<4, 8>(la, lc.cl, s);
  };
  auto width = [&](int P0) { return (npad - P0) < PANEL ? (npad - P0) : PANEL; };
  if ((e = factor_panel(0, width(0))) != cudaSuccess) return e;
  for (int P0 = 0; P0 < npad; P0 += PANEL) {
    const int pw = width(P0);
    const int P1 = P0 + pw;
    const int pw1 = P1 < npad ? width(P1) : 0;
    // the panel's pivot rows, columns from P1 on (the right part of A and all of B)
    gather_rows_kernel<<<dim3((ld / 2 + 255) / 256, pw), 256, 0, s>>>(w.X, ld, w.rec_row + P0, pw, w.R, P1, ld);
    if (pw1 > 0) {
      GemmArgs ga{w.X + P0, ld, w.R + P1, ld, w.X + P1, ld, npad, pw1, pw, w.pivstep, P0, P0 + pw, 0, 0};
      if ((e = launch_gemm(ga, s)) != cudaSuccess) return e;
      if ((e = factor_panel(P1, pw1)) != cudaSuccess) return e;
    }
    GemmArgs gb{w.X + P0, ld, w.R, ld, w.X, ld, npad, ld - P1 - pw1, pw, w.pivstep, P0, P0 + pw, 0, P1 + pw1};
    if ((e = launch_gemm(gb, s, pw1 > 0 ? sms - lc.cl : 0, pw1 > 0 && !debug_sync())) != cudaSuccess) return e;
  }
  solve_gather_kernel<<<dim3((m + 127) / 128, n < 65535 ? n : 65535), 128, 0, s>>>(w.X, ld, npad, w.rec_row, n, m, Xs, ldx);
  finalize_kernel<<<1, 1024, 0, s>>>(n, w.rec_p, w.rec_q, tol, w.smax, ipiv, logabsdet, sign, nullptr, info);
  return cudaGetLastError();
}

// ============================================================================ distributed
// Column-block-cyclic large-n inversion over P ranks: global column block j
// (DB = 128 columns, the panel width) lives on rank j % P.  Rows are complete on every
// rank, so a panel's pivot search is local to its owner; each panel step is
//   owner:  dist_factor  (the panel kernel above, on the owner's local columns) -> W
//   all:    broadcast W + the step record + positions from the owner (caller, NCCL)
//   all:    dist_update  (gather the panel's pivot rows of the local columns, DMMA GEMM)
// and the un-permutation (listing L179-L198) is one all-to-all of columns at the end.
namespace dist {
constexpr int DB = large::PANEL;

__host__ __device__ inline int nblocks(int npad) { return npad / DB; }
__host__ __device__ inline int local_blocks(int npad, int P, int rank) { return (nblocks(npad) - rank + P - 1) / P; }
__host__ __device__ inline int global_col(int lc, int P, int rank) { return ((lc / DB) * P + rank) * DB + lc % DB; }
__host__ __device__ inline int owner(int gc, int P) { return (gc / DB) % P; }
__host__ __device__ inline int local_col(int gc, int P) { return (gc / DB / P) * DB + gc % DB; }

// X_local (npad x nl) = this rank's columns of blockdiag(A, I); A_local holds the rank's
// real columns (global column < n) in increasing order, row stride lda.
__global__ void init_local_kernel(const double* __restrict__ A, int64_t lda, int n, int npad, int P, int rank, int nl,
                                  double* __restrict__ X, unsigned long long* smax) {
  double m = 0.0;
  const int64_t tot = (int64_t)npad * nl;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / nl), lc = (int)(e - (int64_t)i * nl);
    const int gc = global_col(lc, P, rank);
    double v;
    if (i < n && gc < n) {
      v = A[(int64_t)i * lda + lc];   // local real columns come first, in order (gc < n <=> lc < real count)
      m = fmax(m, fabs(v));
    } else {
      v = (i == gc) ? 1.0 : 0.0;
    }
    X[e] = v;
  }
  unsigned long long b = (unsigned long long)__double_as_longlong(m);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long ob = __shfl_xor_sync(0xffffffffu, b, o);
    b = ob > b ? ob : b;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(smax, b);
}

// Exchange plan of the un-permutation Ainv[i][j] = X[rec_row[i]][pivstep[j]] (one CTA):
// for every output column j < n, source compact column c = pivstep[j] on rank owner(c),
// destination rank owner(j).  This rank sends its columns ordered by (destination, j) and
// receives ordered by (source, j).  counts[0..P) = columns sent to each rank,
// counts[P..2P) = columns received from each rank.
constexpr int kPlanThreads = 512, kMaxP = 8;
__global__ void __launch_bounds__(kPlanThreads) unpermute_plan_kernel(int n, int P, int rank, const int* __restrict__ pivstep,
                                                                      int* send_cols, int* recv_cols, int* counts) {
  __shared__ int cs[kMaxP][kPlanThreads + 1], cr[kMaxP][kPlanThreads + 1];
  __shared__ int bs[kMaxP + 1], br[kMaxP + 1];
  const int t = threadIdx.x;
  const int chunk = (n + kPlanThreads - 1) / kPlanThreads;
  const int j0 = t * chunk, j1 = min(n, j0 + chunk);
  int ls[kMaxP], lr[kMaxP];
#pragma unroll
  for (int d = 0; d < kMaxP; ++d) ls[d] = lr[d] = 0;
  for (int j = j0; j < j1; ++j) {
    const int c = pivstep[j];
    const int src = owner(c, P), dst = owner(j, P);
#pragma unroll
    for (int d = 0; d < kMaxP; ++d) {
      if (src == rank && dst == d) ++ls[d];
      if (dst == rank && src == d) ++lr[d];
    }
  }
#pragma unroll
  for (int d = 0; d < kMaxP; ++d) {
    cs[d][t] = ls[d];
    cr[d][t] = lr[d];
  }
  __syncthreads();
  if (t < 2 * kMaxP) {   // exclusive scans over threads, one per (direction, rank)
    int* a = t < kMaxP ? cs[t] : cr[t - kMaxP];
    int run = 0;
    for (int u = 0; u < kPlanThreads; ++u) {
      const int v = a[u];
      a[u] = run;
      run += v;
    }
    a[kPlanThreads] = run;
  }
  __syncthreads();
  if (t == 0) {
    int x = 0, y = 0;
    for (int d = 0; d < kMaxP; ++d) {
      bs[d] = x;
      br[d] = y;
      x += cs[d][kPlanThreads];
      y += cr[d][kPlanThreads];
      if (d < P) {
        counts[d] = cs[d][kPlanThreads];
        counts[P + d] = cr[d][kPlanThreads];
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int d = 0; d < kMaxP; ++d) {
    ls[d] = bs[d] + cs[d][t];
    lr[d] = br[d] + cr[d][t];
  }
  for (int j = j0; j < j1; ++j) {
    const int c = pivstep[j];
    const int src = owner(c, P), dst = owner(j, P);
#pragma unroll
    for (int d = 0; d < kMaxP; ++d) {
      if (src == rank && dst == d) send_cols[ls[d]++] = local_col(c, P);
      if (dst == rank && src == d) recv_cols[lr[d]++] = local_col(j, P);
    }
  }
}

// sendbuf[t][i] = X[rec_row[i]][send_cols[t]] (i < n): row gather of the un-permutation
__global__ void unpermute_pack_kernel(int n, const double* __restrict__ X, int64_t ld, const int* __restrict__ rec_row,
                                      const int* __restrict__ send_cols, int m, double* __restrict__ out) {
  const int i = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= n) return;
  const double* src = X + (int64_t)rec_row[i] * ld;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < m; t += gridDim.x * blockDim.x)
    out[(int64_t)t * n + i] = src[send_cols[t]];
}
// Ainv_local[i][recv_cols[t]] = in[t][i]
__global__ void unpermute_unpack_kernel(int n, const double* __restrict__ in, const int* __restrict__ recv_cols, int m,
                                        double* __restrict__ Y, int64_t ldy) {
  const int i = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= n) return;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < m; t += gridDim.x * blockDim.x)
    Y[(int64_t)i * ldy + recv_cols[t]] = in[(int64_t)t * n + i];
}
}  // namespace dist

void dist_sizes(int n, int P, int rank, int* npad, int* nl, int* nl_real) {
  const int np = (n + dist::DB - 1) / dist::DB * dist::DB;
  *npad = np;
  *nl = dist::local_blocks(np, P, rank) * dist::DB;
  int cnt = 0;
  for (int lc = 0; lc < *nl; ++lc)
    if (dist::global_col(lc, P, rank) < n) ++cnt;
  *nl_real = cnt;
}

cudaError_t dist_init(int n, int P, int rank, const double* A_local, int64_t lda, double* Xl, int* pos, int* pivstep,
                      unsigned long long* smax, cudaStream_t s) {
  int npad, nl, nr;
  dist_sizes(n, P, rank, &npad, &nl, &nr);
  const int sms = device_sm_count();
  large::init_perm_kernel<<<(npad + 255) / 256, 256, 0, s>>>(npad, pos, pivstep);
  cudaMemsetAsync(smax, 0, 8, s);
  if (nl > 0) dist::init_local_kernel<<<sms * 8, 256, 0, s>>>(A_local, lda, n, npad, P, rank, nl, Xl, smax);
  return cudaGetLastError();
}

cudaError_t dist_factor(int n, int P, int rank, int k, double* Xl, int* pos, int* pivstep, double* rec_p, int* rec_q,
                        int* rec_row, double* W, cudaStream_t s) {
  using namespace large;
  int npad, nl, nr;
  dist_sizes(n, P, rank, &npad, &nl, &nr);
  if (k < 0 || k >= dist::nblocks(npad) || k % P != rank) return cudaErrorInvalidValue;
  LeafCfg lc;
  if (!leaf_cfg(npad, &lc)) return cudaErrorInvalidValue;
  const int c0 = (k / P) * dist::DB;
  // the panel kernel also writes W itself, so a following programmatic-dependent GEMM
  // (gj_dist_update part 2) overlaps it directly
  LeafArgs la{Xl, nl, npad, c0, k * dist::DB, dist::DB, pos, pivstep, rec_p, rec_q, rec_row, W};
  return lc.w == 32 ? launch_leaf<32, 1>(la, lc.cl, s)
         : lc.w == 16 ? launch_leaf<16, 2>(la, lc.cl, s)
         : lc.w == 8  ? launch_leaf<8, 4>(la, lc.cl, s)
                      : launch_leaf<4, 8>(la, lc.cl, s);
}

// part 0: every local column except this rank's own panel k (gather + GEMM);
// part 1: gather, then only the local columns of panel k+1 (this rank must own k+1);
// part 2: the local columns outside panels k and k+1, R already gathered by part 1,
//         launched as a programmatic dependent of the preceding kernel (the factorisation
//         of panel k+1) on the SMs its cluster leaves free — the look-ahead of §8e.
cudaError_t dist_update(int n, int P, int rank, int k, int part, double* Xl, const double* W, const int* pivstep,
                        const int* rec_row, double* R, cudaStream_t s) {
  using namespace large;
  int npad, nl, nr;
  dist_sizes(n, P, rank, &npad, &nl, &nr);
  const int nb = dist::nblocks(npad);
  if (k < 0 || k >= nb || part < 0 || part > 2) return cudaErrorInvalidValue;
  if (part > 0 && (k + 1 >= nb || (k + 1) % P != rank)) return cudaErrorInvalidValue;
  if (nl == 0) return cudaSuccess;
  const int k0 = k * dist::DB;
  const bool own = k % P == rank;
  const int c0 = (k / P) * dist::DB;             // local block of panel k (if owned)
  const int c1 = ((k + 1) / P) * dist::DB;       // local block of panel k+1 (if owned)
  LeafCfg lc;
  if (!leaf_cfg(npad, &lc)) return cudaErrorInvalidValue;
  // K4b (TMA-fed DMMA GEMM) with the pivot rows transposed (RT, nl x 128); K4 otherwise
  DgemmArgs d{W, dist::DB, npad, dist::DB, 0, R, nl, Xl, nl, npad, 0, dist::DB, 0, 0, 0, pivstep, k0, k0 + dist::DB};
#ifdef GJ_NO_DGEMM_TMA
  const bool tma_gemm = false;
#else
  const bool tma_gemm = dgemm_tma_supported(d);
#endif
  if (part != 2) {
    if (tma_gemm)
      gather_rows_T_kernel<<<dim3((nl + 31) / 32, dist::DB / 32), dim3(32, 8), 0, s>>>(Xl, nl, rec_row + k0, nl, R);
    else
      gather_rows_kernel<<<dim3((nl / 2 + 255) / 256, dist::DB), 256, 0, s>>>(Xl, nl, rec_row + k0, dist::DB, R, 0, nl);
  }
  if (part == 1) {
    if (tma_gemm) {
      d.N = dist::DB;
      d.c_base = c1;
      return launch_dgemm_tma(d, 0, false, s);
    }
    GemmArgs g{W, dist::DB, R + c1, nl, Xl + c1, nl, npad, dist::DB, dist::DB, pivstep, k0, k0 + dist::DB, 0, 0};
    return launch_gemm(g, s);
  }
  if (part == 0) {
    if (tma_gemm) {
      d.N = nl - (own ? dist::DB : 0);
      d.skip_lo = own ? c0 : 0;
      d.skip_hi = own ? c0 + dist::DB : 0;
      return launch_dgemm_tma(d, 0, false, s);
    }
    GemmArgs g{W, dist::DB, R, nl, Xl, nl, npad, nl - (own ? dist::DB : 0), dist::DB, pivstep, k0, k0 + dist::DB,
               own ? c0 : 0, own ? c0 + dist::DB : 0};
    return launch_gemm(g, s);
  }
  // part 2: skip [c1, c1 + DB) and, when this rank also owns panel k (P == 1: adjacent), [c0, c0 + DB)
  int lo = c1, hi = c1 + dist::DB;
  if (own) {
    lo = c0 < c1 ? c0 : c1;
    hi = (c0 > c1 ? c0 : c1) + dist::DB;
    if (hi - lo != 2 * dist::DB) return cudaErrorInvalidValue;   // only adjacent blocks (P == 1)
  }
  if (tma_gemm) {
    d.N = nl - (hi - lo);
    d.skip_lo = lo;
    d.skip_hi = hi;
    late_ranges(d, device_sm_count(), lc.cl, npad);
    return launch_dgemm_tma(d, device_sm_count(), true, s);
  }
  GemmArgs g{W, dist::DB, R, nl, Xl, nl, npad, nl - (hi - lo), dist::DB, pivstep, k0, k0 + dist::DB, lo, hi};
  return launch_gemm(g, s, device_sm_count() - lc.cl, true);
}

cudaError_t dist_finalize(int n, const double* rec_p, const int* rec_q, double tol, const unsigned long long* smax,
                          int32_t* ipiv, double* logabsdet, int8_t* sign, int32_t* info, cudaStream_t s) {
  large::finalize_kernel<<<1, 1024, 0, s>>>(n, rec_p, rec_q, tol, smax, ipiv, logabsdet, sign, nullptr, info);
  return cudaGetLastError();
}

cudaError_t dist_unpermute_plan(int n, int P, int rank, const int* pivstep, int* send_cols, int* recv_cols, int* counts,
                                cudaStream_t s) {
  if (P > dist::kMaxP) return cudaErrorInvalidValue;
  dist::unpermute_plan_kernel<<<1, dist::kPlanThreads, 0, s>>>(n, P, rank, pivstep, send_cols, recv_cols, counts);
  return cudaGetLastError();
}

cudaError_t dist_unpermute_pack(int n, int P, int rank, const double* Xl, const int* rec_row, const int* send_cols,
                                int m, double* sendbuf, cudaStream_t s) {
  int npad, nl, nr;
  dist_sizes(n, P, rank, &npad, &nl, &nr);
  if (m <= 0 || n <= 0) return cudaSuccess;
  dim3 blk(32, 8), grd((m + 31) / 32 < 64 ? (m + 31) / 32 : 64, (n + 7) / 8);
  dist::unpermute_pack_kernel<<<grd, blk, 0, s>>>(n, Xl, nl, rec_row, send_cols, m, sendbuf);
  return cudaGetLastError();
}

cudaError_t dist_unpermute_unpack(int n, const double* recvbuf, const int* recv_cols, int m, double* Ainv_local,
                                  int64_t ld, cudaStream_t s) {
  if (m <= 0 || n <= 0) return cudaSuccess;
  dim3 blk(32, 8), grd((m + 31) / 32 < 64 ? (m + 31) / 32 : 64, (n + 7) / 8);
  dist::unpermute_unpack_kernel<<<grd, blk, 0, s>>>(n, recvbuf, recv_cols, m, Ainv_local, ld);
  return cudaGetLastError();
}

}  // namespace gj

#ifdef GJ_LEAF_PROF
extern "C" int gj_debug_leaf_prof(unsigned long long* out8, int reset) {
  cudaDeviceSynchronize();
  if (cudaMemcpyFromSymbol(out8, gj::large::g_leaf_prof, 8 * sizeof(unsigned long long)) != cudaSuccess) return -1;
  if (reset) {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(gj::large::g_leaf_prof, z, sizeof(z));
  }
  return 0;
}
#endif

#ifdef GJ_TIMELINE
extern "C" int gj_debug_timeline_gemm(unsigned long long* out, int reset);
extern "C" int gj_debug_timeline(unsigned long long* out, int reset) {   // out: [5][512]
  cudaDeviceSynchronize();
  if (cudaMemcpyFromSymbol(out, gj::g_tl, sizeof(gj::g_tl)) != cudaSuccess) return -1;
  if (reset) {
    static unsigned long long z[2][512];
    cudaMemcpyToSymbol(gj::g_tl, z, sizeof(z));
  }
  return gj_debug_timeline_gemm(out + 2 * 512, reset);
}
#endif
