// K6 — batched Gauss–Jordan with FULL pivoting, n <= 32.
//
// Obs. 2-3: at step k the pivot may be any a_ij with i, j among the
// rows and columns not yet pivoted, brought to the pivot position by swapping rows k, i
// and columns k, j; the element of maximum |a_ij| is taken, and the swaps are undone at
// the end.  Layout and flow follow K1 (lane = row, the row in registers, one matrix per
// NP lanes, NP = next power of two >= n), with both permutations kept LOGICAL:
//   a2  each lane: max |x_ij| over its row's un-pivoted columns (a warp-uniform bitmask);
//       group max; among the rows attaining it the smallest physical row position wins
//       (reading G23: the first maximum of the row-major scan over positions i, j = k..n);
//       that row is published to shared memory and lane j (which also keeps column j's
//       physical position) tests |y_j|: among the columns attaining the maximum the
//       smallest physical column position wins.
//   a3  positions of the swapped row pair and column pair (listing L156-L162, both ways);
//       the record keeps (p, row position, column position, row, column) per step.
//   a4/a5 as K1 with a data-dependent pivot column c: x_i -= (x_ic / p) y (the pivot
//       row un-normalised, scaled once at the store), and column c becomes the compact D
//       column (-x_ic / p; 1 on the pivot row), held scaled by -p so that only the pivot
//       row's entry changes (negated) — undone by one multiply per element at the store.
//   a6  det = (-1)^(row swaps + column swaps) prod p_k (Eq. (13) for A Q), log|det|.
//   a7  with r_k, c_k the row and column of step k, the compact array T satisfies
//       A^-1[c_k][r_m] = T[r_k][c_m] / p_k (the Jordan-exchange form of "undo the row and
//       column swaps"; partial pivoting is the case c_k = k).
// Padding rows/columns (n < NP) start as pivoted, so they are never candidates.
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

constexpr int kFullWarps = 4;

template <int L>
__device__ __forceinline__ uint32_t gmax_u32(uint32_t v) {
  if constexpr (L == 32) {
    return __reduce_max_sync(0xffffffffu, v);
  } else {
#pragma unroll
    for (int o = L / 2; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
  }
}
template <int L>
__device__ __forceinline__ uint32_t gmin_u32(uint32_t v) {
  if constexpr (L == 32) {
    return __reduce_min_sync(0xffffffffu, v);
  } else {
#pragma unroll
    for (int o = L / 2; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
  }
}
template <int L>
__device__ __forceinline__ double gsum(double v) {
#pragma unroll
  for (int o = L / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// |x| as an ordered unsigned key (IEEE bit pattern of a non-negative number is monotone)
__device__ __forceinline__ uint32_t akey(float v) { return __float_as_uint(v) & 0x7fffffffu; }
__device__ __forceinline__ unsigned long long akey(double v) {
  return (unsigned long long)__double_as_longlong(v) & 0x7fffffffffffffffull;
}
template <int L>
__device__ __forceinline__ uint32_t gmax_key(uint32_t v) { return gmax_u32<L>(v); }
template <int L>
__device__ __forceinline__ unsigned long long gmax_key(unsigned long long v) {
  const uint32_t h = gmax_u32<L>((uint32_t)(v >> 32));
  const uint32_t l = gmax_u32<L>((uint32_t)(v >> 32) == h ? (uint32_t)v : 0u);
  return ((unsigned long long)h << 32) | l;
}

// x[c] for a data-dependent c < NP: a select tree on the bits of c (NP - 1 selects)
template <typename T, int NP>
__device__ __forceinline__ T sel_col(const T (&x)[NP], int c) {
  T v[NP];
#pragma unroll
  for (int j = 0; j < NP; ++j) v[j] = x[j];
#pragma unroll
  for (int w = NP / 2, b = 0; w >= 1; w /= 2, ++b) {
    const bool hi = (c >> b) & 1;
#pragma unroll
    for (int j = 0; j < w; ++j) v[j] = hi ? v[2 * j + 1] : v[2 * j];
  }
  return v[0];
}

template <int NP>
__device__ __forceinline__ void ld_masks(uint32_t (&m)[NP], const uint32_t* src) {
  if constexpr (NP % 4 == 0) {
#pragma unroll
    for (int j = 0; j < NP; j += 4) {
      const uint4 v = *reinterpret_cast<const uint4*>(src + j);
      m[j] = v.x; m[j + 1] = v.y; m[j + 2] = v.z; m[j + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < NP; ++j) m[j] = src[j];
  }
}

// the key every NaN maps to (one above +inf's)
template <typename K>
__device__ __forceinline__ K knan() {
  if constexpr (sizeof(K) == 4) return 0x7f800001u;
  else return 0x7ff0000000000001ull;
}

// |x| key with a per-column mask m (all ones: column un-pivoted; 0: pivoted or padding)
__device__ __forceinline__ uint32_t mkey(float v, uint32_t m) { return __float_as_uint(v) & m & 0x7fffffffu; }
__device__ __forceinline__ unsigned long long mkey(double v, uint32_t m) {
  return (unsigned long long)__double_as_longlong(v) & (((unsigned long long)m << 32) | m) & 0x7fffffffffffffffull;
}

template <typename T, int NP>
struct FullSmem {
  static constexpr int MPW = 32 / NP;
  static constexpr int ROWS = MPW * NP;                          // 32
  static constexpr int STAGE = ROWS * (NP + 1) * (int)sizeof(T); // padded rows
  static constexpr int PROW = ROWS * (int)sizeof(T);             // one pivot row per matrix
  static constexpr int RECP = ROWS * (int)sizeof(T);             // p per step
  static constexpr int RECQ = ROWS * 4;                          // packed (qr, qc, row, col)
  static constexpr int PERM = ROWS * 4;
  static constexpr int MVEC = ROWS * 4;                          // per-column masks
  static constexpr int per_warp = (STAGE + PROW + RECP + RECQ + PERM + MVEC + 15) / 16 * 16;
};

// resident CTAs per SM the register budget is sized for (fp64 n = 32 needs the most)
template <typename T, int NP>
constexpr int full_min_blocks() { return NP < 32 ? 4 : (sizeof(T) == 8 ? 2 : 3); }

// STRAT: 2 = full pivoting (Obs. 2-3), 1 = partial (the listing: rows only, column k),
// 0 = none (Eqs. (3)-(10) literally: pivot a_kk).  0 and 1 exist for the strategy /
// rounding-error harness — the same arithmetic under each strategy;
// the product partial-pivoting path is K1/K1b.
template <typename T, int NP, int STRAT>
__global__ void __launch_bounds__(kFullWarps * 32, full_min_blocks<T, NP>()) gj_full_kernel(BatchedArgs a, int32_t* jpiv) {
  using S = FullSmem<T, NP>;
  constexpr int L = NP, MPW = S::MPW;
  using K = decltype(akey(T(0)));
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char* wb = smem_raw + warp * S::per_warp;
  unsigned char* stage = wb;
  T* prow = reinterpret_cast<T*>(wb + S::STAGE);
  T* recp = reinterpret_cast<T*>(wb + S::STAGE + S::PROW);
  uint32_t* recq = reinterpret_cast<uint32_t*>(wb + S::STAGE + S::PROW + S::RECP);
  int* perm = reinterpret_cast<int*>(wb + S::STAGE + S::PROW + S::RECP + S::RECQ);
  uint32_t* mvec = reinterpret_cast<uint32_t*>(wb + S::STAGE + S::PROW + S::RECP + S::RECQ + S::PERM);

  const int n = a.n, nn = n * n;
  const int g = lane / L, li = lane % L;
  const unsigned gmask = (L == 32 ? 0xffffffffu : ((1u << L) - 1u)) << (L * g);
  T* prow_g = prow + g * NP;
  T* recp_g = recp + g * NP;
  uint32_t* recq_g = recq + g * NP;
  int* perm_g = perm + g * NP;
  uint32_t* mvec_g = mvec + g * NP;
  const T* __restrict__ Ag = static_cast<const T*>(a.A);
  T* __restrict__ Xg = static_cast<T*>(a.Ainv);
  auto saddr = [&](int row, int col) { return reinterpret_cast<T*>(stage) + row * (NP + 1) + col; };

  // warp access geometry of the load / store: rows_per_it whole rows of n elements
  constexpr int kMaxIt = NP;   // <= MPW * n rows per task, >= 32 / n rows per access
  const int rows_per_it = 32 / n;
  const int lr = lane / n, lc = lane - (lane / n) * n;
  const bool lact = lr < rows_per_it;
  // staging row of the task's row R (matrix R / n, row R % n): R < 32, so the rounded
  // float quotient is exact
  const float rn = 1.0f / (float)n;
  auto srow = [&](int R) {
    const int m = (int)(((float)R + 0.5f) * rn);
    return m * NP + (R - m * n);
  };

  const int64_t ntasks = (a.batch + MPW - 1) / MPW;
  for (int64_t task = (int64_t)blockIdx.x * kFullWarps + warp; task < ntasks;
       task += (int64_t)gridDim.x * kFullWarps) {
    const int64_t item0 = task * MPW;
    const int64_t left = a.batch - item0;
    const int valid_items = left < MPW ? (int)left : MPW;
    const bool item_ok = g < valid_items;
    // ---- a1: the task's valid_items * n rows, rows_per_it whole rows per warp access
    // (lane -> (row lr, column lc) of the access; consecutive lanes read consecutive
    // addresses), every load of the task in flight before the first store to the stage
    const int nrows = valid_items * n;
    const T* At = Ag + item0 * nn;   // the task's matrices (32-bit offsets from here on)
    T* Xt = Xg != nullptr ? Xg + item0 * nn : nullptr;
    {
      T v[kMaxIt];
#pragma unroll
      for (int it = 0; it < kMaxIt; ++it) {
        const int R = it * rows_per_it + lr;
        v[it] = (lact && R < nrows) ? __ldcs(At + R * n + lc) : T(0);
      }
#pragma unroll
      for (int it = 0; it < kMaxIt; ++it) {
        const int R = it * rows_per_it + lr;
        if (lact && R < nrows) *saddr(srow(R), lc) = v[it];
      }
      __syncwarp();
    }
    const bool real = li < n;
    T x[NP];
#pragma unroll
    for (int j = 0; j < NP; ++j) x[j] = (item_ok && real && j < n) ? *saddr(g * NP + li, j) : T(li == j ? 1 : 0);
    __syncwarp();
    T rowmax = T(0);
#pragma unroll
    for (int j = 0; j < NP; ++j)
      if (real && j < n) rowmax = fmax(rowmax, fabs(x[j]));
    double smax;
    if constexpr (sizeof(T) == 4) {
      smax = (double)__uint_as_float(gmax_u32<L>(__float_as_uint(rowmax)));
    } else {
      smax = __longlong_as_double((long long)gmax_key<L>(akey(rowmax)));
    }
    const T tau = round_down_to(a.tol * smax, T(0));

    int pos = li, cpos = li;            // physical row position; physical position of column li
    bool rdone = !real, cdone_l = !real;
    mvec_g[li] = li < n ? 0xffffffffu : 0u;   // column masks: all ones = un-pivoted
    __syncwarp();

#pragma unroll 1
    for (int k = 0; k < n; ++k) {
      // ---- a2: the row's best key over its un-pivoted columns, group max
      int qr, rsrc, qc, c;
      bool piv;
      if constexpr (STRAT == 2) {
        uint32_t cm[NP];
        ld_masks<NP>(cm, mvec_g);
        K km = 0;
#pragma unroll
        for (int j = 0; j < NP; ++j) {
          const K kj = mkey(x[j], cm[j]);
          km = kj > km ? kj : km;
        }
        // a singular item turns its rows into NaN after a zero pivot (1/0 * 0); all NaN keys
        // are mapped to one value just above +inf, so the candidate searches below always
        // find a row and a column (the item is flagged; its inverse is unspecified)
        km = km > knan<K>() ? knan<K>() : km;
        const K m = gmax_key<L>(rdone ? K(0) : km);
        // smallest physical row position among the rows attaining m
        const uint32_t rc = (!rdone && km == m) ? ((uint32_t)pos << 8 | (uint32_t)li) : 0xffffffu;
        const uint32_t rw = gmin_u32<L>(rc);
        qr = (int)(rw >> 8);
        rsrc = (int)(rw & 0xffu);
        piv = li == rsrc;
        st_row_if<T, NP>(piv, prow_g, x);
        __syncwarp();
        // smallest physical column position among the pivot row's columns attaining m
        const T yl = prow_g[li];
        K ky = akey(yl);
        ky = ky > knan<K>() ? knan<K>() : ky;
        const uint32_t cc = (!cdone_l && ky == m) ? ((uint32_t)cpos << 8 | (uint32_t)li) : 0xffffffu;
        const uint32_t cw = gmin_u32<L>(cc);
        qc = (int)(cw >> 8);
        c = (int)(cw & 0xffu);
      } else if constexpr (STRAT == 1) {
        // the listing's search (L151-L153): column k, max |x_ik| over the un-pivoted rows,
        // ties -> smallest physical row position (G3); columns never move
        c = k;
        qc = k;
        K key = akey(sel_col<T, NP>(x, k));
        key = key > knan<K>() ? knan<K>() : key;
        const K m = gmax_key<L>(rdone ? K(0) : key);
        const uint32_t rc = (!rdone && key == m) ? ((uint32_t)pos << 8 | (uint32_t)li) : 0xffffffu;
        const uint32_t rw = gmin_u32<L>(rc);
        qr = (int)(rw >> 8);
        rsrc = (int)(rw & 0xffu);
        piv = li == rsrc;
        st_row_if<T, NP>(piv, prow_g, x);
        __syncwarp();
      } else {
        // no pivoting: the pivot is a_kk (Eqs. (3)-(10)); nothing ever moves
        c = k;
        qc = k;
        qr = k;
        rsrc = k;
        piv = li == k;
        st_row_if<T, NP>(piv, prow_g, x);
        __syncwarp();
      }
      const T p = prow_g[c];
      __syncwarp();
      // the pivot column's entry of the broadcast row is 0: the update leaves column c alone
      // (its D entries are kept SCALED, see below)
      if (li == c) prow_g[li] = T(0);
      __syncwarp();
      T y[NP];
      ld_row<T, NP>(y, prow_g);
      if (li == 0) {
        recp_g[k] = p;
        recq_g[k] = (uint32_t)qr | (uint32_t)qc << 8 | (uint32_t)rsrc << 16 | (uint32_t)c << 24;
      }
      // ---- a4/a5.  Column c becomes a compact D column, held scaled by sigma_c = -p: the
      // D entry of a row i != r, -x_ic / p, is then x_ic itself — unchanged, as the
      // broadcast row has y_c = 0.  The pivot row is negated (nf = -2: x - 2x, exact; its
      // deferred row scale becomes -p) except its entry c, which stays p = 1 * (-p) * (-p).
      // Later updates are linear in rows and columns, so both scalings persist; the store
      // undoes them with one multiply each.  No register is written at a data-dependent
      // index; x_ic is read by a 5-level select on the bits of c.
      const T xc = sel_col<T, NP>(x, c);
      const T nf = piv ? T(-2) : -(xc * rcp(p));
      if constexpr (sizeof(T) == 4) {
#pragma unroll
        for (int j = 0; j < NP; j += 2) ffma2(x[j], x[j + 1], nf, y[j], y[j + 1]);
      } else {
#pragma unroll
        for (int j = 0; j < NP; ++j) x[j] = fma(nf, y[j], x[j]);
      }
      if (STRAT == 2 && li == c) mvec_g[li] = 0u;
      // ---- a3: positions of the swapped rows and columns
      if (pos == k) pos = qr;
      if (piv) { pos = k; rdone = true; }
      if (cpos == k) cpos = qc;
      if (li == c) { cpos = k; cdone_l = true; }
      __syncwarp();   // prow_g is rewritten by the next step
    }

    // ---- a6: det / ipiv / jpiv / singular flag from the record (lane li <-> step li)
    unsigned failb = 0;
    int nswap = 0, nneg = 0;
    double lgl = 0.0;
    {
      const bool stepk = li < n;
      const T pk = stepk ? recp_g[li] : T(1);
      const uint32_t qk = stepk ? recq_g[li] : 0u;
      const int qrk = (int)(qk & 0xffu), qck = (int)((qk >> 8) & 0xffu);
      const unsigned fb = __ballot_sync(0xffffffffu, stepk && fabs(pk) <= tau) & gmask;
      if (fb != 0) failb = (unsigned)(__ffs(fb) - g * L);
      nswap = __popc(__ballot_sync(0xffffffffu, stepk && qrk != li) & gmask) +
              __popc(__ballot_sync(0xffffffffu, stepk && qck != li) & gmask);
      nneg = __popc(__ballot_sync(0xffffffffu, stepk && pk < T(0)) & gmask);
      if (stepk) lgl = log_abs(pk);
      if (item_ok && stepk) {
        if (a.ipiv) a.ipiv[(item0 + g) * n + li] = qrk + 1;
        if (jpiv) jpiv[(item0 + g) * n + li] = qck + 1;
      }
    }
    const int info = (int)failb;
    const double lg = gsum<L>(lgl);
    const int sgn = ((nswap ^ nneg) & 1) ? -1 : 1;
    if (item_ok && li == 0) {
      const int64_t item = item0 + g;
      if (a.info) a.info[item] = info;
      if (a.logabsdet) a.logabsdet[item] = info ? -INFINITY : lg;
      if (a.sign) a.sign[item] = info ? 0 : (int8_t)sgn;
      if (a.det) static_cast<T*>(a.det)[item] = info ? T(0) : (T)(sgn * exp(lg));
    }

    // ---- a7 + a8: A^-1[c_k][r_m] = T[r_k][c_m] / p_k through the staging rows
    if (Xg != nullptr) {
      if (real) {
        perm_g[li] = (int)((recq_g[cpos] >> 16) & 0xffu);   // output column of column li
        prow_g[li] = -rcp(recp_g[cpos]);                     // 1 / sigma of column li
      }
      __syncwarp();
      if (real) {
        const T rp = -rcp(recp_g[pos]);                      // 1 / the deferred row scale -p
        const int orow = (int)(recq_g[pos] >> 24);          // output row of this row
        T cs[NP];
        ld_row<T, NP>(cs, prow_g);
        uint32_t oc[NP];
        ld_masks<NP>(oc, reinterpret_cast<const uint32_t*>(perm_g));
        T* dst = saddr(g * NP + orow, 0);
#pragma unroll
        for (int j = 0; j < NP; ++j)
          if (j < n) dst[oc[j]] = (rp * x[j]) * cs[j];
      }
      __syncwarp();
#pragma unroll
      for (int it = 0; it < kMaxIt; ++it) {
        const int R = it * rows_per_it + lr;
        if (lact && R < nrows) __stcs(Xt + R * n + lc, *saddr(srow(R), lc));
      }
    }
    __syncwarp();
  }
}

template <typename T, int NP, int STRAT>
cudaError_t launch_full_t(const BatchedArgs& a, int32_t* jpiv, cudaStream_t s) {
  using S = FullSmem<T, NP>;
  const int smem = kFullWarps * S::per_warp;
  const int64_t ntasks = (a.batch + S::MPW - 1) / S::MPW;
  const int64_t need = (ntasks + kFullWarps - 1) / kFullWarps;
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gj_full_kernel<T, NP, STRAT>, kFullWarps * 32, smem);
  if (e != cudaSuccess) return e;
  const int64_t cap = (int64_t)device_sm_count() * (per_sm > 0 ? per_sm : 1);
  const int grid = (int)(need < cap ? need : cap);
  gj_full_kernel<T, NP, STRAT><<<grid, kFullWarps * 32, smem, s>>>(a, jpiv);
  return cudaGetLastError();
}

template <typename T, int STRAT>
cudaError_t launch_full_dt(const BatchedArgs& a, int32_t* jpiv, cudaStream_t s) {
  if (a.n <= 2) return launch_full_t<T, 2, STRAT>(a, jpiv, s);
  if (a.n <= 4) return launch_full_t<T, 4, STRAT>(a, jpiv, s);
  if (a.n <= 8) return launch_full_t<T, 8, STRAT>(a, jpiv, s);
  if (a.n <= 16) return launch_full_t<T, 16, STRAT>(a, jpiv, s);
  return launch_full_t<T, 32, STRAT>(a, jpiv, s);
}

template <typename T>
cudaError_t launch_strat(const BatchedArgs& a, int32_t* jpiv, int strategy, cudaStream_t s) {
  if (strategy == 0) return launch_full_dt<T, 0>(a, jpiv, s);
  if (strategy == 1) return launch_full_dt<T, 1>(a, jpiv, s);
  return launch_full_dt<T, 2>(a, jpiv, s);
}

}  // namespace

cudaError_t launch_batched_strategy(gj_dtype dt, const BatchedArgs& a, int32_t* jpiv, int strategy, cudaStream_t s) {
  if (a.n < 1 || a.n > 32 || strategy < 0 || strategy > 2) return cudaErrorInvalidValue;
  return dt == GJ_F32 ? launch_strat<float>(a, jpiv, strategy, s) : launch_strat<double>(a, jpiv, strategy, s);
}

}  // namespace gj
