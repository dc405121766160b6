// Row operations shared by the batched kernels (K1 gj_batched.cu, K2 gj_batched64.cu):
// the rotated elimination update of Eq. (15), the pivot-row publish/broadcast, the
// per-step (p, q) record and log|p|.
#pragma once
#include <cuda_runtime.h>
#include <cmath>
#include <cstdint>

#include "gj_ptx.cuh"

namespace gj {
namespace rowops {

using namespace ptx;

// ------------------------------------------------------------------ a5: rotated update
template <int NP>
__device__ __forceinline__ void update_first(float (&x)[NP], const float (&y)[NP], float nf) {
  x[1] = fmaf(nf, y[1], x[1]);
#pragma unroll
  for (int j = 2; j < NP; j += 2) ffma2(x[j], x[j + 1], nf, y[j], y[j + 1]);
}
template <int NP>
__device__ __forceinline__ void update_first(double (&x)[NP], const double (&y)[NP], double nf) {
#pragma unroll
  for (int j = 1; j < NP; ++j) x[j] = fma(nf, y[j], x[j]);
}
template <int NP>
__device__ __forceinline__ void update_second_rot(float (&x)[NP], const float (&y)[NP], float nf, float dcol) {
  const float c0 = fmaf(nf, y[0], x[0]);
#pragma unroll
  for (int j = 0; j + 3 < NP; j += 2) {
    float a = x[j + 2], b = x[j + 3];
    ffma2(a, b, nf, y[j + 2], y[j + 3]);
    x[j] = a;
    x[j + 1] = b;
  }
  x[NP - 2] = c0;
  x[NP - 1] = dcol;
}
template <int NP>
__device__ __forceinline__ void update_second_rot(double (&x)[NP], const double (&y)[NP], double nf, double dcol) {
  const double c0 = fma(nf, y[0], x[0]);
#pragma unroll
  for (int j = 0; j + 2 < NP; ++j) x[j] = fma(nf, y[j + 2], x[j + 2]);
  x[NP - 2] = c0;
  x[NP - 1] = dcol;
}

// Pivot-row publish (predicated, no branch) and broadcast read.
template <typename T, int NP>
__device__ __forceinline__ void st_row_if(bool pred, T* dst, const T (&x)[NP]) {
  if constexpr ((NP * sizeof(T)) % 16 == 0) {
    const uint32_t a = smem_u32(dst);
#pragma unroll
    for (int j = 0; j < NP; j += 16 / (int)sizeof(T)) {
      if constexpr (sizeof(T) == 4) {
        st_shared_v4_if(pred, a + 4u * j, x[j], x[j + 1], x[j + 2], x[j + 3]);
      } else {
        st_shared_v2_if(pred, a + 8u * j, x[j], x[j + 1]);
      }
    }
  } else {
    if (pred) {
#pragma unroll
      for (int j = 0; j < NP; ++j) dst[j] = x[j];
    }
  }
}
template <typename T, int NP>
__device__ __forceinline__ void ld_row(T (&y)[NP], const T* src) {
  if constexpr ((NP * sizeof(T)) % 16 == 0) {
#pragma unroll
    for (int j = 0; j < NP; j += 16 / (int)sizeof(T)) {
      if constexpr (sizeof(T) == 4) {
        const float4 v = *reinterpret_cast<const float4*>(src + j);
        y[j] = v.x; y[j + 1] = v.y; y[j + 2] = v.z; y[j + 3] = v.w;
      } else {
        const double2 v = *reinterpret_cast<const double2*>(src + j);
        y[j] = v.x; y[j + 1] = v.y;
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < NP; ++j) y[j] = src[j];
  }
}

// Per-step record (p, q); one lane per group writes it.
__device__ __forceinline__ void rec_store(unsigned char* rec, int idx, float p, int q) {
  *reinterpret_cast<uint2*>(rec + 8 * idx) = make_uint2(__float_as_uint(p), (uint32_t)q);
}
__device__ __forceinline__ void rec_store(unsigned char* rec, int idx, double p, int q) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(p);
  *reinterpret_cast<uint4*>(rec + 16 * idx) = make_uint4((uint32_t)b, (uint32_t)(b >> 32), (uint32_t)q, 0u);
}
__device__ __forceinline__ void rec_load(const unsigned char* rec, int idx, float& p, int& q) {
  const uint2 u = *reinterpret_cast<const uint2*>(rec + 8 * idx);
  p = __uint_as_float(u.x);
  q = (int)u.y;
}
__device__ __forceinline__ void rec_load(const unsigned char* rec, int idx, double& p, int& q) {
  const uint4 u = *reinterpret_cast<const uint4*>(rec + 16 * idx);
  p = __longlong_as_double((long long)(((unsigned long long)u.y << 32) | u.x));
  q = (int)u.z;
}

// log|p| in fp64.  For fp32 pivots the hardware log2 (rel. error ~2^-22 of log2|p|,
// far below the fp32 pivots' own rounding) suffices; fp64 uses the full-precision log.
__device__ __forceinline__ double log_abs(float p) {
  // log2|p| = e + log2(m), m in [1, 2): exact (0) for powers of two
  const uint32_t b = __float_as_uint(p) & 0x7fffffffu;
  const int e = (int)(b >> 23) - 127;
  const float m = __uint_as_float((b & 0x7fffffu) | 0x3f800000u);
  return ((double)e + (double)__log2f(m)) * 0.6931471805599453;
}
__device__ __forceinline__ double log_abs(double p) { return log(fabs(p)); }

}  // namespace rowops
}  // namespace gj
