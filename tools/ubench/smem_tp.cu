// Shared-memory pipe cost (SM cycles per warp instruction, 32 warps/SM, independent ops) of
// the access patterns the batched kernels use: broadcast LDS of 32/64/128 bits with 1, 2
// or 4 distinct addresses per warp, and predicated STS.128 / STS.32 with few active lanes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench/smem_tp tools/ubench/smem_tp.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITERS = 2048;

template <int OP>
__global__ void __launch_bounds__(256) k(float* out, int salt) {
  __shared__ __align__(16) float s[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) s[i] = (float)i;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(s) + w * 1024;
  float a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  uint32_t off;
  // distinct-address groups: 1 (all lanes), 2 (half-warps), 4 (quarter-warps), 32
  if (OP % 4 == 0) off = 0;
  else if (OP % 4 == 1) off = (lane >> 4) * 448;
  else if (OP % 4 == 2) off = (lane >> 3) * 448;
  else off = lane * 16;
  const int kind = OP / 4;   // 0 LDS.32, 1 LDS.64, 2 LDS.128, 3 STS.128 pred (1 lane/half), 4 STS.128 pred 4 lanes, 5 STS.32 scatter
#pragma unroll 8
  for (int i = 0; i < ITERS; ++i) {
    const uint32_t ad = base + ((off + (i & 7) * 16) & 1023);
    if (kind == 0) {
      float v; asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(ad) : "memory"); a0 += v;
    } else if (kind == 1) {
      float v0, v1; asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(v0), "=f"(v1) : "r"(ad) : "memory"); a0 += v0; a1 += v1;
    } else if (kind == 2) {
      float v0, v1, v2, v3;
      asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v0), "=f"(v1), "=f"(v2), "=f"(v3) : "r"(ad) : "memory");
      a0 += v0; a1 += v1; a2 += v2; a3 += v3;
    } else if (kind == 3) {
      // predicated STS.128: lanes (salt + 16 h) % 32 active (2 lanes, one per half-warp)
      const bool p = ((lane - salt - (i & 3)) & 15) == 0;
      asm volatile("{.reg .pred q; setp.ne.u32 q, %0, 0; @q st.shared.v4.f32 [%1], {%2,%2,%2,%2};}" ::"r"(p ? 1u : 0u),
                   "r"(base + ((((lane & 15) + (lane >> 4) * 7) * 16 + i * 512) & 1023)), "f"(a0) : "memory");
    } else if (kind == 4) {
      const bool p = ((lane - salt - (i & 3)) & 7) == 0;   // 4 lanes, one per quarter
      asm volatile("{.reg .pred q; setp.ne.u32 q, %0, 0; @q st.shared.v4.f32 [%1], {%2,%2,%2,%2};}" ::"r"(p ? 1u : 0u),
                   "r"(base + ((((lane & 7) + (lane >> 3) * 9) * 16 + i * 512) & 1023)), "f"(a0) : "memory");
    } else if (kind >= 6 && kind <= 11) {
      // predicated STS.32 / .64 / .128 with 1 lane per half-warp (kind 6,7,8) or all lanes (9,10,11)
      const bool p = kind >= 9 ? true : (((lane - salt - (i & 3)) & 15) == 0);
      const int wd = (kind - 6) % 3;
      const uint32_t ad = base + ((lane * (4 << wd) + i * 512) & 1023);
      if (wd == 0) asm volatile("{.reg .pred q; setp.ne.u32 q, %0, 0; @q st.shared.f32 [%1], %2;}" ::"r"(p ? 1u : 0u), "r"(ad), "f"(a0) : "memory");
      else if (wd == 1) asm volatile("{.reg .pred q; setp.ne.u32 q, %0, 0; @q st.shared.v2.f32 [%1], {%2,%2};}" ::"r"(p ? 1u : 0u), "r"(ad), "f"(a0) : "memory");
      else asm volatile("{.reg .pred q; setp.ne.u32 q, %0, 0; @q st.shared.v4.f32 [%1], {%2,%2,%2,%2};}" ::"r"(p ? 1u : 0u), "r"(ad), "f"(a0) : "memory");
    } else if (kind == 5) {
      // STS.32 scatter: lane -> row (lane * 5 + i) % 32 of a 32 x 32 tile, column (i * 7) % 32, 128-B swizzle
      const int row = (lane * 5 + i) & 31, col = (i * 7 + (lane >> 4) * 13) & 31;
      const uint32_t b = row * 128 + ((((col >> 2) ^ (row & 7)) << 4) | ((col & 3) << 2));
      asm volatile("st.shared.f32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(s) + (w & 1) * 4096 + b), "f"(a0) : "memory");
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3;
}

template <int OP>
void run(const char* name, float* out, int sms) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k<OP><<<sms * 4, 256>>>(out, 3);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) k<OP><<<sms * 4, 256>>>(out, 3);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double cycles = ms / 5 * 1e-3 * clk * 1e3;
  printf("%-40s %6.2f SM cycles per warp instruction\n", name, cycles / (32.0 * ITERS));
}

int main() {
  float* out;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaMalloc(&out, sms * 4 * 256 * 4);
  run<0>("LDS.32  1 addr", out, sms);
  run<1>("LDS.32  2 addr (half-warps)", out, sms);
  run<2>("LDS.32  4 addr (quarters)", out, sms);
  run<3>("LDS.32  32 addr (distinct banks)", out, sms);
  run<4>("LDS.64  1 addr", out, sms);
  run<5>("LDS.64  2 addr", out, sms);
  run<6>("LDS.64  4 addr", out, sms);
  run<7>("LDS.64  32 addr", out, sms);
  run<8>("LDS.128 1 addr", out, sms);
  run<9>("LDS.128 2 addr", out, sms);
  run<10>("LDS.128 4 addr", out, sms);
  run<11>("LDS.128 32 addr", out, sms);
  run<12>("STS.128 pred, 2 lanes (1/half)", out, sms);
  run<16>("STS.128 pred, 4 lanes (1/quarter)", out, sms);
  run<20>("STS.32 scatter (swz128, 2 matrices)", out, sms);
  run<24>("STS.32 pred, 2 lanes", out, sms);
  run<28>("STS.64 pred, 2 lanes", out, sms);
  run<32>("STS.128 pred, 2 lanes (again)", out, sms);
  run<36>("STS.32 all lanes distinct", out, sms);
  run<40>("STS.64 all lanes distinct", out, sms);
  run<44>("STS.128 all lanes distinct", out, sms);
  return 0;
}
