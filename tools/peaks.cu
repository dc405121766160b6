// K9 — micro-benchmarks for the roofline denominators MEASURED_PEAKS.json lacks
// (FP32 FFMA / FFMA2, FP64 DFMA, FP64 DMMA via mma.sync, HBM copy, device facts).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/peaks tools/peaks.cu
// Prints one JSON object on stdout. Not part of the product path.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int ITERS = 4096;

__global__ void k_ffma(float* out, float a, float b) {
  float x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fmaf(x[i], a, b);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 1234.5f) out[0] = s;
}

__global__ void k_ffma2(float* out, float a, float b) {
  unsigned long long x[8];
  unsigned long long av, bv;
  asm("mov.b64 %0, {%1,%1};" : "=l"(av) : "f"(a));
  asm("mov.b64 %0, {%1,%1};" : "=l"(bv) : "f"(b));
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float lo = threadIdx.x * 1e-3f + i, hi = lo + 0.5f;
    asm("mov.b64 %0, {%1,%2};" : "=l"(x[i]) : "f"(lo), "f"(hi));
  }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[i]) : "l"(av), "l"(bv));
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float lo, hi;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(lo), "=f"(hi) : "l"(x[i]));
    s += lo + hi;
  }
  if (s == 1234.5f) out[0] = s;
}

__global__ void k_dfma(double* out, double a, double b) {
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 1234.5) out[0] = s;
}

// DMMA m8n8k4 (sm_80 shape): D(8x8) += A(8x4) B(4x8); per warp 2*8*8*4 = 512 flop
__global__ void k_dmma884(double* out, double a0) {
  double acc[4][2];
#pragma unroll
  for (int t = 0; t < 4; ++t) acc[t][0] = acc[t][1] = 0.0;
  double av = a0 + threadIdx.x, bv = a0 - threadIdx.x;
  for (int it = 0; it < ITERS / 4; ++it) {
#pragma unroll
    for (int t = 0; t < 4; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[t][0]), "+d"(acc[t][1]) : "d"(av), "d"(bv));
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 4; ++t) s += acc[t][0] + acc[t][1];
  if (s == 1234.5) out[0] = s;
}

// DMMA m16n8k16 (sm_90+ shape): per warp 2*16*8*16 = 4096 flop
__global__ void k_dmma16816(double* out, double a0) {
  double acc[2][4];
#pragma unroll
  for (int t = 0; t < 2; ++t)
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[t][i] = 0.0;
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = a0 + threadIdx.x + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = a0 - threadIdx.x - i;
  for (int it = 0; it < ITERS / 32; ++it) {
#pragma unroll
    for (int t = 0; t < 2; ++t)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
                   "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(acc[t][0]), "+d"(acc[t][1]), "+d"(acc[t][2]), "+d"(acc[t][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 2; ++t)
#pragma unroll
    for (int i = 0; i < 4; ++i) s += acc[t][i];
  if (s == 1234.5) out[0] = s;
}

__global__ void k_copy(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) b[i] = a[i];
}

template <typename F>
static float time_ms(F f, int reps) {
  cudaEvent_t s, e;
  cudaEventCreate(&s); cudaEventCreate(&e);
  f();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(s);
    f();
    cudaEventRecord(e);
    cudaEventSynchronize(e);
    float ms; cudaEventElapsedTime(&ms, s, e);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  int clk = 0, memclk = 0, smemOptin = 0, l2 = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaDeviceGetAttribute(&smemOptin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  cudaDeviceGetAttribute(&memclk, cudaDevAttrMemoryClockRate, 0);
  const int sms = p.multiProcessorCount;
  float* fo; double* dd;
  CK(cudaMalloc(&fo, 64)); CK(cudaMalloc(&dd, 64));
  const int blocks = sms * 8, threads = 256;
  const double nthr = (double)blocks * threads;
  float t_ffma = time_ms([&] { k_ffma<<<blocks, threads>>>(fo, 0.999f, 0.001f); }, 5);
  float t_ffma2 = time_ms([&] { k_ffma2<<<blocks, threads>>>(fo, 0.999f, 0.001f); }, 5);
  float t_dfma = time_ms([&] { k_dfma<<<blocks, threads>>>(dd, 0.999, 0.001); }, 5);
  float t_d884 = time_ms([&] { k_dmma884<<<blocks, threads>>>(dd, 0.5); }, 5);
  float t_d16816 = time_ms([&] { k_dmma16816<<<blocks, threads>>>(dd, 0.5); }, 5);
  CK(cudaGetLastError());
  const double ffma_flop = nthr * ITERS * 16 * 2;
  const double ffma2_flop = nthr * ITERS * 8 * 4;
  const double dfma_flop = nthr * (ITERS / 4) * 16 * 2;
  const double nwarps = nthr / 32;
  const double d884_flop = nwarps * (ITERS / 4) * 4 * 512.0;
  const double d16816_flop = nwarps * (ITERS / 32) * 2 * 4096.0;
  size_t bytes = (size_t)4 << 30;
  float4 *a, *b;
  CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes));
  cudaMemset(a, 0, bytes);
  size_t n4 = bytes / 16;
  float t_copy = time_ms([&] { k_copy<<<sms * 16, 512>>>(a, b, n4); }, 10);
  float t_memcpy = time_ms([&] { cudaMemcpyAsync(b, a, bytes, cudaMemcpyDeviceToDevice); }, 10);
  CK(cudaGetLastError());
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_khz\": %d, \"mem_clock_khz\": %d, \"smem_optin\": %d, "
         "\"l2_bytes\": %d, \"regs_per_sm\": %d, \"cc\": \"%d.%d\", "
         "\"ffma_tflops\": %.2f, \"ffma2_tflops\": %.2f, \"dfma_tflops\": %.2f, "
         "\"dmma_m8n8k4_tflops\": %.2f, \"dmma_m16n8k16_tflops\": %.2f, "
         "\"copy_kernel_gbs\": %.1f, \"memcpy_d2d_gbs\": %.1f}\n",
         p.name, sms, clk, memclk, smemOptin, l2, p.regsPerMultiprocessor, p.major, p.minor,
         ffma_flop / t_ffma / 1e9, ffma2_flop / t_ffma2 / 1e9, dfma_flop / t_dfma / 1e9,
         d884_flop / t_d884 / 1e9, d16816_flop / t_d16816 / 1e9,
         2.0 * bytes / t_copy / 1e6, 2.0 * bytes / t_memcpy / 1e6);
  return 0;
}
