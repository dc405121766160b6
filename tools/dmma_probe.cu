// Probe: (1) verify the assumed per-thread fragment layout of
// mma.sync.aligned.m16n8k16.row.col.f64 (and m16n8k8, m8n8k4) against a host GEMM,
// (2) measure sustained DMMA throughput with many independent accumulator chains.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_probe tools/dmma_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>

__global__ void k_layout16(const double* A, const double* B, double* D) {
  // A 16x16 row-major, B 16x8 (B[k][n] row-major), D 16x8
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double a[8], b[4], c[4] = {0, 0, 0, 0};
  for (int i = 0; i < 4; ++i) {
    a[2 * i] = A[g * 16 + t + 4 * i];
    a[2 * i + 1] = A[(g + 8) * 16 + t + 4 * i];
    b[i] = B[(t + 4 * i) * 8 + g];
  }
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
               "{%12,%13,%14,%15}, {%0,%1,%2,%3};"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                 "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  D[g * 8 + 2 * t] = c[0];
  D[g * 8 + 2 * t + 1] = c[1];
  D[(g + 8) * 8 + 2 * t] = c[2];
  D[(g + 8) * 8 + 2 * t + 1] = c[3];
}

__global__ void k_layout8(const double* A, const double* B, double* D) {
  // A 16x8, B 8x8, D 16x8 (m16n8k8)
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double a[4], b[2], c[4] = {0, 0, 0, 0};
  for (int i = 0; i < 2; ++i) {
    a[2 * i] = A[g * 8 + t + 4 * i];
    a[2 * i + 1] = A[(g + 8) * 8 + t + 4 * i];
    b[i] = B[(t + 4 * i) * 8 + g];
  }
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
  D[g * 8 + 2 * t] = c[0];
  D[g * 8 + 2 * t + 1] = c[1];
  D[(g + 8) * 8 + 2 * t] = c[2];
  D[(g + 8) * 8 + 2 * t + 1] = c[3];
}

template <int CH>
__global__ void k_tput16(double* out, double a0, int iters) {
  double acc[CH][4];
#pragma unroll
  for (int c = 0; c < CH; ++c)
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[c][i] = 0.0;
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = a0 + 1e-3 * (threadIdx.x + i);
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = a0 - 1e-3 * (threadIdx.x + i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
                   "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(acc[c][0]), "+d"(acc[c][1]), "+d"(acc[c][2]), "+d"(acc[c][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c)
#pragma unroll
    for (int i = 0; i < 4; ++i) s += acc[c][i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int CH>
__global__ void k_tput884(double* out, double a0, int iters) {
  double acc[CH][2];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c][0] = acc[c][1] = 0.0;
  double av = a0 + 1e-3 * threadIdx.x, bv = a0 - 1e-3 * threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(av), "d"(bv));
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c][0] + acc[c][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  // ---- layout checks
  double hA[256], hB[128], hD[128], ref[128];
  srand(1);
  for (int i = 0; i < 256; ++i) hA[i] = (rand() % 17) - 8;
  for (int i = 0; i < 128; ++i) hB[i] = (rand() % 17) - 8;
  double *dA, *dB, *dD;
  cudaMalloc(&dA, sizeof hA); cudaMalloc(&dB, sizeof hB); cudaMalloc(&dD, sizeof hD);
  cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
  k_layout16<<<1, 32>>>(dA, dB, dD);
  cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost);
  double err16 = 0;
  for (int m = 0; m < 16; ++m)
    for (int nn = 0; nn < 8; ++nn) {
      double s = 0;
      for (int k = 0; k < 16; ++k) s += hA[m * 16 + k] * hB[k * 8 + nn];
      ref[m * 8 + nn] = s;
      err16 = fmax(err16, fabs(s - hD[m * 8 + nn]));
    }
  // m16n8k8 uses A as 16x8 (first 128 entries), B 8x8 (first 64)
  k_layout8<<<1, 32>>>(dA, dB, dD);
  cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost);
  double err8 = 0;
  for (int m = 0; m < 16; ++m)
    for (int nn = 0; nn < 8; ++nn) {
      double s = 0;
      for (int k = 0; k < 8; ++k) s += hA[m * 8 + k] * hB[k * 8 + nn];
      err8 = fmax(err8, fabs(s - hD[m * 8 + nn]));
    }
  cudaError_t e = cudaGetLastError();
  // ---- throughput
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, sizeof(double) * sms * 16 * 256);
  cudaEvent_t s0, s1;
  cudaEventCreate(&s0); cudaEventCreate(&s1);
  auto timeit = [&](auto kern, int blocks, int threads, int iters, double flop_per_warp_iter) {
    kern<<<blocks, threads>>>(out, 0.5, iters);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(s0);
      kern<<<blocks, threads>>>(out, 0.5, iters);
      cudaEventRecord(s1);
      cudaEventSynchronize(s1);
      float ms; cudaEventElapsedTime(&ms, s0, s1);
      best = fminf(best, ms);
    }
    const double warps = (double)blocks * threads / 32;
    return warps * iters * flop_per_warp_iter / (best * 1e-3) / 1e12;
  };
  const int it = 2048;
  double t16_4 = timeit(k_tput16<4>, sms * 4, 256, it, 4 * 4096.0);
  double t16_8 = timeit(k_tput16<8>, sms * 2, 256, it, 8 * 4096.0);
  double t16_2w = timeit(k_tput16<4>, sms * 1, 128, it, 4 * 4096.0);
  double t884_8 = timeit(k_tput884<8>, sms * 4, 256, it * 4, 8 * 512.0);
  printf("{\"err_m16n8k16\": %g, \"err_m16n8k8\": %g, \"cuda\": \"%s\", \"dmma16816_tflops_4ch\": %.2f, "
         "\"dmma16816_tflops_8ch\": %.2f, \"dmma16816_tflops_1cta_per_sm_4warps\": %.2f, \"dmma884_tflops_8ch\": %.2f}\n",
         err16, err8, cudaGetErrorString(e), t16_4, t16_8, t16_2w, t884_8);
  return 0;
}
