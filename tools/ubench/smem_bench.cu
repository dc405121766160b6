// Micro-benchmarks for the K1 redesign: shared-memory LDS.128 broadcast patterns,
// predicated STS.128, SHFL, redux.sync and FFMA2 throughput per SM (cycles / warp-instr).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 2048
#define WARPS 16

template <int PAT>
__device__ __forceinline__ uint32_t lds_addr(uint32_t base, int lane) {
  if (PAT == 0) return base;                                  // all same
  if (PAT == 1) return base + (lane >> 4) * 16;               // 2 groups, diff banks
  if (PAT == 2) return base + (lane >> 4) * 128;              // 2 groups, same banks
  if (PAT == 3) return base + (lane >> 3) * 16;               // 4 groups diff banks
  if (PAT == 4) return base + (lane >> 3) * 128;              // 4 groups same banks
  if (PAT == 5) return base + (lane >> 2) * 16;               // 8 groups diff banks
  if (PAT == 6) return base + lane * 16;                      // all distinct (512 B)
  if (PAT == 7) return base + (lane >> 4) * 16 + 0;           // = 1 (placeholder)
  return base;
}

template <int PAT>
__global__ void k_lds(float* out, long long* cyc) {
  __shared__ __align__(16) float s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i * 0.5f;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  uint32_t base = (uint32_t)__cvta_generic_to_shared(s) + warp * 1024 % 8192;
  uint32_t a = lds_addr<PAT>(base, lane);
  float acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < ITERS; ++i) {
    float x, y, z, w;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(x), "=f"(y), "=f"(z), "=f"(w) : "r"(a + (i & 7) * 256));
    acc0 += x; acc1 += y; acc2 += z; acc3 += w;
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 + acc1 + acc2 + acc3;
  if (lane == 0) cyc[blockIdx.x * WARPS + warp] = t1 - t0;
}

// predicated STS.128: NACT active lanes (distinct banks)
template <int NACT>
__global__ void k_sts(float* out, long long* cyc) {
  __shared__ __align__(16) float s[8192];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  uint32_t a = (uint32_t)__cvta_generic_to_shared(s) + warp * 2048 + lane * 16;
  bool p = lane < NACT;
  float v = lane;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < ITERS; ++i) {
    asm volatile("{.reg .pred q; setp.ne.b32 q, %5, 0; @q st.shared.v4.f32 [%0], {%1,%2,%3,%4};}"
                 :: "r"(a + (i & 3) * 512), "f"(v), "f"(v), "f"(v), "f"(v), "r"((int)p) : "memory");
  }
  long long t1 = clock64();
  __syncthreads();
  out[blockIdx.x * blockDim.x + threadIdx.x] = s[threadIdx.x];
  if (lane == 0) cyc[blockIdx.x * WARPS + warp] = t1 - t0;
}

__global__ void k_shfl(float* out, long long* cyc) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  float v0 = lane, v1 = lane + 1, v2 = lane + 2, v3 = lane + 3;
  int src = (lane * 7) & 31;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < ITERS; ++i) {
    v0 = __shfl_sync(0xffffffffu, v0, src); v1 = __shfl_sync(0xffffffffu, v1, src);
    v2 = __shfl_sync(0xffffffffu, v2, src); v3 = __shfl_sync(0xffffffffu, v3, src);
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = v0 + v1 + v2 + v3;
  if (lane == 0) cyc[blockIdx.x * WARPS + warp] = t1 - t0;
}

__global__ void k_redux(float* out, long long* cyc) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  unsigned v0 = lane * 3, v1 = lane * 5, v2 = lane * 7, v3 = lane * 11;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < ITERS; ++i) {
    v0 = __reduce_max_sync(0xffffffffu, v0) ^ lane; v1 = __reduce_max_sync(0xffffffffu, v1) ^ lane;
    v2 = __reduce_max_sync(0xffffffffu, v2) ^ lane; v3 = __reduce_max_sync(0xffffffffu, v3) ^ lane;
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)(v0 + v1 + v2 + v3);
  if (lane == 0) cyc[blockIdx.x * WARPS + warp] = t1 - t0;
}

// latency: one dependent chain
__global__ void k_redux_lat(float* out, long long* cyc) {
  const int lane = threadIdx.x & 31;
  unsigned v0 = lane * 3;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < ITERS; ++i) v0 = __reduce_max_sync(0xffffffffu, v0) ^ lane;
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)v0;
  if (lane == 0) cyc[0] = t1 - t0;
}
__global__ void k_lds_lat(float* out, long long* cyc) {
  __shared__ __align__(16) unsigned s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (i + 4) & 1023;
  __syncwarp();
  unsigned a = threadIdx.x & 31;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < ITERS; ++i) a = s[a];
  long long t1 = clock64();
  out[threadIdx.x] = (float)a;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void k_ffma2(float* out, long long* cyc) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  float a[16];
  for (int j = 0; j < 16; ++j) a[j] = lane + j;
  float f = 0.999f, y0 = 0.5f, y1 = 0.25f;
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 16; j += 2) {
      asm volatile("{.reg .b64 d, x, y, ff; mov.b64 x, {%0,%1}; mov.b64 y, {%3,%4}; mov.b64 ff, {%2,%2}; fma.rn.f32x2 d, ff, y, x; mov.b64 {%0,%1}, d;}"
                   : "+f"(a[j]), "+f"(a[j + 1]) : "f"(f), "f"(y0), "f"(y1));
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int j = 0; j < 16; ++j) s += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (lane == 0) cyc[blockIdx.x * WARPS + warp] = t1 - t0;
}

template <typename K>
void run(const char* name, K kern, int ninstr_per_iter, int warps) {
  float* out; long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * WARPS * 8);
  kern<<<148, warps * 32>>>(out, cyc);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<<<148, warps * 32>>>(out, cyc);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long h[148 * WARPS];
  cudaMemcpy(h, cyc, sizeof(long long) * 148 * warps, cudaMemcpyDeviceToHost);
  double mx = 0; for (int i = 0; i < warps; ++i) mx = h[i] > mx ? h[i] : mx;
  double per = mx / ((double)ITERS * ninstr_per_iter);   // cycles per instr per warp
  printf("%-28s warps/SM=%2d  cyc/instr/warp=%7.2f  => SM cyc per warp-instr=%6.3f  (%s, %.3f ms)\n", name, warps, per,
         per / warps, cudaGetErrorString(err), ms);
  cudaFree(out); cudaFree(cyc);
}

int main() {
  for (int w : {1, 16}) {
    run("LDS.128 all-same", k_lds<0>, 1, w);
    run("LDS.128 2grp diffbank", k_lds<1>, 1, w);
    run("LDS.128 2grp samebank", k_lds<2>, 1, w);
    run("LDS.128 4grp diffbank", k_lds<3>, 1, w);
    run("LDS.128 4grp samebank", k_lds<4>, 1, w);
    run("LDS.128 8grp diffbank", k_lds<5>, 1, w);
    run("LDS.128 32 distinct", k_lds<6>, 1, w);
    run("STS.128 0 active", k_sts<0>, 1, w);
    run("STS.128 1 active", k_sts<1>, 1, w);
    run("STS.128 2 active", k_sts<2>, 1, w);
    run("STS.128 8 active", k_sts<8>, 1, w);
    run("STS.128 32 active", k_sts<32>, 1, w);
    run("SHFL idx", k_shfl, 4, w);
    run("REDUX.MAX", k_redux, 4, w);
    run("FFMA2", k_ffma2, 8, w);
  }
  run("REDUX latency (1 warp chain)", k_redux_lat, 1, 1);
  run("LDS.32 latency (1 warp chain)", k_lds_lat, 1, 1);
  return 0;
}
