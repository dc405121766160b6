// Shared-memory wavefronts per LDS.128 / STS for broadcast patterns (read with ncu:
// l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum / smsp__inst_executed_op_shared_ld.sum).
#include <cstdio>
#include <cuda_runtime.h>
template <int PAT>
__global__ void k(float* out) {
  __shared__ __align__(16) float s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  int off;
  if (PAT == 0) off = 0;                       // all 32 lanes one address
  else if (PAT == 1) off = (lane >> 4) * 112;  // two half-warps, two addresses (distinct banks)
  else if (PAT == 2) off = (lane >> 3) * 112;  // four quarter-warps
  else if (PAT == 3) off = lane * 4;           // all distinct (512 B)
  else if (PAT == 4) off = (lane >> 4) * 4;    // two half-warps, adjacent 16-byte chunks
  else if (PAT == 5) off = (lane >> 4) * 8;    // two half-warps, 32 bytes apart
  else off = (lane >> 4) * 16;                 // two half-warps, 64 bytes apart (same 128-B line)
  float a = 0;
  for (int i = 0; i < 1024; ++i) {
    float4 v; asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"((unsigned)__cvta_generic_to_shared(s + ((off + (i & 7) * 32) & 4095))));
    a += v.x + v.y + v.z + v.w;
  }
  out[threadIdx.x] = a;
}
int main() {
  float* o; cudaMalloc(&o, 4096);
  k<0><<<1, 32>>>(o); k<1><<<1, 32>>>(o); k<2><<<1, 32>>>(o); k<3><<<1, 32>>>(o); k<4><<<1, 32>>>(o); k<5><<<1, 32>>>(o); k<6><<<1, 32>>>(o);
  cudaDeviceSynchronize(); printf("ok\n"); return 0;
}
