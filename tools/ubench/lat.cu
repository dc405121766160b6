// Dependent-chain latency (1 warp) and issue throughput (16 warps/SM) of the warp-collective
// and MIO operations the batched pivot chain is built from (sm_100a):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench/lat tools/ubench/lat.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITERS = 512;

template <int OP>
__device__ __forceinline__ uint32_t step(uint32_t v, int lane, const uint32_t* sm) {
  if constexpr (OP == 0) return __reduce_max_sync(0xffffffffu, v) + lane;                 // CREDUX.MAX + add
  if constexpr (OP == 1) return __shfl_sync(0xffffffffu, v, (v + lane) & 31) + 1;          // SHFL.IDX + add
  if constexpr (OP == 2) return max(v, __shfl_xor_sync(0xffffffffu, v, 1)) + 1;            // SHFL.BFLY + max + add
  if constexpr (OP == 3) return __ballot_sync(0xffffffffu, (v & 1) != 0) + v;              // VOTE + add
  if constexpr (OP == 4) return (v + 1) ^ lane;                                            // 2 ALU ops
  if constexpr (OP == 5) return sm[(v + lane) & 255] + 1;                                  // LDS + add
  if constexpr (OP == 6) return __float_as_uint(__frcp_rn(__uint_as_float(v | 0x3f800000u))) + 1;
  if constexpr (OP == 7) {
    float r; asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(__uint_as_float(v | 0x3f800000u)));
    return __float_as_uint(r) + 1;
  }
  if constexpr (OP == 8) {  // group max for two 16-lane groups (the K1b pattern)
    const int g = lane >> 4;
    const uint32_t a = __reduce_max_sync(0xffffffffu, g == 0 ? v : 0u);
    const uint32_t b = __reduce_max_sync(0xffffffffu, g == 1 ? v : 0u);
    return (g ? b : a) + lane;
  }
  if constexpr (OP == 9) {  // 16-lane butterfly max (4 levels)
    v = max(v, __shfl_xor_sync(0xffffffffu, v, 1));
    v = max(v, __shfl_xor_sync(0xffffffffu, v, 2));
    v = max(v, __shfl_xor_sync(0xffffffffu, v, 4));
    v = max(v, __shfl_xor_sync(0xffffffffu, v, 8));
    return v + lane;
  }
  if constexpr (OP == 10) {  // 8-lane butterfly max (3 levels)
    v = max(v, __shfl_xor_sync(0xffffffffu, v, 1));
    v = max(v, __shfl_xor_sync(0xffffffffu, v, 2));
    v = max(v, __shfl_xor_sync(0xffffffffu, v, 4));
    return v + lane;
  }
  if constexpr (OP == 11) {  // redux with a per-group (non-uniform) member mask
    const unsigned gm = 0xffffu << (lane & 16);
    return __reduce_max_sync(gm, v) + lane;
  }
  return v;
}

template <int OP>
__global__ void chain(uint32_t* out, long long* cyc) {
  __shared__ uint32_t sm[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) sm[i] = i * 7u;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  uint32_t v = lane;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < ITERS; ++i) v = step<OP>(v, lane, sm);
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = v;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

template <int OP>
void run(const char* name, uint32_t* out, long long* cyc, int sms) {
  long long c;
  chain<OP><<<1, 32>>>(out, cyc);
  cudaDeviceSynchronize();
  chain<OP><<<1, 32>>>(out, cyc);
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double lat = (double)c / ITERS;
  // throughput: 16 warps per SM, every SM
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  chain<OP><<<sms * 4, 128>>>(out, cyc);
  cudaEventRecord(a);
  for (int r = 0; r < 10; ++r) chain<OP><<<sms * 4, 128>>>(out, cyc);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double cycles = ms / 10 * 1e-3 * clk * 1e3;
  const double per_sm_warp_ops = (double)16 * ITERS;   // warp-steps per SM
  printf("%-28s latency %6.1f cyc/step   16 warps/SM: %6.2f cyc per warp-step per SM\n", name, lat,
         cycles / per_sm_warp_ops);
}

// throughput with 4 independent chains per warp (32 warps/SM)
template <int OP>
__global__ void tp4(uint32_t* out) {
  const int lane = threadIdx.x & 31;
  uint32_t v0 = lane, v1 = lane * 3, v2 = lane * 5, v3 = lane * 7;
#pragma unroll 8
  for (int i = 0; i < ITERS; ++i) {
    if constexpr (OP == 0) {
      v0 = __reduce_max_sync(0xffffffffu, v0) ^ lane; v1 = __reduce_max_sync(0xffffffffu, v1) ^ lane;
      v2 = __reduce_max_sync(0xffffffffu, v2) ^ lane; v3 = __reduce_max_sync(0xffffffffu, v3) ^ lane;
    } else if constexpr (OP == 1) {
      v0 = __shfl_sync(0xffffffffu, v0, v3 & 31) ^ lane; v1 = __shfl_sync(0xffffffffu, v1, v0 & 31) ^ lane;
      v2 = __shfl_sync(0xffffffffu, v2, v1 & 31) ^ lane; v3 = __shfl_sync(0xffffffffu, v3, v2 & 31) ^ lane;
    } else {
      v0 = __ballot_sync(0xffffffffu, v0 & 1) ^ lane; v1 = __ballot_sync(0xffffffffu, v1 & 1) ^ lane;
      v2 = __ballot_sync(0xffffffffu, v2 & 1) ^ lane; v3 = __ballot_sync(0xffffffffu, v3 & 1) ^ lane;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = v0 + v1 + v2 + v3;
}
template <int OP>
void runtp(const char* name, uint32_t* out, int sms) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  tp4<OP><<<sms * 4, 256>>>(out);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) tp4<OP><<<sms * 4, 256>>>(out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double cycles = ms / 5 * 1e-3 * clk * 1e3;
  printf("%-28s throughput %6.2f SM cycles per warp op (32 warps/SM, 4 chains)\n", name, cycles / (32.0 * ITERS * 4));
}

int main() {
  uint32_t* out;
  long long* cyc;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaMalloc(&out, sms * 4 * 128 * 4);
  cudaMalloc(&cyc, 8);
  run<0>("redux.max + iadd", out, cyc, sms);
  run<1>("shfl.idx + iadd", out, cyc, sms);
  run<2>("shfl.bfly + max + iadd", out, cyc, sms);
  run<3>("vote.ballot + iadd", out, cyc, sms);
  run<4>("iadd + lop (2 alu)", out, cyc, sms);
  run<5>("lds + iadd", out, cyc, sms);
  run<6>("rcp.rn.f32 + iadd", out, cyc, sms);
  run<7>("rcp.approx + iadd", out, cyc, sms);
  run<8>("2-group redux (K1b)", out, cyc, sms);
  run<9>("16-lane butterfly (4 lv)", out, cyc, sms);
  run<10>("8-lane butterfly (3 lv)", out, cyc, sms);
  run<11>("redux, per-group mask", out, cyc, sms);
  uint32_t* o2;
  cudaMalloc(&o2, sms * 4 * 256 * 4);
  runtp<0>("redux.max", o2, sms);
  runtp<1>("shfl.idx", o2, sms);
  runtp<2>("vote.ballot", o2, sms);
  return 0;
}
