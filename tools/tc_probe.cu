// Probe: one tcgen05.mma kind::tf32 tile (M = 128, N = 128, K = 128) with TMA-loaded
// K-major 128-byte-swizzled operands and the accumulator in TMEM, read back with
// tcgen05.ld — checks the descriptor encodings used by the library's TF32 path against a
// host reference (small integers: exact in tf32).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tc_probe tools/tc_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc_k_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3fff);          // start address
  d |= (uint64_t)1 << 16;                          // LBO = 16 B (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;                // SBO = 1024 B between 8-row groups
  d |= (uint64_t)1 << 46;                          // version (sm100)
  d |= (uint64_t)2 << 61;                          // SWIZZLE_128B
  return d;
}

constexpr int M = 128, N = 128, K = 128, KB = 32;

__global__ void k_probe(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, float* D) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* sA = base;                       // [K/KB][M][KB] fp32
  unsigned char* sB = base + (K / KB) * M * KB * 4;
  __shared__ uint64_t bar_tma, bar_mma;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar_tma)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar_mma)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar_tma)), "r"((M + N) * K * 4));
    for (int kb = 0; kb < K / KB; ++kb) {
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(smem_u32(sA + kb * M * KB * 4)), "l"(&ta), "r"(kb * KB), "r"(0), "r"(smem_u32(&bar_tma)) : "memory");
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(smem_u32(sB + kb * N * KB * 4)), "l"(&tb), "r"(kb * KB), "r"(0), "r"(smem_u32(&bar_tma)) : "memory");
    }
  }
  {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{ .reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0; selp.u32 %0, 1, 0, P; }"
                   : "=r"(ok) : "r"(smem_u32(&bar_tma)) : "memory");
  }
  if (tid == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    // instruction descriptor: D f32, A/B tf32, K-major both, N >> 3, M >> 4
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    for (int kb = 0; kb < K / KB; ++kb) {
      for (int kk = 0; kk < KB / 8; ++kk) {
        const uint64_t ad = desc_k_sw128(smem_u32(sA + kb * M * KB * 4) + kk * 32);
        const uint64_t bd = desc_k_sw128(smem_u32(sB + kb * N * KB * 4) + kk * 32);
        const uint32_t acc = (kb | kk) ? 1u : 0u;
        asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p; }"
                     ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar_mma)) : "memory");
  }
  {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{ .reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0; selp.u32 %0, 1, 0, P; }"
                   : "=r"(ok) : "r"(smem_u32(&bar_mma)) : "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int row = warp * 32 + (tid & 31);
  for (int c = 0; c < N; c += 8) {
    uint32_t v[8];
    const uint32_t ta_ = tmem + ((uint32_t)(warp * 32) << 16) + c;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(ta_));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 8; ++j) D[row * N + c + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  std::vector<float> A(M * K), B(N * K), D(M * N);
  srand(1);
  for (auto& a : A) a = (float)(rand() % 7 - 3);
  for (auto& b : B) b = (float)(rand() % 7 - 3);
  float *dA, *dB, *dD;
  CK(cudaMalloc(&dA, A.size() * 4)); CK(cudaMalloc(&dB, B.size() * 4)); CK(cudaMalloc(&dD, D.size() * 4));
  CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q));
  EncodeFn enc = (EncodeFn)fp;
  CUtensorMap ta, tb;
  cuuint64_t dimsA[2] = {K, M}, strA[1] = {K * 4};
  cuuint64_t dimsB[2] = {K, N}, strB[1] = {K * 4};
  cuuint32_t boxA[2] = {KB, M}, boxB[2] = {KB, N}, es[2] = {1, 1};
  if (enc(&ta, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dA, dimsA, strA, boxA, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS ||
      enc(&tb, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dB, dimsB, strB, boxB, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    printf("encode failed\n");
    return 1;
  }
  const int smem = (M + N) * K * 4 + 1024;
  CK(cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  k_probe<<<1, 128, smem>>>(ta, tb, dD);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  double maxerr = 0;
  int bad = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      double r = 0;
      for (int k = 0; k < K; ++k) r += (double)A[i * K + k] * B[j * K + k];
      const double e = fabs(r - D[i * N + j]);
      if (e > maxerr) maxerr = e;
      if (e > 0 && bad < 5) { printf("mismatch (%d,%d): got %f want %f\n", i, j, D[i * N + j], r); ++bad; }
    }
  printf("tcgen05 tf32 probe: max abs err %g %s\n", maxerr, maxerr == 0 ? "EXACT" : "WRONG");
  return maxerr == 0 ? 0 : 2;
}
