// Probe: tcgen05.mma kind::tf32 with M = 128, N = 32, K = 32, A K-major (128-byte swizzle)
// and B MN-major (128-byte swizzle, N contiguous), both written to shared memory by plain
// stores with the swizzle applied by hand; accumulator in TMEM, read back by tcgen05.ld.
// Also checks accumulate-onto-initial-TMEM contents (tcgen05.st first).  Validates the
// operand layouts a batched n = 32 tensor-core elimination would use.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tc_probe_mn tools/tc_probe_mn.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3fff);
  d |= (uint64_t)((lbo >> 4) & 0x3fff) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3fff) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

constexpr int M = 128, N = 32, K = 32;

// byte offset of element (r, c) in a [rows][32 x 4 B] array with the 128-byte swizzle
__device__ __forceinline__ uint32_t sw128(int r, int c) {
  return (uint32_t)(r * 128 + ((((c * 4) >> 4) ^ (r & 7)) << 4) + ((c * 4) & 15));
}

__global__ void k_probe(const float* A, const float* B, const float* C0, float* D, int bmajor_mn, int lbo, int sbo_b) {
  __shared__ __align__(1024) unsigned char sA[M * 128];
  __shared__ __align__(1024) unsigned char sB[K * 128];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // A: row m = tid, 32 K values
  for (int k = 0; k < K; ++k) *reinterpret_cast<float*>(sA + sw128(tid, k)) = A[tid * K + k];
  // B: MN-major: K rows of N = 32 contiguous (row k), or K-major: N rows of K
  if (tid < 32) {
    for (int c = 0; c < 32; ++c) {
      if (bmajor_mn) *reinterpret_cast<float*>(sB + sw128(tid, c)) = B[tid * N + c];        // row k = tid, n = c
      else *reinterpret_cast<float*>(sB + sw128(tid, c)) = B[c * N + tid];                   // row n = tid, k = c
    }
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  // initial accumulator: C0 row tid
  {
    uint32_t v[32];
    for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(C0[tid * N + j]);
    const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16);
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
        ::"r"(ta), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
          "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]),
          "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]),
          "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(bmajor_mn ? 1 : 0) << 16) |
                           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    for (int kk = 0; kk < K / 8; ++kk) {
      const uint64_t ad = desc_sw128(smem_u32(sA) + kk * 32, 16, 1024);
      const uint64_t bd = bmajor_mn ? desc_sw128(smem_u32(sB) + kk * 1024, lbo, sbo_b)
                                    : desc_sw128(smem_u32(sB) + kk * 32, 16, 1024);
      asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p; }"
                   ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(1));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
  }
  {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{ .reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0; selp.u32 %0, 1, 0, P; }"
                   : "=r"(ok) : "r"(smem_u32(&bar)) : "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  {
    uint32_t v[8];
    for (int c = 0; c < N; c += 8) {
      const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + c;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                   : "r"(ta));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      for (int j = 0; j < 8; ++j) D[tid * N + c + j] = __uint_as_float(v[j]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

int main() {
  std::vector<float> A(M * K), B(K * N), C0(M * N), D(M * N);
  srand(3);
  for (auto& a : A) a = (float)(rand() % 7 - 3);
  for (auto& b : B) b = (float)(rand() % 7 - 3);
  for (auto& c : C0) c = (float)(rand() % 5 - 2);
  float *dA, *dB, *dC, *dD;
  CK(cudaMalloc(&dA, A.size() * 4)); CK(cudaMalloc(&dB, B.size() * 4)); CK(cudaMalloc(&dC, C0.size() * 4));
  CK(cudaMalloc(&dD, D.size() * 4));
  CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dC, C0.data(), C0.size() * 4, cudaMemcpyHostToDevice));
  struct V { int mn, lbo, sbo; } vs[] = {{0, 16, 1024}, {1, 16, 1024}, {1, 1024, 16}, {1, 0, 1024}, {1, 1024, 1024}};
  for (auto v : vs) {
    CK(cudaMemset(dD, 0, D.size() * 4));
    k_probe<<<1, 128>>>(dA, dB, dC, dD, v.mn, v.lbo, v.sbo);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
    double maxerr = 0;
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j) {
        double r = C0[i * N + j];
        for (int k = 0; k < K; ++k) r += (double)A[i * K + k] * B[k * N + j];
        maxerr = fmax(maxerr, fabs(r - D[i * N + j]));
      }
    printf("B %s-major lbo=%d sbo=%d: max abs err %g %s\n", v.mn ? "MN" : "K", v.lbo, v.sbo, maxerr, maxerr == 0 ? "EXACT" : "WRONG");
  }
  return 0;
}
