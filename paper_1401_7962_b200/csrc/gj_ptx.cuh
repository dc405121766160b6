// Device-side PTX helpers shared by the libgjinv kernels (sm_100a): shared-memory
// addresses, mbarriers, TMA (cp.async.bulk.tensor) loads/stores, bulk async groups,
// proxy fences, FFMA2 (fma.rn.f32x2) and reciprocals.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace gj {
namespace ptx {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// All lanes wait, then reconverge (the per-lane try_wait loop may exit at different
// iterations; everything after it relies on a converged warp).
__device__ __forceinline__ void mbar_wait_warp(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
  __syncwarp();
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, int c0, int r0, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(r0), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* tm, int c0, int r0, const void* src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(tm)),
               "r"(c0), "r"(r0), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void bulk_prefetch_l2(const void* g, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(g), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

// x0,x1 += nf * (y0,y1) as one FFMA2 (fma.rn.f32x2, sm_100+).
__device__ __forceinline__ void ffma2(float& x0, float& x1, float nf, float y0, float y1) {
  unsigned long long xv, yv, fv;
  asm("mov.b64 %0, {%1,%2};" : "=l"(xv) : "f"(x0), "f"(x1));
  asm("mov.b64 %0, {%1,%2};" : "=l"(yv) : "f"(y0), "f"(y1));
  asm("mov.b64 %0, {%1,%1};" : "=l"(fv) : "f"(nf));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(xv) : "l"(fv), "l"(yv));
  asm("mov.b64 {%0,%1}, %2;" : "=f"(x0), "=f"(x1) : "l"(xv));
}

// 1/p: MUFU approximation + one Newton step (branch-free, within 1 ulp; exact for powers
// of two).  fp64 keeps the IEEE round-to-nearest reciprocal.
__device__ __forceinline__ float rcp(float p) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(p));
  const float e = fmaf(-p, r, 1.0f);
  return fmaf(r, e, r);
}
__device__ __forceinline__ double rcp(double p) { return __drcp_rn(p); }

// Largest T <= t (t >= 0), so that |p| <= tau is decided exactly in T's precision.
__device__ __forceinline__ float round_down_to(double t, float) { return __double2float_rd(t); }
__device__ __forceinline__ double round_down_to(double t, double) { return t; }

// Predicated vector store to shared memory without a branch.
__device__ __forceinline__ void st_shared_v4_if(bool pred, uint32_t addr, float a, float b, float c, float d) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %0, 0;\n\t@p st.shared.v4.f32 [%1], {%2, %3, %4, %5};\n}" ::"r"(
          pred ? 1u : 0u),
      "r"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
      : "memory");
}
__device__ __forceinline__ void st_shared_v2_if(bool pred, uint32_t addr, double a, double b) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %0, 0;\n\t@p st.shared.v2.f64 [%1], {%2, %3};\n}" ::"r"(
                   pred ? 1u : 0u),
               "r"(addr), "d"(a), "d"(b)
               : "memory");
}

}  // namespace ptx
}  // namespace gj
