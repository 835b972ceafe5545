// device_common.cuh -- sm_100a PTX helpers shared by the kernels.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace fpmm_b200 {
namespace dev {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// FP64 tensor-core MMA: D(8x8) += A(8x4, row) * B(4x8, col); lowers to DMMA.8x8x4.
// Lane t holds A[t/4][t%4], B[t%4][t/4], D[t/4][2(t%4)+{0,1}].
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// ---- mbarrier (shared::cta) ----
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra LAB_DONE;\n"
      "bra LAB_WAIT;\n"
      "LAB_DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Wait with a sleep between polls: for warps that wait whole MMA passes
// (epilogue), so the spin does not steal issue slots or power from the SM.
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
      "selp.u32 %0, 1, 0, P1;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity, unsigned ns) {
  while (!mbar_test(bar, parity)) __nanosleep(ns);
}

// ---- TMA 1-D bulk copy global -> shared, completion on an mbarrier ----
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ double2 lds128(const double* p) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(smem_u32(p)));
  return v;
}

// In-register reduction of an exact integer |x| <= 2^53 to |r| <= p/2 + 2:
// r = x - rint(x q) p, with rint from the 1.5*2^52 magic constant (single
// rounding of the fma; |x q| < 2^51).  All three ops are exact or correctly
// rounded; r is an integer below 2^52 so the final fma is exact.
__device__ __forceinline__ double reduce_signed(double x, double p, double q) {
#if FPMM_B200_RINT_REDUCE
  const double c = rint(x * q);
#else
  const double M = 6755399441055744.0;  // 1.5 * 2^52
  const double c = __fma_rn(x, q, M) - M;
#endif
  return __fma_rn(-c, p, x);
}

// (t * w) mod p for t < 2^64, w < p < 2^63 with Shoup's precomputed
// ws = floor(w 2^64 / p); result in [0, p).
__device__ __forceinline__ uint64_t shoup_mulmod(uint64_t t, uint64_t w, uint64_t ws, uint64_t p) {
  const uint64_t qh = __umul64hi(t, ws);
  uint64_t r = t * w - qh * p;
  return r >= p ? r - p : r;
}

}  // namespace dev
}  // namespace fpmm_b200
