// kt_async.cuh -- mbarrier / bulk-async-copy helpers (sm_100a PTX) shared by
// the tcgen05 GEMM (kt_gemm.cu) and the shared-memory-staged LSTM cell
// (kt_kernels.cu).
#pragma once

#include <cstdint>

namespace kt {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(n) : "memory");
}
// arrive (count 1) and raise the phase's expected transaction bytes
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
// wait for the phase of parity `phase` to complete
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t phase) {
  uint32_t ok = 0;
  for (uint32_t spin = 0;; ++spin) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok) : "r"(a), "r"(phase) : "memory");
    if (ok) return;
    if (spin > (1u << 26)) __trap();   // never hang the GPU on a protocol bug
  }
}

// 1-D bulk copy global -> shared (TMA engine), completion counted in bytes on
// the mbarrier.  dst, src 16-B aligned; bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(mbar)
      : "memory");
}

}  // namespace kt
