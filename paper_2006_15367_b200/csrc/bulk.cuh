// Blackwell / Hopper bulk asynchronous copies (the TMA unit's 1-D mode):
// cp.async.bulk global -> shared with mbarrier completion (SASS UBLKCP) and
// cp.async.bulk.prefetch.L2 (SASS UBLKPF).  Used by the fused M2M / L2L
// kernels (interp_fused.cuh) to stage contiguous per-parent blocks without
// per-thread address arithmetic and to pull the next parent's data into L2
// while the current one computes.
#ifndef HFMM_B200_BULK_CUH
#define HFMM_B200_BULK_CUH

#include <cstdint>

namespace hfmm_b200 {
namespace bulk {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}

// Makes mbarrier initialisations visible to the asynchronous proxy (before the
// first bulk copy that signals them); follow with a CTA barrier.
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

// Orders earlier generic-proxy accesses of shared memory (reads of a buffer,
// writes of a staged result) before later asynchronous-proxy accesses (a bulk
// copy that overwrites or reads the same bytes).
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

// Arrive (one thread) announcing `bytes` of transaction on the barrier.
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}

// Block until the barrier's phase `parity` has completed.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

// dst (shared) <- src (global), `bytes` a multiple of 16, both 16-byte aligned;
// completion is signalled on `bar` (complete_tx).
__device__ __forceinline__ void copy_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

// dst (global) <- src (shared), `bytes` a multiple of 16, as one bulk-group entry.
__device__ __forceinline__ void copy_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst), "r"(smem_addr(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void commit_group() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
// Waits until the bulk groups of this thread have finished READING their shared source.
__device__ __forceinline__ void wait_group_read0() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }

// Hint: bring [src, src + bytes) into L2 (bytes a multiple of 16).
__device__ __forceinline__ void prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}

}  // namespace bulk
}  // namespace hfmm_b200

#endif
