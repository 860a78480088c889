// ek_tma.cuh -- one-dimensional bulk asynchronous copies (the TMA engine's
// cp.async.bulk global -> shared) completed on an mbarrier: a single lane arms the barrier
// with the byte count and issues the copy; the warp waits on the barrier's phase parity
// before reading the data.  Addresses and sizes must be multiples of 16 bytes.
#pragma once
#include <cuda_runtime.h>

namespace ekb {

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// makes the initialisation visible to the async proxy (the TMA unit)
__device__ __forceinline__ void mbar_init_fence() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
// orders this thread's (and, after a __syncwarp, the warp's) earlier generic-proxy accesses to
// shared memory before later async-proxy writes (a bulk copy into a buffer just read)
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// one lane: expect `bytes` on `bar` (one arrival) and copy [src, src + bytes) to dst
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// wait until the barrier's phase with this parity has completed
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{ .reg .pred p;\n"
      "EKB_MBAR_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra EKB_MBAR_WAIT_%=;\n"
      "}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

}  // namespace ekb
