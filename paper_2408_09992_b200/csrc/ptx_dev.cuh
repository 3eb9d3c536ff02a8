// ptx_dev.cuh — mbarrier / TMA bulk-copy helpers shared by the K2 kernels
// (sm_100a; the asynchronous copies complete on an mbarrier transaction count).
#pragma once
#include <stdint.h>
#include <cstdio>

namespace pq {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(bytes) : "memory");
}
#ifndef PQTOPK_CHECKED
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}"
        :: "r"(bar), "r"(parity) : "memory");
}
#else
// checked builds: a bounded wait (a lost TMA completion traps instead of hanging)
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    for (long long n = 0;; ++n) {
        uint32_t ok;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n}"
            : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
        if (ok) return;
        if (n > (1ll << 26)) {
            printf("PQ_DCHECK failed: mbarrier wait timed out (block %d thread %d)\n", (int)blockIdx.x,
                   (int)threadIdx.x);
            __trap();
        }
    }
}
#endif
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        :: "r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
// Programmatic dependent launch (PDL): a kernel launched with launch_pdl() may
// start while its stream predecessor is still running; pdl_wait() blocks until
// the predecessor has completed and its writes are visible, and must precede
// every access to memory a predecessor writes.  pdl_trigger() lets this
// kernel's own dependent be scheduled early.  Both are no-ops without PDL.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

}  // namespace pq
