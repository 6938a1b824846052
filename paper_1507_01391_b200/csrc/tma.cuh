// tma.cuh -- the Blackwell bulk-copy (TMA) and mbarrier primitives the batch kernels use to
// stream instances between HBM and shared memory without registers: cp.async.bulk global ->
// shared with mbarrier complete_tx, L2 prefetch of the next instance, parity waits.
#pragma once

#include <cstdint>

namespace dmmdev {

__device__ __forceinline__ uint32_t sptr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sptr(bar)) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tma_load(uint32_t* dst, const uint32_t* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sptr(bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(sptr(dst)), "l"(src), "r"(bytes), "r"(sptr(bar))
                 : "memory");
}
// the same load split into `parts` bulk copies issued by lanes 0 .. parts-1 of the calling warp
// (several copies in flight instead of one long one); the whole warp calls it
__device__ __forceinline__ void tma_load_split(uint32_t* dst, const uint32_t* src, uint32_t bytes, uint64_t* bar,
                                               int lane, int parts) {
    if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sptr(bar)), "r"(bytes) : "memory");
    __syncwarp();
    const uint32_t part = bytes / parts;
    if (lane < parts)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(sptr(dst + lane * (part / 4))), "l"(src + lane * (part / 4)), "r"(part), "r"(sptr(bar))
                     : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(sptr(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void prefetch_l2(const uint32_t* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// shared -> global bulk copy (one bulk group), and the wait until its source has been read
__device__ __forceinline__ void tma_store(uint32_t* dst, const uint32_t* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(sptr(src)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// the same store with an L2 evict-first policy: the result streams out without displacing the
// inputs prefetched into L2 for the next machines
__device__ __forceinline__ void tma_store_evict_first(uint32_t* dst, const uint32_t* src, uint32_t bytes) {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
                 "r"(sptr(src)), "r"(bytes), "l"(pol)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }


}  // namespace dmmdev
