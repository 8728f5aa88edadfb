// tma.cuh -- mbarrier and TMA (cp.async.bulk.tensor) primitives for sm_100a.
#pragma once
#include <cstdint>

namespace rlb {
namespace tmaop {

__device__ __forceinline__ uint32_t sptr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sptr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sptr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred P;\n"
        "RLB_TMAOP_WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
        " @!P bra RLB_TMAOP_WAIT_%=;\n}" ::"r"(sptr(b)),
        "r"(parity)
        : "memory");
}
// 3D box load into shared memory, completing `bar`'s transaction count.
__device__ __forceinline__ void tma3d(void* dst, const void* map, uint64_t* bar, int x, int y, int z) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
        "[%2];" ::"r"(sptr(dst)),
        "l"(map), "r"(sptr(bar)), "r"(x), "r"(y), "r"(z)
        : "memory");
}

}  // namespace tmaop
}  // namespace rlb
