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
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sptr(b)) : "memory");
}
// try_wait with a suspend-time hint (ns): the waiting warp sleeps instead of spinning.
__device__ __forceinline__ void mbar_wait_hint(uint64_t* b, uint32_t parity, uint32_t hint_ns) {
    asm volatile(
        "{\n .reg .pred P;\n"
        "RLB_TMAOP_WAITH_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1, %2;\n"
        " @!P bra RLB_TMAOP_WAITH_%=;\n}" ::"r"(sptr(b)),
        "r"(parity), "r"(hint_ns)
        : "memory");
}
// 2D box load into shared memory, completing `bar`'s transaction count.
__device__ __forceinline__ void tma2d(void* dst, const void* map, uint64_t* bar, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            sptr(dst)),
        "l"(map), "r"(sptr(bar)), "r"(x), "r"(y)
        : "memory");
}
// 1D bulk copy global -> shared with an L2 cache policy.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
            "r"(sptr(dst)),
        "l"(src), "r"(bytes), "r"(sptr(bar)), "l"(pol)
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

// Ring of S shared-memory stages of STAGE doubles, followed by S full and S
// empty mbarriers.  One producer thread fills stage k % S; consumer warps
// release it with one arrive per warp.
template <int S, int STAGE>
struct Ring {
    double* base;
    uint64_t* full;
    uint64_t* empty;
    __device__ Ring(double* smem) : base(smem) {
        full = reinterpret_cast<uint64_t*>(smem + S * STAGE);
        empty = full + S;
    }
    __device__ double* stage(int k) const { return base + (k % S) * STAGE; }
    __device__ void init(int consumers) {
        if (threadIdx.x == 0) {
            for (int s = 0; s < S; ++s) {
                mbar_init(full + s, 1);
                mbar_init(empty + s, consumers);
            }
            mbar_fence_init();
        }
        __syncthreads();
    }
    __device__ void wait_full(int k) { mbar_wait(full + (k % S), (uint32_t)((k / S) & 1)); }
    // One arrive per warp once the whole warp has finished reading stage k.
    __device__ void release(int k) {
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(empty + (k % S));
    }
    // Producer: before refilling the stage that held item k, wait until every
    // consumer warp released item k.
    __device__ void wait_empty(int k) { mbar_wait(empty + (k % S), (uint32_t)((k / S) & 1)); }
    // Producer: fill stage k with a 2D box of `bytes`.
    __device__ void issue2d(int k, const void* map, int x, int y, uint32_t bytes) {
        uint64_t* bar = full + (k % S);
        mbar_expect_tx(bar, bytes);
        tma2d(stage(k), map, bar, x, y);
    }
};

}  // namespace tmaop
}  // namespace rlb
