// cp.async.bulk (1D) global->shared streaming bandwidth vs chunk size and
// stages in flight (one elected thread issues, all threads wait).
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t sptr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void stream_bulk(const uint8_t* __restrict__ src, size_t total, uint32_t chunk, int stages, double* sink) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + (size_t)stages * chunk);
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sptr(bar + s)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const size_t per_cta = (total / gridDim.x) / chunk * chunk;
    const uint8_t* base = src + per_cta * blockIdx.x;
    const int n = (int)(per_cta / chunk);
    auto issue = [&](int k) {
        uint64_t* b = bar + (k % stages);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sptr(b)), "r"(chunk) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(sptr(smem + (size_t)(k % stages) * chunk)), "l"(base + (size_t)k * chunk), "r"(chunk), "r"(sptr(b)) : "memory");
    };
    if (threadIdx.x == 0) for (int k = 0; k < stages && k < n; ++k) issue(k);
    double acc = 0;
    for (int k = 0; k < n; ++k) {
        asm volatile("{\n .reg .pred P;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra W_%=;\n}"
                     ::"r"(sptr(bar + (k % stages))), "r"((k / stages) & 1) : "memory");
        acc += reinterpret_cast<const double*>(smem + (size_t)(k % stages) * chunk)[threadIdx.x % (chunk / 8)];
        __syncthreads();
        if (threadIdx.x == 0 && k + stages < n) issue(k + stages);
    }
    if (acc == 42.0) sink[0] = acc;
}

int main() {
    size_t total = 2ull << 30;
    uint8_t* src; cudaMalloc(&src, total); cudaMemset(src, 0, total);
    double* sink; cudaMalloc(&sink, 8);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaFuncSetAttribute(stream_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int ctas : {148, 296}) for (uint32_t chunk : {4096u, 16384u, 32768u}) for (int stages : {2, 3, 4, 6}) {
        size_t sm = (size_t)stages * chunk + 64;
        if (sm > 200 * 1024 || (ctas == 296 && sm > 100 * 1024)) continue;
        for (int t : {256, 1024}) {
            stream_bulk<<<ctas, t, sm>>>(src, total, chunk, stages, sink);
            cudaEventRecord(a);
            stream_bulk<<<ctas, t, sm>>>(src, total, chunk, stages, sink);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            printf("ctas %d threads %4d chunk %6u stages %d: %7.1f GB/s\n", ctas, t, chunk, stages, (double)((total / ctas) / chunk * chunk * ctas) / ms / 1e6);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
