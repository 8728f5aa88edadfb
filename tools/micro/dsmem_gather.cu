// Microbenchmark: random 8-byte gathers from (a) local shared memory,
// (b) distributed shared memory across a cluster, (c) an L2-resident global
// vector.  Reports gathers per SM per cycle.  Build: nvcc -gencode
// arch=compute_100a,code=sm_100a -O3 -o dsmem_gather dsmem_gather.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;

constexpr int kWords = 16384;  // doubles per CTA smem (128 KB)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

template <int CL>
__global__ void __cluster_dims__(CL, 1, 1) gather_dsmem(int iters, double* out) {
    extern __shared__ double sm[];
    for (int i = threadIdx.x; i < kWords; i += blockDim.x) sm[i] = i * 1e-3;
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    double acc = 0;
    uint32_t h = hash32(blockIdx.x * 1024 + threadIdx.x);
    for (int it = 0; it < iters; ++it) {
#pragma unroll 8
        for (int k = 0; k < 8; ++k) {
            h = hash32(h + k);
            const int rank = (h >> 20) % CL;
            const int w = h % kWords;
            double* remote = cl.map_shared_rank(sm, rank);
            acc += remote[w];
        }
    }
    cl.sync();
    if (acc == 42.0) out[0] = acc;
}

__global__ void gather_local(int iters, double* out) {
    extern __shared__ double sm[];
    for (int i = threadIdx.x; i < kWords; i += blockDim.x) sm[i] = i * 1e-3;
    __syncthreads();
    double acc = 0;
    uint32_t h = hash32(blockIdx.x * 1024 + threadIdx.x);
    for (int it = 0; it < iters; ++it) {
#pragma unroll 8
        for (int k = 0; k < 8; ++k) {
            h = hash32(h + k);
            acc += sm[h % kWords];
        }
    }
    if (acc == 42.0) out[0] = acc;
}

__global__ void gather_global(int iters, const double* __restrict__ x, uint32_t n, double* out) {
    double acc = 0;
    uint32_t h = hash32(blockIdx.x * 1024 + threadIdx.x);
    for (int it = 0; it < iters; ++it) {
#pragma unroll 8
        for (int k = 0; k < 8; ++k) {
            h = hash32(h + k);
            acc += __ldg(x + (h % n));
        }
    }
    if (acc == 42.0) out[0] = acc;
}

int main() {
    double* out; cudaMalloc(&out, 8);
    double* x; uint32_t n = 4u << 20;  // 32 MB, L2-resident
    cudaMalloc(&x, (size_t)n * 8); cudaMemset(x, 0, (size_t)n * 8);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int iters = 2000, threads = 512, smem = kWords * 8;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto report = [&](const char* name, int blocks, float ms) {
        double gathers = (double)blocks * threads * iters * 8;
        double cyc = ms * 1e-3 * clk * 1e3;
        printf("%-22s blocks=%5d  %.3f ms  %.2f Ggather/s  %.3f gathers/SM/cycle(@%d MHz)\n", name, blocks, ms,
               gathers / ms / 1e6, gathers / 148.0 / cyc, clk / 1000);
    };
    cudaFuncSetAttribute(gather_local, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(gather_dsmem<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(gather_dsmem<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(gather_dsmem<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int rep = 0; rep < 2; ++rep) {
        float ms;
        cudaEventRecord(a); gather_local<<<148, threads, smem>>>(iters, out); cudaEventRecord(b);
        cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b); report("local smem", 148, ms);
        cudaEventRecord(a); gather_dsmem<2><<<148, threads, smem>>>(iters, out); cudaEventRecord(b);
        cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b); report("dsmem cluster=2", 148, ms);
        cudaEventRecord(a); gather_dsmem<4><<<144, threads, smem>>>(iters, out); cudaEventRecord(b);
        cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b); report("dsmem cluster=4", 144, ms);
        cudaEventRecord(a); gather_dsmem<8><<<144, threads, smem>>>(iters, out); cudaEventRecord(b);
        cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b); report("dsmem cluster=8", 144, ms);
        cudaEventRecord(a); gather_global<<<148 * 4, threads>>>(iters, x, n, out); cudaEventRecord(b);
        cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b); report("global L2 (32MB)", 148 * 4, ms);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
