// SM-driven PCIe copies (zero-copy loads from / stores to pinned host memory)
// against copy-engine copies: 32 MiB H2D, 32 MiB D2H, both at once.  Does
// the SM path avoid the copy engines' ~7 us per-piece cost and reach the
// bidirectional rate the e2e SpMV pipeline needs?
#include <cstdio>
#include <cuda_runtime.h>

__global__ void copy_kernel(const int4* __restrict__ src, int4* __restrict__ dst, size_t n16, int unroll_dummy) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n16; i += 4 * stride) {
        int4 a = src[i], b = src[i + stride], c = src[i + 2 * stride], d = src[i + 3 * stride];
        dst[i] = a; dst[i + stride] = b; dst[i + 2 * stride] = c; dst[i + 3 * stride] = d;
    }
    for (; i < n16; i += stride) dst[i] = src[i];
}

int main() {
    const size_t n = 32ull << 20;
    char *hx, *hy, *dx, *dy;
    cudaHostAlloc(&hx, n, cudaHostAllocMapped);
    cudaHostAlloc(&hy, n, cudaHostAllocMapped);
    cudaMalloc(&dx, n);
    cudaMalloc(&dy, n);
    cudaStream_t s1, s2;
    cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto timeit = [&](auto&& fn) {
        for (int w = 0; w < 3; ++w) fn();
        cudaDeviceSynchronize();
        float best = 1e9;
        for (int r = 0; r < 10; ++r) {
            cudaEventRecord(a, 0);
            cudaStreamWaitEvent(s1, a, 0);
            cudaStreamWaitEvent(s2, a, 0);
            fn();
            cudaEvent_t e1, e2;
            cudaEventCreate(&e1); cudaEventCreate(&e2);
            cudaEventRecord(e1, s1); cudaEventRecord(e2, s2);
            cudaStreamWaitEvent(0, e1, 0); cudaStreamWaitEvent(0, e2, 0);
            cudaEventRecord(b, 0);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            best = ms < best ? ms : best;
            cudaEventDestroy(e1); cudaEventDestroy(e2);
        }
        return best;
    };
    const size_t n16 = n / 16;
    printf("CE: H2D %.3f ms, D2H %.3f ms, both %.3f ms\n",
           timeit([&] { cudaMemcpyAsync(dx, hx, n, cudaMemcpyHostToDevice, s1); }),
           timeit([&] { cudaMemcpyAsync(hy, dy, n, cudaMemcpyDeviceToHost, s2); }),
           timeit([&] { cudaMemcpyAsync(dx, hx, n, cudaMemcpyHostToDevice, s1);
                        cudaMemcpyAsync(hy, dy, n, cudaMemcpyDeviceToHost, s2); }));
    for (int P : {8, 16}) {
        printf("CE %d+%d pieces: both %.3f ms\n", P, P, timeit([&] {
                   for (int p = 0; p < P; ++p) {
                       cudaMemcpyAsync(dx + p * (n / P), hx + p * (n / P), n / P, cudaMemcpyHostToDevice, s1);
                       cudaMemcpyAsync(hy + p * (n / P), dy + p * (n / P), n / P, cudaMemcpyDeviceToHost, s2);
                   }
               }));
    }
    for (int G : {16, 32, 64, 148, 296}) {
        for (int T : {256, 1024}) {
            float h2d = timeit([&] { copy_kernel<<<G, T, 0, s1>>>((const int4*)hx, (int4*)dx, n16, 0); });
            float d2h = timeit([&] { copy_kernel<<<G, T, 0, s2>>>((const int4*)dy, (int4*)hy, n16, 0); });
            float both = timeit([&] {
                copy_kernel<<<G, T, 0, s1>>>((const int4*)hx, (int4*)dx, n16, 0);
                copy_kernel<<<G, T, 0, s2>>>((const int4*)dy, (int4*)hy, n16, 0);
            });
            float mix = timeit([&] {
                copy_kernel<<<G, T, 0, s1>>>((const int4*)hx, (int4*)dx, n16, 0);
                cudaMemcpyAsync(hy, dy, n, cudaMemcpyDeviceToHost, s2);
            });
            float mix2 = timeit([&] {
                cudaMemcpyAsync(dx, hx, n, cudaMemcpyHostToDevice, s1);
                copy_kernel<<<G, T, 0, s2>>>((const int4*)dy, (int4*)hy, n16, 0);
            });
            printf("SM G=%d T=%d: H2D %.3f ms (%.1f GB/s), D2H %.3f ms (%.1f GB/s), both %.3f ms, "
                   "SM H2D + CE D2H %.3f ms, CE H2D + SM D2H %.3f ms\n",
                   G, T, h2d, n / h2d / 1e6, d2h, n / d2h / 1e6, both, mix, mix2);
        }
    }
    return 0;
}
