// Premise check for a column-sorted SpMV layout: random 8-byte gathers from an
// L2-resident 32 MiB x run at ~1 per SM per cycle (dsmem_gather.cu).  If the
// nonzeros of a B-nonzero block (columns uniform in a 132K-column window, as
// in the BASELINE band) are visited in column order, a warp instruction's 32
// gathers fall on ~32 * 132K / (16 B) ... fewer 128-byte lines.  This times
// gather+multiply-accumulate over 64M entries for block sizes B, sorted vs
// unsorted, and prints G gathers/s.
#include <algorithm>
#include <cstdio>
#include <cstdint>
#include <random>
#include <vector>
#include <cuda_runtime.h>

__global__ void gather(const int* __restrict__ col, const double* __restrict__ x, size_t n, double* out) {
    double acc = 0.0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    for (; i + 7 * stride < n; i += 8 * stride) {
        int c[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) c[u] = __ldcs(col + i + u * stride);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += __ldg(x + c[u]);
    }
    for (; i < n; i += stride) acc += __ldg(x + col[i]);
    if (acc == 42.0) out[0] = acc;
}

// block-contiguous: warp w of the grid walks entries [w * per_warp, ...) 32 at a time
__global__ void gather_blocked(const int* __restrict__ col, const double* __restrict__ x, size_t n, double* out) {
    const size_t warps = (size_t)gridDim.x * blockDim.x / 32;
    const size_t w = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) / 32;
    const int lane = threadIdx.x & 31;
    const size_t per = (n / warps) / 256 * 256;
    const int* cp = col + w * per;
    double acc = 0.0;
    for (size_t j = lane; j + 7 * 32 < per; j += 8 * 32) {
        int c[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) c[u] = __ldcs(cp + j + u * 32);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += __ldg(x + c[u]);
    }
    if (acc == 42.0) out[0] = acc;
}

int main() {
    const int nx = 1 << 22;
    const size_t n = 1ull << 26;
    double *x, *out;
    int* col;
    cudaMalloc(&x, nx * 8);
    cudaMemset(x, 0, nx * 8);
    cudaMalloc(&out, 8);
    cudaMalloc(&col, n * 4);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    std::mt19937_64 rng(1);
    std::vector<int> h(n);
    for (int B : {0, 4096, 8192, 16384, 32768}) {
        // entries in blocks of B; block b's columns uniform in a 132K window that slides
        // with the block (like 16 nnz/row rows B/16 at a time); B = 0: no sorting
        const size_t blk = B ? B : 4096;
        for (size_t b0 = 0; b0 < n; b0 += blk) {
            const long row0 = (long)(b0 / 16) % nx;
            for (size_t j = b0; j < b0 + blk && j < n; ++j) {
                long c = row0 - 65536 + (long)(rng() % 131072);
                h[j] = (int)std::min<long>(std::max<long>(c, 0), nx - 1);
            }
            if (B) std::sort(h.begin() + b0, h.begin() + std::min(n, b0 + blk));
        }
        cudaMemcpy(col, h.data(), n * 4, cudaMemcpyHostToDevice);
        for (int mode = 0; mode < 2; ++mode) {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            for (int it = 0; it < 2; ++it) {
                cudaEventRecord(e0);
                if (mode == 0) gather<<<sms * 8, 256>>>(col, x, n, out);
                else gather_blocked<<<sms * 8, 256>>>(col, x, n, out);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
            }
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("block %6d sorted %d  %s: %.3f ms  %.1f G gathers/s\n", B, B ? 1 : 0,
                   mode ? "warp-contiguous" : "grid-stride    ", ms, n / ms / 1e6);
        }
    }
    return 0;
}
