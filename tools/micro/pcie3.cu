// PCIe transfer strategies for the SpMV plan's x-in / y-out (32 MiB each):
//  A: copy engines, P pieces per direction (cudaMemcpyAsync from C++)
//  B: SM-driven copies through mapped pinned memory (ld/st.global on the
//     host pointer), H2D and D2H kernels on two streams
#include <cstdio>
#include <vector>
#include <chrono>
#include <cuda_runtime.h>

__global__ void sm_copy(const double2* __restrict__ src, double2* __restrict__ dst, size_t n2) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    constexpr int U = 8;
    for (; i + (U - 1) * stride < n2; i += U * stride) {
        double2 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = src[i + u * stride];
#pragma unroll
        for (int u = 0; u < U; ++u) dst[i + u * stride] = v[u];
    }
    for (; i < n2; i += stride) dst[i] = src[i];
}

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

int main() {
    const size_t n = 32ull << 20;
    double *hx, *hy, *dx, *dy;
    cudaHostAlloc(&hx, n, cudaHostAllocDefault);
    cudaHostAlloc(&hy, n, cudaHostAllocDefault);
    cudaMalloc(&dx, n);
    cudaMalloc(&dy, n);
    cudaStream_t s1, s2;
    cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    std::vector<cudaEvent_t> ev(64);
    for (auto& e : ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    for (int P : {1, 2, 4, 8, 16}) {
        double best = 1e9;
        for (int rep = 0; rep < 5; ++rep) {
            cudaDeviceSynchronize();
            double t0 = now();
            const size_t m = n / P;
            for (int i = 0; i < P; ++i) {
                cudaMemcpyAsync((char*)dx + i * m, (char*)hx + i * m, m, cudaMemcpyHostToDevice, s1);
                cudaEventRecord(ev[i], s1);
            }
            for (int i = 0; i < P; ++i) {
                cudaStreamWaitEvent(s2, ev[i], 0);
                cudaMemcpyAsync((char*)hy + i * m, (char*)dy + i * m, m, cudaMemcpyDeviceToHost, s2);
            }
            cudaDeviceSynchronize();
            best = std::min(best, now() - t0);
        }
        printf("CE  pieces %2d: %.3f ms (%.1f GB/s total)\n", P, best * 1e3, 2 * n / best / 1e9);
    }
    for (int ctas : {8, 16, 32, 64, 148}) {
        for (int mode = 0; mode < 3; ++mode) {  // 0 H2D only, 1 D2H only, 2 both
            double best = 1e9;
            for (int rep = 0; rep < 5; ++rep) {
                cudaDeviceSynchronize();
                double t0 = now();
                if (mode != 1) sm_copy<<<ctas, 512, 0, s1>>>((const double2*)hx, (double2*)dx, n / 16);
                if (mode != 0) sm_copy<<<ctas, 512, 0, s2>>>((const double2*)dy, (double2*)hy, n / 16);
                cudaDeviceSynchronize();
                best = std::min(best, now() - t0);
            }
            printf("SM  ctas %3d %s: %.3f ms (%.1f GB/s)\n", ctas, mode == 0 ? "h2d " : mode == 1 ? "d2h " : "both",
                   best * 1e3, (mode == 2 ? 2 : 1) * n / best / 1e9);
        }
    }
    // mixed: SM-driven H2D, CE D2H
    for (int ctas : {16, 32, 64}) {
        double best = 1e9;
        for (int rep = 0; rep < 5; ++rep) {
            cudaDeviceSynchronize();
            double t0 = now();
            sm_copy<<<ctas, 512, 0, s1>>>((const double2*)hx, (double2*)dx, n / 16);
            cudaMemcpyAsync(hy, dy, n, cudaMemcpyDeviceToHost, s2);
            cudaDeviceSynchronize();
            best = std::min(best, now() - t0);
        }
        printf("mix SM-h2d %d ctas + CE-d2h: %.3f ms (%.1f GB/s total)\n", ctas, best * 1e3, 2 * n / best / 1e9);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
