// Do the FP64 FMA pipe (DFMA) and the FP64 tensor pipe (DMMA.8x8x4) issue
// concurrently on sm_100a?  Modes: 0 DFMA only, 1 DMMA only, 2 half the warps
// of every CTA DFMA and half DMMA, 3 every warp interleaves 1 DMMA : R DFMA.
// If mode 2's combined flop rate is ~ the sum of modes 0 and 1, a tensor-core
// stencil can move operand preparation onto DFMA for free.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int MODE, int R>
__global__ void pipes(uint64_t iters, double* sink, double* acc_out) {
    const int warp = threadIdx.x >> 5;
    double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999;
    double f[8], d[4][2];
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = j * 1e-3;
#pragma unroll
    for (int j = 0; j < 4; ++j) d[j][0] = d[j][1] = 0.0;
    const bool do_f = MODE == 0 || MODE == 3 || (MODE == 2 && (warp & 1) == 0);
    const bool do_m = MODE == 1 || MODE == 3 || (MODE == 2 && (warp & 1) == 1);
    for (uint64_t i = 0; i < iters; ++i) {
        if (do_m) {
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma(d[j][0], d[j][1], a, b);
        }
        if (do_f) {
#pragma unroll
            for (int rr = 0; rr < R; ++rr)
#pragma unroll
                for (int j = 0; j < 8; ++j) f[j] = fma(f[j], b, a);
        }
    }
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += f[j];
#pragma unroll
    for (int j = 0; j < 4; ++j) s += d[j][0] + d[j][1];
    if (s == 42.0) sink[threadIdx.x] = s;
}

template <int MODE, int R>
void run(const char* name, int sms) {
    double* sink;
    cudaMalloc(&sink, 4096);
    const int threads = 256, blocks = sms * 8;
    const uint64_t iters = 20000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    pipes<MODE, R><<<blocks, threads>>>(100, sink, nullptr);
    cudaEventRecord(e0);
    pipes<MODE, R><<<blocks, threads>>>(iters, sink, nullptr);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double warps = (double)blocks * threads / 32;
    double fwarps = 0, mwarps = 0;
    if (MODE == 0) fwarps = warps;
    if (MODE == 1) mwarps = warps;
    if (MODE == 2) fwarps = mwarps = warps / 2;
    if (MODE == 3) fwarps = mwarps = warps;
    const double ff = fwarps * 32 * (double)iters * R * 8 * 2;   // DFMA flops
    const double mf = mwarps * (double)iters * 4 * 512;          // DMMA flops
    printf("%-28s %8.3f ms  DFMA %6.2f TF/s  DMMA %6.2f TF/s  total %6.2f TF/s\n", name, ms,
           ff / ms * 1e-9, mf / ms * 1e-9, (ff + mf) / ms * 1e-9);
    cudaFree(sink);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<0, 1>("DFMA only", sms);
    run<1, 1>("DMMA only", sms);
    run<2, 1>("half warps DFMA / DMMA", sms);
    run<2, 2>("half warps, DFMA x2", sms);
    run<3, 1>("interleaved 4 DMMA : 8 DFMA", sms);
    run<3, 2>("interleaved 4 DMMA : 16 DFMA", sms);
    run<3, 4>("interleaved 4 DMMA : 32 DFMA", sms);
    return 0;
}
