// The e2e SpMV pipeline's copy pattern without compute: 8 H2D pieces of x on
// one stream, 8 D2H pieces of y on another, D2H piece c waiting on an event
// recorded after H2D piece c + lag.  How much do the cross-stream waits cost
// against the same copies issued without waits?  Also: one SM copy kernel
// per y piece (zero-copy stores) instead of the D2H copy-engine copies.
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

__global__ void copy_kernel(const int4* __restrict__ src, int4* __restrict__ dst, size_t n16) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) dst[i] = src[i];
}

int main() {
    const size_t n = 32ull << 20;
    char *hx, *hy, *dx, *dy;
    cudaHostAlloc(&hx, n, cudaHostAllocMapped);
    cudaHostAlloc(&hy, n, cudaHostAllocMapped);
    cudaMalloc(&dx, n);
    cudaMalloc(&dy, n);
    cudaStream_t s1, s2, s3;
    cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s3, cudaStreamNonBlocking);
    std::vector<cudaEvent_t> ev(64), ev2(64);
    for (auto& e : ev2) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    for (auto& e : ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    cudaEvent_t a, b, f;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventCreateWithFlags(&f, cudaEventDisableTiming);
    auto run = [&](int P, int lag, int mode, bool graph) {
        // mode 0: D2H CE copies with waits; 1: no waits; 2: SM copy kernel per y piece with waits;
        // 3: the plan's two hops (a third stream waits on the H2D event and records its own, D2H waits on that)
        auto body = [&] {
            cudaEventRecord(f, s1);
            cudaStreamWaitEvent(s2, f, 0);
            cudaStreamWaitEvent(s3, f, 0);
            const size_t pc = n / P;
            for (int p = 0; p < P; ++p) {
                cudaMemcpyAsync(dx + p * pc, hx + p * pc, pc, cudaMemcpyHostToDevice, s1);
                cudaEventRecord(ev[p], s1);
            }
            for (int p = 0; p < P; ++p) {
                if (mode == 3) {
                    cudaStreamWaitEvent(s3, ev[std::min(P - 1, p + lag)], 0);
                    cudaEventRecord(ev2[p], s3);
                    cudaStreamWaitEvent(s2, ev2[p], 0);
                } else if (mode != 1) cudaStreamWaitEvent(s2, ev[std::min(P - 1, p + lag)], 0);
                if (mode == 2)
                    copy_kernel<<<64, 1024, 0, s2>>>((const int4*)(dy + p * pc), (int4*)(hy + p * pc), pc / 16);
                else
                    cudaMemcpyAsync(hy + p * pc, dy + p * pc, pc, cudaMemcpyDeviceToHost, s2);
            }
            cudaEventRecord(ev[63], s2);
            cudaStreamWaitEvent(s1, ev[63], 0);
            cudaEventRecord(ev2[63], s3);
            cudaStreamWaitEvent(s1, ev2[63], 0);
        };
        cudaGraphExec_t ge = nullptr;
        if (graph) {
            cudaGraph_t g;
            cudaStreamBeginCapture(s1, cudaStreamCaptureModeThreadLocal);
            body();
            cudaStreamEndCapture(s1, &g);
            cudaGraphInstantiate(&ge, g, 0);
            cudaGraphDestroy(g);
        }
        float best = 1e9;
        for (int r = 0; r < 12; ++r) {
            cudaEventRecord(a, s1);
            if (graph) cudaGraphLaunch(ge, s1);
            else body();
            cudaEventRecord(b, s1);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (r >= 2) best = ms < best ? ms : best;
        }
        if (ge) cudaGraphExecDestroy(ge);
        return best;
    };
    for (int graph = 0; graph < 2; ++graph)
        for (int P : {1, 2, 4, 8, 16})
            printf("graph %d pieces %2d: no waits %.3f ms, CE waits lag 1 %.3f, lag 0 %.3f, SM y copies lag 1 %.3f, "
                   "two hops lag 0 %.3f\n",
                   graph, P, run(P, 1, 1, graph), run(P, 1, 0, graph), run(P, 0, 0, graph), run(P, 1, 2, graph),
                   run(P, 0, 3, graph));
    return 0;
}
