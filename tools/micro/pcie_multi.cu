// Does round-robining the pieces of a 32 MiB H2D + 32 MiB D2H transfer over
// K streams per direction hide the per-copy setup cost?  (pcie3.cu: one
// stream per direction loses ~7 us per piece: 94 GB/s at 1 piece, 72 GB/s at
// 16 pieces.)  Prints GB/s of the 64 MiB for P pieces x K streams, plus the
// device's asyncEngineCount.
#include <chrono>
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    printf("asyncEngineCount %d\n", p.asyncEngineCount);
    const size_t n = 32ull << 20;
    char *hx, *hy, *dx, *dy;
    cudaHostAlloc(&hx, n, cudaHostAllocDefault);
    cudaHostAlloc(&hy, n, cudaHostAllocDefault);
    cudaMalloc(&dx, n);
    cudaMalloc(&dy, n);
    std::vector<cudaStream_t> sin(8), sout(8);
    for (int i = 0; i < 8; ++i) {
        cudaStreamCreateWithFlags(&sin[i], cudaStreamNonBlocking);
        cudaStreamCreateWithFlags(&sout[i], cudaStreamNonBlocking);
    }
    for (int dir = 0; dir < 3; ++dir) {  // 0 both, 1 H2D only, 2 D2H only
        for (int P : {1, 4, 8, 16, 32}) {
            for (int K : {1, 2, 4, 8}) {
                if (K > P) continue;
                double best = 1e9;
                for (int rep = 0; rep < 6; ++rep) {
                    cudaDeviceSynchronize();
                    const double t0 = now();
                    const size_t piece = n / P;
                    for (int i = 0; i < P; ++i) {
                        if (dir != 2) cudaMemcpyAsync(dx + i * piece, hx + i * piece, piece, cudaMemcpyHostToDevice, sin[i % K]);
                        if (dir != 1) cudaMemcpyAsync(hy + i * piece, dy + i * piece, piece, cudaMemcpyDeviceToHost, sout[i % K]);
                    }
                    cudaDeviceSynchronize();
                    const double t = now() - t0;
                    if (rep && t < best) best = t;
                }
                const double bytes = dir == 0 ? 2.0 * n : (double)n;
                printf("%-9s P %2d K %d: %.3f ms  %.1f GB/s\n", dir == 0 ? "both" : (dir == 1 ? "h2d" : "d2h"), P, K,
                       best * 1e3, bytes / best / 1e9);
            }
        }
    }
    return 0;
}
