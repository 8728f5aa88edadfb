// gemv.cu -- dense FP64 GEMV y = A*x (SURVEY.md §8f "next" #4; the
// reference models it as gemv_model, kernels.cpp:88-101: W = 2mn,
// Q = (mn + m + n)*8; PAPER.md:155-165 uses it as the baseline for SpMV and
// for the "Speedup_A100(GEMV) < 1.05" workload ceiling).  A is row-major
// m x n; HBM-bound at Q bytes.
//
//  CUDA core: a warp owns R rows; each lane streams 4 consecutive columns of
//      every row per step (256-bit loads of A, evict_first) and the matching
//      x vector (L1/L2-resident), DFMA, then one xor-shuffle reduction per row.
//  Tensor core: a warp owns an 8-row block; lane 4r+c holds 4 consecutive
//      columns A[r][k0+4c .. +3] and x[k0+4c .. +3]; component j feeds DMMA j
//      with A[r][c] = A-element, B[c][n] = x-element (identical for every n),
//      so every column of D accumulates the 8 row dot products -- 1/8 of the
//      datapath does useful work, as the paper's bound assumes.
#include "common.cuh"
#include "kernels.h"

namespace rlb {
namespace {

template <int R, int UK>
__global__ void __launch_bounds__(256) gemv_cc(uint64_t m, uint64_t n, const double* __restrict__ A,
                                               const double* __restrict__ x, double* __restrict__ y) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t pol = policy_evict_first();
    const bool vec = (n % 4 == 0) && aligned32(A) && aligned32(x);
    for (uint64_t r0 = warp * R; r0 < m; r0 += nwarps * R) {
        double acc[R];
#pragma unroll
        for (int q = 0; q < R; ++q) acc[q] = 0.0;
        if (vec) {
            // UK column steps of 128 per iteration: all R*UK loads issued first
            for (uint64_t kb = 4 * (uint64_t)lane; kb < n; kb += 128 * UK) {
                d4 xv[UK], a[UK][R];
#pragma unroll
                for (int u = 0; u < UK; ++u) {
                    const uint64_t k = kb + 128 * u;
                    const bool kin = k < n;
                    xv[u] = kin ? ld4_cached(x + k) : d4{0, 0, 0, 0};
#pragma unroll
                    for (int q = 0; q < R; ++q)
                        a[u][q] = (kin && r0 + q < m) ? ld4_stream(A + (r0 + q) * n + k, pol) : d4{0, 0, 0, 0};
                }
#pragma unroll
                for (int u = 0; u < UK; ++u)
#pragma unroll
                    for (int q = 0; q < R; ++q) {
                        acc[q] = fma(a[u][q].x, xv[u].x, acc[q]);
                        acc[q] = fma(a[u][q].y, xv[u].y, acc[q]);
                        acc[q] = fma(a[u][q].z, xv[u].z, acc[q]);
                        acc[q] = fma(a[u][q].w, xv[u].w, acc[q]);
                    }
            }
        } else {
            for (uint64_t k = lane; k < n; k += 32) {
                const double xv = ld_cached(x + k);
#pragma unroll
                for (int q = 0; q < R; ++q)
                    if (r0 + q < m) acc[q] = fma(A[(r0 + q) * n + k], xv, acc[q]);
            }
        }
#pragma unroll
        for (int q = 0; q < R; ++q) {
            double a = acc[q];
#pragma unroll
            for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
            if (lane == q && r0 + q < m) y[r0 + q] = a;
        }
    }
}

__global__ void __launch_bounds__(256) gemv_tc(uint64_t m, uint64_t n, const double* __restrict__ A,
                                               const double* __restrict__ x, double* __restrict__ y) {
    const int lane = threadIdx.x & 31, r = lane >> 2, c = lane & 3;
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t pol = policy_evict_first();
    const bool vec = (n % 4 == 0) && aligned32(A) && aligned32(x);
    for (uint64_t r0 = warp * 8; r0 < m; r0 += nwarps * 8) {
        const uint64_t row = r0 + r;
        const bool rok = row < m;
        const double* Ar = A + (rok ? row : r0) * n;
        // U 16-column chunks in flight per iteration, two accumulator chains
        constexpr int U = 4;
        double d0[2] = {0.0, 0.0}, d1[2] = {0.0, 0.0};
        for (uint64_t kb = 0; kb < n; kb += 16 * U) {
            d4 a[U], xv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint64_t k = kb + 16 * u + 4 * c;
                if (vec && k + 4 <= n) {
                    a[u] = rok ? ld4_stream(Ar + k, pol) : d4{0, 0, 0, 0};
                    xv[u] = ld4_cached(x + k);
                } else {
                    double av[4], xx[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const bool ok = k + j < n;
                        av[j] = (ok && rok) ? Ar[k + j] : 0.0;
                        xx[j] = ok ? x[k + j] : 0.0;
                    }
                    a[u] = d4{av[0], av[1], av[2], av[3]};
                    xv[u] = d4{xx[0], xx[1], xx[2], xx[3]};
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                double& e0 = d0[u & 1];
                double& e1 = d1[u & 1];
                dmma_m8n8k4(e0, e1, a[u].x, xv[u].x, e0, e1);
                dmma_m8n8k4(e0, e1, a[u].y, xv[u].y, e0, e1);
                dmma_m8n8k4(e0, e1, a[u].z, xv[u].z, e0, e1);
                dmma_m8n8k4(e0, e1, a[u].w, xv[u].w, e0, e1);
            }
        }
        // every column of D holds the row sums; lane 4r holds D[r][0]
        if (c == 0 && rok) y[row] = d0[0] + d0[1];
    }
}

}  // namespace

cudaError_t launch_gemv(int unit, uint64_t m, uint64_t n, const double* A, const double* x, double* y,
                        cudaStream_t s) {
    if (m == 0 || n == 0) return cudaSuccess;
    const unsigned max_blocks = kNumSMs * 8;
    if (unit == 1) {
        uint64_t blocks = (m + 63) / 64;
        if (blocks > max_blocks) blocks = max_blocks;
        gemv_tc<<<(unsigned)blocks, 256, 0, s>>>(m, n, A, x, y);
    } else {
        const int R = tuning().gemv_rows, UK = tuning().gemv_unroll;
        uint64_t blocks = (m + 8 * R - 1) / (8 * R);
        if (blocks > max_blocks) blocks = max_blocks;
#define RLB_GEMV(RR, UU) gemv_cc<RR, UU><<<(unsigned)blocks, 256, 0, s>>>(m, n, A, x, y)
        if (R == 2) { if (UK == 2) RLB_GEMV(2, 2); else if (UK == 4) RLB_GEMV(2, 4); else RLB_GEMV(2, 1); }
        else if (R == 4) { if (UK == 2) RLB_GEMV(4, 2); else if (UK == 4) RLB_GEMV(4, 4); else RLB_GEMV(4, 1); }
        else { if (UK == 2) RLB_GEMV(8, 2); else RLB_GEMV(8, 1); }
#undef RLB_GEMV
    }
    note_launch();
    return cudaGetLastError();
}

}  // namespace rlb
