// spmv.cu -- K3/K4: CSR SpMV y = A*x, FP64 values,
// int32 row pointers and column indices (kDefaultIndexBytes = 4,
// reference kernels.hpp:77).  Algorithmic bytes per call are the reference's
// spmv_csr_model (kernels.cpp:123-135): (nnz+m+n)*8 + (nnz+m+1)*4.
//
// Both variants share one data path: a lane owns 4 consecutive nonzeros of a
// row (one 256-bit load of val, one 128-bit load of col when the row start
// is 4-aligned, element-guarded scalar loads otherwise) and gathers its 4 x
// values through L2 with an evict_last policy (x is reused by every row of
// the band; val/col stream through with evict_first, bypassing L1).
//
//  K3 (CUDA core): 4 lanes per row, DFMA, 2-step xor-shuffle row reduction.
//      A warp covers 8 rows per step and R steps per iteration for MLP.
//  K4 (tensor core, DASP-style row block): a warp owns an
//      8-row block.  Lane L = 4r+c holds A[r][c] = val and B[c][r] = x[col] of
//      the same nonzero, so D = A*B accumulates, on its diagonal,
//      D[r][r] = sum_k val[r][k] * x[col[r][k]] -- the row sums -- over
//      ceil(maxlen/16) x 4 DMMA m8n8k4 steps (rows shorter than the block's
//      longest row are zero-padded).  Off-diagonal products are discarded:
//      1/8 utilisation, as the paper's bound assumes.
#include "common.cuh"
#include "kernels.h"

namespace rlb {
namespace {

struct Nz4 {
    double v[4];
    int c[4];
    int n;  // valid slots (a prefix); padded slots carry val = 0 and are never gathered
};

// Load the (up to) 4 nonzeros [j, j+4) of a row ending at e.
__device__ __forceinline__ Nz4 load_nz4(const int* __restrict__ col,
                                        const double* __restrict__ val, int64_t j, int64_t e,
                                        int col_pad, uint64_t pol) {
    Nz4 z;
    if (((j & 3) == 0) && j + 4 <= e) {
        const d4 v = ld4_stream(val + j, pol);
        int4 ci;
        asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
            : "=r"(ci.x), "=r"(ci.y), "=r"(ci.z), "=r"(ci.w)
            : "l"(col + j), "l"(pol));
        z.v[0] = v.x; z.v[1] = v.y; z.v[2] = v.z; z.v[3] = v.w;
        z.c[0] = ci.x; z.c[1] = ci.y; z.c[2] = ci.z; z.c[3] = ci.w;
        z.n = 4;
    } else {
        const int64_t left = e - j;
        z.n = left <= 0 ? 0 : (left >= 4 ? 4 : (int)left);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const bool ok = j + k < e;
            z.v[k] = ok ? ld_stream(val + j + k, pol) : 0.0;
            z.c[k] = ok ? ld_stream_i32(col + j + k, pol) : col_pad;
        }
    }
    return z;
}

__device__ __forceinline__ double ld_x(const double* p, uint64_t pol, int hint) {
    double v;
    if (hint == 1)
        asm("ld.global.nc.L1::evict_last.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    else if (hint == 2)
        asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    else
        asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}

// Gather x for 4 nonzeros; padded slots get 0 (so 0*x never meets a non-finite x).
template <int XH = 0>
__device__ __forceinline__ void gather4(double (&xv)[4], const Nz4& z,
                                        const double* __restrict__ x, int64_t col_base,
                                        uint64_t polx) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
        xv[k] = k < z.n ? ld_x(x + ((int64_t)z.c[k] - col_base), polx, XH) : 0.0;
}

// K3: CUDA core.  Row of warp-step u for group q: wbase + 8u + q.
// SCHED 0: warps stride over the whole row range (grid-stride);
// SCHED 1: each CTA owns one contiguous row range (x-window locality in L1).
template <int R, int SCHED, int XH>
__global__ void __launch_bounds__(1024) spmv_cc_v4(uint64_t r0, uint64_t r1,
                                                  const int* __restrict__ rp,
                                                  const int* __restrict__ col,
                                                  const double* __restrict__ val,
                                                  const double* __restrict__ x, int64_t col_base,
                                                  double* __restrict__ y) {
    const int lane = threadIdx.x & 31;
    const int c = lane & 3, q = lane >> 2;
    const uint64_t pol = policy_evict_first(), polx = policy_evict_last();
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const int col_pad = 0;
    uint64_t first, stride, last;
    if (SCHED == 0) {
        first = r0 + warp * 8 * R;
        stride = nwarps * 8 * R;
        last = r1;
    } else {
        const uint64_t per = ((r1 - r0) + gridDim.x - 1) / gridDim.x;
        const uint64_t b0 = r0 + (uint64_t)blockIdx.x * per;
        first = b0 + (threadIdx.x >> 5) * 8 * R;
        stride = (blockDim.x >> 5) * 8 * R;
        last = min(r1, b0 + per);
    }
    for (uint64_t wbase = first; wbase < last; wbase += stride) {
        const uint64_t rend = last;
        int64_t s[R], e[R];
#pragma unroll
        for (int u = 0; u < R; ++u) {
            const uint64_t row = wbase + 8 * u + q;
            const bool ok = row < rend;
            s[u] = ok ? __ldg(rp + row) : 0;
            e[u] = ok ? __ldg(rp + row + 1) : 0;
        }
        Nz4 z[R];
#pragma unroll
        for (int u = 0; u < R; ++u) z[u] = load_nz4(col, val, s[u] + 4 * c, e[u], col_pad, pol);
        double acc[R];
#pragma unroll
        for (int u = 0; u < R; ++u) {
            double xv[4];
            gather4<XH>(xv, z[u], x, col_base, polx);
            double a = z[u].v[0] * xv[0];
            a = fma(z[u].v[1], xv[1], a);
            a = fma(z[u].v[2], xv[2], a);
            a = fma(z[u].v[3], xv[3], a);
            acc[u] = a;
        }
        // rows longer than 16 nonzeros (not in the banded config)
#pragma unroll
        for (int u = 0; u < R; ++u) {
            for (int64_t j = s[u] + 16 + 4 * c; j < e[u]; j += 16) {
                Nz4 t = load_nz4(col, val, j, e[u], col_pad, pol);
                double xv[4];
                gather4<XH>(xv, t, x, col_base, polx);
#pragma unroll
                for (int k = 0; k < 4; ++k) acc[u] = fma(t.v[k], xv[k], acc[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < R; ++u) {
            double a = acc[u];
            a += __shfl_xor_sync(0xffffffffu, a, 1);
            a += __shfl_xor_sync(0xffffffffu, a, 2);
            const uint64_t row = wbase + 8 * u + q;
            if (c == 0 && row < rend) y[row] = a;
        }
    }
}

// K4: tensor core.  A warp owns RB 8-row blocks per iteration (independent
// DMMA accumulator chains); SCHED as in K3.
template <int RB, int SCHED>
__global__ void __launch_bounds__(1024) spmv_tc(uint64_t r0, uint64_t r1,
                                                const int* __restrict__ rp,
                                                const int* __restrict__ col,
                                                const double* __restrict__ val,
                                                const double* __restrict__ x, int64_t col_base,
                                                double* __restrict__ y) {
    const int lane = threadIdx.x & 31;
    const int r = lane >> 2, c = lane & 3;
    const uint64_t pol = policy_evict_first(), polx = policy_evict_last();
    const int col_pad = 0;
    uint64_t first, stride, last;
    if (SCHED == 0) {
        const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
        const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
        first = r0 + warp * 8 * RB;
        stride = nwarps * 8 * RB;
        last = r1;
    } else {
        const uint64_t per = ((r1 - r0) + gridDim.x - 1) / gridDim.x;
        const uint64_t b0 = r0 + (uint64_t)blockIdx.x * per;
        first = b0 + (threadIdx.x >> 5) * 8 * RB;
        stride = (blockDim.x >> 5) * 8 * RB;
        last = min(r1, b0 + per);
    }
    for (uint64_t base = first; base < last; base += stride) {
        int64_t s[RB], e[RB];
        int len = 0;
#pragma unroll
        for (int q = 0; q < RB; ++q) {
            const uint64_t row = base + 8 * q + r;
            const bool ok = row < last;
            s[q] = ok ? __ldg(rp + row) : 0;
            e[q] = ok ? __ldg(rp + row + 1) : 0;
            len = max(len, (int)(e[q] - s[q]));
        }
        const int maxlen = __reduce_max_sync(0xffffffffu, len);
        double d0[RB], d1[RB];
#pragma unroll
        for (int q = 0; q < RB; ++q) d0[q] = d1[q] = 0.0;
        for (int off = 0; off < maxlen; off += 16) {
            Nz4 z[RB];
#pragma unroll
            for (int q = 0; q < RB; ++q) z[q] = load_nz4(col, val, s[q] + off + 4 * c, e[q], col_pad, pol);
#pragma unroll
            for (int q = 0; q < RB; ++q) {
                double xv[4];
                gather4(xv, z[q], x, col_base, polx);
                // A[r][c] = val, B[c][r] = x[col]: one k-slice per vector component.
                dmma_m8n8k4(d0[q], d1[q], z[q].v[0], xv[0], d0[q], d1[q]);
                dmma_m8n8k4(d0[q], d1[q], z[q].v[1], xv[1], d0[q], d1[q]);
                dmma_m8n8k4(d0[q], d1[q], z[q].v[2], xv[2], d0[q], d1[q]);
                dmma_m8n8k4(d0[q], d1[q], z[q].v[3], xv[3], d0[q], d1[q]);
            }
        }
        // D[r][r] lives in lane 4r + r/2, element r%2.
#pragma unroll
        for (int q = 0; q < RB; ++q) {
            const uint64_t row = base + 8 * q + r;
            if (c == (r >> 1) && row < last) y[row] = (r & 1) ? d1[q] : d0[q];
        }
    }
}

}  // namespace

cudaError_t launch_spmv(int unit, uint64_t r0, uint64_t r1, const int* rp, const int* col,
                        const double* val, const double* x, int64_t col_base, double* y,
                        double avg_nnz_per_row, cudaStream_t s) {
    (void)avg_nnz_per_row;
    if (r1 <= r0) return cudaSuccess;
    const Tuning& t = tuning();
    const int threads = 256;
    const uint64_t rows = r1 - r0;
    const uint64_t max_blocks = (uint64_t)kNumSMs * (uint64_t)t.spmv_blocks_per_sm;
    if (unit == 1) {
        const int tthreads = t.spmv_tc_threads, RB = t.spmv_tc_rows;
        uint64_t blocks = (rows + (uint64_t)(tthreads / 32) * 8 * RB - 1) / ((uint64_t)(tthreads / 32) * 8 * RB);
        const uint64_t cap = (uint64_t)kNumSMs * (uint64_t)t.spmv_tc_blocks_per_sm;
        if (blocks > cap) blocks = cap;
#define RLB_TC(R, S) spmv_tc<R, S><<<(unsigned)blocks, tthreads, 0, s>>>(r0, r1, rp, col, val, x, col_base, y)
        if (t.spmv_sched == 0) { if (RB == 2) RLB_TC(2, 0); else RLB_TC(1, 0); }
        else { if (RB == 2) RLB_TC(2, 1); else RLB_TC(1, 1); }
#undef RLB_TC
        note_launch();
        return cudaGetLastError();
    }
    const int R = t.spmv_rows;
    const int cthreads = t.spmv_threads;
    const uint64_t rows_per_block = (uint64_t)(cthreads / 32) * 8ull * (uint64_t)R;
    uint64_t blocks = (rows + rows_per_block - 1) / rows_per_block;
    const uint64_t cap = (uint64_t)kNumSMs * (uint64_t)t.spmv_blocks_per_sm;
    if (blocks > cap) blocks = cap;
    const int sched = t.spmv_sched, xh = t.spmv_xhint;
#define RLB_SPMV(RR, SS, XX)                                                                      \
    do {                                                                                          \
        if (t.spmv_l1_carveout >= 0)                                                              \
            cudaFuncSetAttribute(spmv_cc_v4<RR, SS, XX>,                                          \
                                 cudaFuncAttributePreferredSharedMemoryCarveout, t.spmv_l1_carveout); \
        spmv_cc_v4<RR, SS, XX><<<(unsigned)blocks, cthreads, 0, s>>>(r0, r1, rp, col, val, x, col_base, y); \
    } while (0)
#define RLB_SPMV_R(SS, XX)                        \
    do {                                          \
        if (R == 1) RLB_SPMV(1, SS, XX);          \
        else if (R == 2) RLB_SPMV(2, SS, XX);     \
        else RLB_SPMV(4, SS, XX);                 \
    } while (0)
    if (sched == 0) {
        if (xh == 1) RLB_SPMV_R(0, 1); else if (xh == 2) RLB_SPMV_R(0, 2); else RLB_SPMV_R(0, 0);
    } else {
        if (xh == 1) RLB_SPMV_R(1, 1); else if (xh == 2) RLB_SPMV_R(1, 2); else RLB_SPMV_R(1, 0);
    }
#undef RLB_SPMV_R
#undef RLB_SPMV
    note_launch();
    return cudaGetLastError();
}

}  // namespace rlb
