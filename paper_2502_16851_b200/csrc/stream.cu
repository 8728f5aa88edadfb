// stream.cu -- K1/K2: STREAM Scale a[i] = q * b[i].
//
// Both variants move exactly the model's bytes (scale_model, reference
// kernels.cpp:74-86: 16 B per element) with 256-bit LDG/STG, streamed
// through L2 with evict_first and past L1 (no_allocate).  HBM-bound: the
// roofline is 16 B/element at the measured copy bandwidth.
//
//  K1 (CUDA core): one DMUL per element.
//  K2 (tensor core): the paper's A = B*(qI) on DMMA
//      m8n8k4.  A warp owns 256 contiguous doubles per step.  Lane L loads
//      v0 = b[4L..4L+3] and v1 = b[128+4L..128+4L+3]; each component j of v0
//      (v1) is the A fragment of one MMA whose B = q*[I4 | 0] (q*[0 | I4]).
//      Lane L=4r+c then holds, across the 8 MMAs, the 8 contiguous outputs
//      a[16r+8c .. +7] (c<2, from the [I|0] MMAs) or a[128+16r+8(c-2) .. +7]
//      (c>=2, from the [0|I] MMAs), so the D fragments need no shuffles and
//      leave as two 256-bit stores per lane.  Every product but one per
//      output is an exact +-0, so the result is round(q*b): bit-exact with
//      the CUDA-core variant for finite b (b = -0 gives +0).  Utilisation is
//      1/8 of the DMMA datapath by construction (bounds.cpp:127-135).
#include "common.cuh"
#include "kernels.h"

namespace rlb {
namespace {

template <int UNROLL>
__global__ void __launch_bounds__(256) scale_cc_v4(double* __restrict__ a,
                                                   const double* __restrict__ b, double q,
                                                   uint64_t nvec) {
    const uint64_t pol = policy_evict_first();
    const uint64_t bd = blockDim.x;
    const uint64_t stride = (uint64_t)gridDim.x * bd * UNROLL;
    for (uint64_t base = (uint64_t)blockIdx.x * bd * UNROLL + threadIdx.x; base < nvec;
         base += stride) {
        d4 v[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            const uint64_t i = base + u * bd;
            if (i < nvec) v[u] = ld4_stream(b + 4 * i, pol);
        }
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            const uint64_t i = base + u * bd;
            if (i < nvec) {
                d4 o{q * v[u].x, q * v[u].y, q * v[u].z, q * v[u].w};
                st4_stream(a + 4 * i, o, pol);
            }
        }
    }
}

__global__ void scale_cc_scalar(double* __restrict__ a, const double* __restrict__ b, double q,
                                uint64_t n) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        a[i] = q * b[i];
}

// One 256-element warp chunk on the tensor core.  FULL: all 256 valid and
// 32-byte aligned (vector path); otherwise element-guarded scalar accesses.
template <bool FULL>
__device__ __forceinline__ void scale_tc_chunk(double* __restrict__ a,
                                               const double* __restrict__ b, uint64_t rem,
                                               double blo, double bhi, int lane, uint64_t pol) {
    d4 v0, v1;
    if (FULL) {
        v0 = ld4_stream(b + 4 * lane, pol);
        v1 = ld4_stream(b + 128 + 4 * lane, pol);
    } else {
        const uint64_t e0 = 4 * lane, e1 = 128 + 4 * lane;
        v0.x = e0 + 0 < rem ? b[e0 + 0] : 0.0;
        v0.y = e0 + 1 < rem ? b[e0 + 1] : 0.0;
        v0.z = e0 + 2 < rem ? b[e0 + 2] : 0.0;
        v0.w = e0 + 3 < rem ? b[e0 + 3] : 0.0;
        v1.x = e1 + 0 < rem ? b[e1 + 0] : 0.0;
        v1.y = e1 + 1 < rem ? b[e1 + 1] : 0.0;
        v1.z = e1 + 2 < rem ? b[e1 + 2] : 0.0;
        v1.w = e1 + 3 < rem ? b[e1 + 3] : 0.0;
    }
    double l0[4], l1[4], h0[4], h1[4];
    dmma_m8n8k4(l0[0], l1[0], v0.x, blo, 0.0, 0.0);
    dmma_m8n8k4(l0[1], l1[1], v0.y, blo, 0.0, 0.0);
    dmma_m8n8k4(l0[2], l1[2], v0.z, blo, 0.0, 0.0);
    dmma_m8n8k4(l0[3], l1[3], v0.w, blo, 0.0, 0.0);
    dmma_m8n8k4(h0[0], h1[0], v1.x, bhi, 0.0, 0.0);
    dmma_m8n8k4(h0[1], h1[1], v1.y, bhi, 0.0, 0.0);
    dmma_m8n8k4(h0[2], h1[2], v1.z, bhi, 0.0, 0.0);
    dmma_m8n8k4(h0[3], h1[3], v1.w, bhi, 0.0, 0.0);
    const int r = lane >> 2, c = lane & 3;
    const bool lo = c < 2;
    const uint64_t off = lo ? 16 * r + 8 * c : 128 + 16 * r + 8 * (c - 2);
    d4 o0{lo ? l0[0] : h0[0], lo ? l0[1] : h0[1], lo ? l0[2] : h0[2], lo ? l0[3] : h0[3]};
    d4 o1{lo ? l1[0] : h1[0], lo ? l1[1] : h1[1], lo ? l1[2] : h1[2], lo ? l1[3] : h1[3]};
    if (FULL) {
        st4_stream(a + off, o0, pol);
        st4_stream(a + off + 4, o1, pol);
    } else {
        const double o[8] = {o0.x, o0.y, o0.z, o0.w, o1.x, o1.y, o1.z, o1.w};
#pragma unroll
        for (int k = 0; k < 8; ++k)
            if (off + k < rem) a[off + k] = o[k];
    }
}

template <bool ALIGNED>
__global__ void __launch_bounds__(256) scale_tc(double* __restrict__ a,
                                                const double* __restrict__ b, double q,
                                                uint64_t n) {
    const int lane = threadIdx.x & 31;
    const int r = lane >> 2, c = lane & 3;
    // B fragment: lane holds B[k=c][col=r].  [I4|0]: col == k; [0|I4]: col == 4+k.
    const double blo = (r == c) ? q : 0.0;
    const double bhi = (r == c + 4) ? q : 0.0;
    const uint64_t pol = policy_evict_first();
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t nfull = n >> 8;
    for (uint64_t ch = warp; ch < nfull; ch += nwarps) {
        if (ALIGNED)
            scale_tc_chunk<true>(a + (ch << 8), b + (ch << 8), 256, blo, bhi, lane, pol);
        else
            scale_tc_chunk<false>(a + (ch << 8), b + (ch << 8), 256, blo, bhi, lane, pol);
    }
    const uint64_t rem = n - (nfull << 8);
    if (rem && warp == nfull % nwarps)
        scale_tc_chunk<false>(a + (nfull << 8), b + (nfull << 8), rem, blo, bhi, lane, pol);
}

}  // namespace

cudaError_t launch_scale(int unit, double* a, const double* b, double q, uint64_t n,
                         cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const Tuning& t = tuning();
    const int threads = 256;
    const uint64_t max_blocks = (uint64_t)kNumSMs * (uint64_t)t.scale_blocks_per_sm;
    if (unit == 1) {
        const uint64_t warps_needed = (n + 255) / 256;
        uint64_t blocks = (warps_needed + 7) / 8;
        if (blocks > max_blocks) blocks = max_blocks;
        if (aligned32(a) && aligned32(b))
            scale_tc<true><<<(unsigned)blocks, threads, 0, s>>>(a, b, q, n);
        else
            scale_tc<false><<<(unsigned)blocks, threads, 0, s>>>(a, b, q, n);
        note_launch();
        return cudaGetLastError();
    }
    // CUDA core: peel to a common 32-byte alignment, 256-bit body, scalar tail.
    const uintptr_t pa = reinterpret_cast<uintptr_t>(a), pb = reinterpret_cast<uintptr_t>(b);
    if ((pa & 31) != (pb & 31) || (pa & 7) != 0) {
        uint64_t blocks = (n + threads - 1) / threads;
        if (blocks > max_blocks) blocks = max_blocks;
        scale_cc_scalar<<<(unsigned)blocks, threads, 0, s>>>(a, b, q, n); note_launch();
        return cudaGetLastError();
    }
    uint64_t head = ((32 - (pa & 31)) & 31) / 8;
    if (head > n) head = n;
    if (head) { scale_cc_scalar<<<1, 32, 0, s>>>(a, b, q, head); note_launch(); }
    const uint64_t body = n - head;
    const uint64_t nvec = body / 4;
    if (nvec) {
        const int U = t.scale_unroll;
        uint64_t blocks = (nvec + (uint64_t)threads * U - 1) / ((uint64_t)threads * U);
        if (blocks > max_blocks) blocks = max_blocks;
        if (U == 1) scale_cc_v4<1><<<(unsigned)blocks, threads, 0, s>>>(a + head, b + head, q, nvec);
        else if (U == 2) scale_cc_v4<2><<<(unsigned)blocks, threads, 0, s>>>(a + head, b + head, q, nvec);
        else if (U == 8) scale_cc_v4<8><<<(unsigned)blocks, threads, 0, s>>>(a + head, b + head, q, nvec);
        else scale_cc_v4<4><<<(unsigned)blocks, threads, 0, s>>>(a + head, b + head, q, nvec);
        note_launch();
    }
    const uint64_t tail = body - nvec * 4;
    if (tail) { scale_cc_scalar<<<1, 32, 0, s>>>(a + head + nvec * 4, b + head + nvec * 4, q, tail); note_launch(); }
    return cudaGetLastError();
}

}  // namespace rlb
