// gen.cu -- deterministic input generators (device) and the K11 FP64 peak
// microbenchmarks.  The generators reproduce, bit for bit, the inputs that
// oracle/oracle.c builds on the host (counter-based RNG, common.cuh), so
// every GPU parity test and the benchmark create their inputs in HBM without
// a host round trip.
#include "common.cuh"
#include "kernels.h"

namespace rlb {
namespace {

__global__ void fill_uniform_kernel(double* __restrict__ out, uint64_t n, uint64_t key,
                                    uint64_t idx0, int kind) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const double u = u01(mix(key, idx0 + i));
        out[i] = kind ? 2.0 * u - 1.0 : u;
    }
}

// One thread per row: k distinct sorted columns in the band (rejection
// sampling in a fixed draw order, then insertion sort) -- BASELINE configs[1].
__global__ void gen_band_csr_kernel(uint64_t m_local, uint64_t row0, uint64_t n, uint32_t k,
                                    uint64_t hb, uint64_t kc, uint64_t kv, int* __restrict__ rp,
                                    int* __restrict__ col, double* __restrict__ val) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < m_local; r += stride) {
        const uint64_t i = row0 + r;
        const uint64_t lo = i > hb ? i - hb : 0;
        const uint64_t hi = (i + hb < n - 1) ? i + hb : n - 1;
        const uint64_t width = hi - lo + 1;
        int c[64];
        uint32_t cnt = 0;
        const uint64_t rowkey = mix(kc, i);
        for (uint64_t t = 0; cnt < k; ++t) {
            const uint64_t h = mix(rowkey, t);
            const uint64_t cand = lo + (((h >> 32) * width) >> 32);
            bool dup = false;
            for (uint32_t j = 0; j < cnt; ++j) dup |= (c[j] == (int)cand);
            if (!dup) c[cnt++] = (int)cand;
        }
        for (uint32_t a = 1; a < k; ++a) {
            const int v = c[a];
            int b = (int)a - 1;
            while (b >= 0 && c[b] > v) { c[b + 1] = c[b]; --b; }
            c[b + 1] = v;
        }
        for (uint32_t j = 0; j < k; ++j) {
            col[r * k + j] = c[j];
            val[r * k + j] = 2.0 * u01(mix(kv, i * k + j)) - 1.0;
        }
        rp[r] = (int)(r * k);
        if (r == m_local - 1) rp[m_local] = (int)(m_local * k);
    }
}

// Global grid nx * ny (* nz); the buffer holds outer indices [o0, o0 + n_outer).
__global__ void stencil_init_kernel(double* __restrict__ u, uint64_t nx, uint64_t ny,
                                    uint64_t nz, int dim, uint64_t o0, uint64_t n_outer,
                                    int radius, uint64_t key) {
    const uint64_t per_outer = dim == 2 ? nx : nx * ny;
    const uint64_t total = per_outer * n_outer;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t r = (uint64_t)radius;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += stride) {
        const uint64_t o = o0 + t / per_outer;  // global row (2D) or plane (3D)
        const uint64_t in = t % per_outer;
        const uint64_t x = in % nx;
        const uint64_t y = dim == 2 ? o : in / nx;
        const bool zin = dim == 2 || (o >= r && o + r < nz);
        const bool yin = y >= r && y + r < ny;
        const bool xin = x >= r && x + r < nx;
        const uint64_t g = o * per_outer + in;
        u[t] = (zin && yin && xin) ? u01(mix(key, g)) : 0.0;
    }
}

// K11a: DFMA throughput.  8 independent chains per thread.
__global__ void __launch_bounds__(256) peak_dfma(uint64_t iters, double* sink) {
    double a[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = 1.0 + 1e-9 * (threadIdx.x + j);
    const double m = 0.9999999999, c = 1e-12;
    for (uint64_t i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = fma(a[j], m, c);
    }
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += a[j];
    if (s == 42.0) sink[threadIdx.x] = s;  // never true; defeats dead-code elimination
}

// K11b: DMMA throughput.  4 independent m8n8k4 accumulation chains per warp.
__global__ void __launch_bounds__(256) peak_dmma(uint64_t iters, double* sink) {
    const double a = 1e-3 * (threadIdx.x & 31), b = 1e-3;
    double d[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
    for (uint64_t i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_m8n8k4(d[j][0], d[j][1], a, b, d[j][0], d[j][1]);
    }
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j) s += d[j][0] + d[j][1];
    if (s == 42.0) sink[threadIdx.x] = s;
}

unsigned grid_for(uint64_t n, int threads) {
    uint64_t b = (n + threads - 1) / threads;
    const uint64_t cap = (uint64_t)kNumSMs * 32;
    if (b > cap) b = cap;
    if (b == 0) b = 1;
    return (unsigned)b;
}

}  // namespace

cudaError_t launch_fill_uniform(double* out, uint64_t n, uint64_t seed, uint64_t stream_id,
                                uint64_t idx0, int kind, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    fill_uniform_kernel<<<grid_for(n, 256), 256, 0, s>>>(out, n, stream_key(seed, stream_id), idx0,
                                                         kind); note_launch();
    return cudaGetLastError();
}

cudaError_t launch_gen_band_csr(uint64_t m_local, uint64_t row0, uint64_t n, uint32_t k,
                                uint64_t hb, uint64_t seed, int* rp, int* col, double* val,
                                cudaStream_t s) {
    if (m_local == 0) return cudaMemsetAsync(rp, 0, sizeof(int), s);
    gen_band_csr_kernel<<<grid_for(m_local, 128), 128, 0, s>>>(
        m_local, row0, n, k, hb, stream_key(seed, 2), stream_key(seed, 3), rp, col, val); note_launch();
    return cudaGetLastError();
}

cudaError_t launch_stencil_init(double* u, uint64_t nx, uint64_t ny, uint64_t nz, int dim,
                                uint64_t outer_begin, uint64_t outer_end, int radius,
                                uint64_t seed, cudaStream_t s) {
    const uint64_t n_outer = outer_end - outer_begin;
    const uint64_t total = (dim == 2 ? nx : nx * ny) * n_outer;
    if (total == 0) return cudaSuccess;
    stencil_init_kernel<<<grid_for(total, 256), 256, 0, s>>>(u, nx, ny, nz, dim, outer_begin,
                                                             n_outer, radius, stream_key(seed, 5)); note_launch();
    return cudaGetLastError();
}

cudaError_t launch_fp64_peak(int unit, uint64_t iters, double* sink, double* flops,
                             cudaStream_t s) {
    const int threads = 256;
    const unsigned blocks = kNumSMs * 8;
    if (unit == 1) {
        peak_dmma<<<blocks, threads, 0, s>>>(iters, sink); note_launch();
        *flops = (double)blocks * (threads / 32) * (double)iters * 4.0 * 512.0;
    } else {
        peak_dfma<<<blocks, threads, 0, s>>>(iters, sink); note_launch();
        *flops = (double)blocks * threads * (double)iters * 8.0 * 2.0;
    }
    return cudaGetLastError();
}

}  // namespace rlb
