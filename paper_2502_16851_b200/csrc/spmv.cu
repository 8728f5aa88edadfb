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
#include <map>
#include <mutex>
#include <tuple>
#include <utility>

#include "common.cuh"
#include "kernels.h"

namespace rlb {
namespace {

// val / col streaming loads.  RLB_SPMV_STREAM_L1 = 1 lets them allocate in
// L1 (an experiment: L1::no_allocate scattered loads measured 2.4x slower
// than allocating ones, tools/micro/tma_gather.cu).
#ifndef RLB_SPMV_STREAM_L1
#define RLB_SPMV_STREAM_L1 0
#endif
#if RLB_SPMV_STREAM_L1
#define RLB_SP_NOALLOC ""
#else
#define RLB_SP_NOALLOC ".L1::no_allocate"
#endif
__device__ __forceinline__ d4 sp_ld4(const double* p, uint64_t pol) {
    d4 v;
    asm("ld.global.nc" RLB_SP_NOALLOC ".L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
        : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
        : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ int4 sp_ld4_i32(const int* p, uint64_t pol) {
    int4 ci;
    asm("ld.global.nc" RLB_SP_NOALLOC ".L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
        : "=r"(ci.x), "=r"(ci.y), "=r"(ci.z), "=r"(ci.w)
        : "l"(p), "l"(pol));
    return ci;
}
__device__ __forceinline__ double sp_ld(const double* p, uint64_t pol) {
    double v;
    asm("ld.global.nc" RLB_SP_NOALLOC ".L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ int sp_ld_i32(const int* p, uint64_t pol) {
    int v;
    asm("ld.global.nc" RLB_SP_NOALLOC ".L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}

struct Nz4 {
    double v[4];
    int c[4];
    int n;  // valid slots (a prefix); padded slots carry val = 0 and are never gathered
};

// Load the (up to) 4 nonzeros [j, j+4) of a row ending at e.
__device__ __forceinline__ Nz4 load_nz4(const int* __restrict__ col,
                                        const double* __restrict__ val, int64_t j, int64_t e,
                                        int col_pad, uint64_t pol, bool vec) {
    Nz4 z;
    if (vec && ((j & 3) == 0) && j + 4 <= e) {
        const d4 v = sp_ld4(val + j, pol);
        const int4 ci = sp_ld4_i32(col + j, pol);
        z.v[0] = v.x; z.v[1] = v.y; z.v[2] = v.z; z.v[3] = v.w;
        z.c[0] = ci.x; z.c[1] = ci.y; z.c[2] = ci.z; z.c[3] = ci.w;
        z.n = 4;
    } else {
        const int64_t left = e - j;
        z.n = left <= 0 ? 0 : (left >= 4 ? 4 : (int)left);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const bool ok = j + k < e;
            z.v[k] = ok ? sp_ld(val + j + k, pol) : 0.0;
            z.c[k] = ok ? sp_ld_i32(col + j + k, pol) : col_pad;
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

// Rows longer than lr.lmax nonzeros leave the per-row kernels (they would
// hold a warp for ~len/16 steps while its other rows finish in one): the
// lane that owns the row's start appends it, with its piece count, to the
// list (see LongRows), and spmv_long computes the pieces load-balanced.
// lr.ctr == nullptr disables the diversion.
__device__ __forceinline__ bool divert_long(const LongRows& lr, uint64_t row, int64_t& s, int64_t& e,
                                            bool leader) {
    if (lr.ctr == nullptr || e - s <= lr.lmax) return false;
    if (leader) {
        const unsigned long long np = (unsigned long long)((e - s + lr.piece - 1) / lr.piece);
        const unsigned long long old =
            atomicAdd(reinterpret_cast<unsigned long long*>(lr.ctr), (1ull << kLongIndexShift) | np);
        const unsigned i = (unsigned)(old >> kLongIndexShift);
        lr.rows[i] = (int)row;
        lr.base[i] = (unsigned)(old & ((1ull << kLongIndexShift) - 1));
    }
    e = s;
    return true;
}

// Nonzeros [j, j+4) clipped to [lo, hi): vector loads when aligned and whole.
struct Nz4m {
    double v[4];
    int c[4];
    bool ok[4];
};
__device__ __forceinline__ Nz4m load_nz4_rng(const int* __restrict__ col, const double* __restrict__ val,
                                             int64_t j, int64_t lo, int64_t hi, uint64_t pol, bool vec) {
    Nz4m z;
    if (vec && ((j & 3) == 0) && j >= lo && j + 4 <= hi) {
        const d4 v = sp_ld4(val + j, pol);
        const int4 ci = sp_ld4_i32(col + j, pol);
        z.v[0] = v.x; z.v[1] = v.y; z.v[2] = v.z; z.v[3] = v.w;
        z.c[0] = ci.x; z.c[1] = ci.y; z.c[2] = ci.z; z.c[3] = ci.w;
        z.ok[0] = z.ok[1] = z.ok[2] = z.ok[3] = true;
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            z.ok[k] = j + k >= lo && j + k < hi;
            z.v[k] = z.ok[k] ? sp_ld(val + j + k, pol) : 0.0;
            z.c[k] = z.ok[k] ? sp_ld_i32(col + j + k, pol) : 0;
        }
    }
    return z;
}
__device__ __forceinline__ void gather4m(double (&xv)[4], const Nz4m& z, const double* __restrict__ x,
                                         int64_t col_base, uint64_t polx) {
#pragma unroll
    for (int k = 0; k < 4; ++k) xv[k] = z.ok[k] ? ld_x(x + ((int64_t)z.c[k] - col_base), polx, 0) : 0.0;
}

// Sum of nonzeros [lo, hi) of one row by a group of GL lanes (GL = 32: the
// whole warp), valid in every lane of the group.  CUDA core: lanes stride
// 4-wide aligned groups; fixed-order xor reduction within the group.
template <int GL = 32>
__device__ __forceinline__ double group_segment_cc(const int* __restrict__ col, const double* __restrict__ val,
                                                   const double* __restrict__ x, int64_t col_base, int64_t lo,
                                                   int64_t hi, uint64_t pol, uint64_t polx, bool vec) {
    const int lane = threadIdx.x & 31, gl = lane & (GL - 1);
    const unsigned gmask = GL == 32 ? 0xffffffffu : (((1u << GL) - 1u) << (lane & ~(GL - 1)));
    constexpr int U = 4;  // 4 x 4 GL nonzeros in flight per group step (loads first, then gathers)
    double acc[U] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t j0 = (lo & ~int64_t(3)) + 4 * gl; j0 < hi; j0 += 4 * GL * U) {
        Nz4m z[U];
#pragma unroll
        for (int u = 0; u < U; ++u) z[u] = load_nz4_rng(col, val, j0 + 4 * GL * u, lo, hi, pol, vec);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            double xv[4];
            gather4m(xv, z[u], x, col_base, polx);
#pragma unroll
            for (int k = 0; k < 4; ++k) acc[u] = fma(z[u].v[k], xv[k], acc[u]);
        }
    }
    double a = (acc[0] + acc[1]) + (acc[2] + acc[3]);
#pragma unroll
    for (int o = GL / 2; o; o >>= 1) a += __shfl_xor_sync(gmask, a, o);
    return a;
}

// Tensor core, eight independent segments at once: virtual row r of the
// DASP-style block (lanes 4r..4r+3) walks its own [lo, hi) (the lanes of a
// virtual row pass the same range; empty ranges are allowed).  Returns
// virtual row r's sum, valid in lane 4r + r/2 (where D[r][r] lives).
__device__ __forceinline__ double warp_multi_tc(const int* __restrict__ col, const double* __restrict__ val,
                                                const double* __restrict__ x, int64_t col_base, int64_t lo,
                                                int64_t hi, uint64_t pol, uint64_t polx, bool vec) {
    const int lane = threadIdx.x & 31, r = lane >> 2, c = lane & 3;
    const int64_t base = lo & ~int64_t(3);
    constexpr int U = 4;  // 4 steps of 16 per virtual row in flight
    double d0[U] = {0.0, 0.0, 0.0, 0.0}, d1[U] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t off0 = 0; __any_sync(0xffffffffu, base + off0 < hi); off0 += 16 * U) {
        Nz4m z[U];
#pragma unroll
        for (int u = 0; u < U; ++u) z[u] = load_nz4_rng(col, val, base + off0 + 16 * u + 4 * c, lo, hi, pol, vec);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            double xv[4];
            gather4m(xv, z[u], x, col_base, polx);
            dmma_m8n8k4(d0[u], d1[u], z[u].v[0], xv[0], d0[u], d1[u]);
            dmma_m8n8k4(d0[u], d1[u], z[u].v[1], xv[1], d0[u], d1[u]);
            dmma_m8n8k4(d0[u], d1[u], z[u].v[2], xv[2], d0[u], d1[u]);
            dmma_m8n8k4(d0[u], d1[u], z[u].v[3], xv[3], d0[u], d1[u]);
        }
    }
    const double e0 = (d0[0] + d0[1]) + (d0[2] + d0[3]), e1 = (d1[0] + d1[1]) + (d1[2] + d1[3]);
    return (r & 1) ? e1 : e0;
}

// Longest row of [r0, r1): the one-time probe behind row_profile().
__global__ void __launch_bounds__(256) spmv_maxlen(uint64_t r0, uint64_t r1, const int* __restrict__ rp,
                                                   int* __restrict__ out) {
    int m = 0;
    for (uint64_t i = r0 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < r1;
         i += (uint64_t)gridDim.x * blockDim.x)
        m = max(m, __ldg(rp + i + 1) - __ldg(rp + i));
    m = (int)__reduce_max_sync(0xffffffffu, (unsigned)m);
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// The diverted rows, after the per-row kernel (stream order).  Warp w of W
// takes the contiguous run of pieces [w P/W, (w+1) P/W) -- pieces are at
// most lr.piece nonzeros, so the runs balance whatever the row lengths.  It
// finds its first row with a 32-ary search over base[] (3 round trips for
// 32 K rows), then its groups of GL lanes (CUDA core: 8, so four pieces --
// e.g. four short rows -- are in flight per warp; tensor core: the whole
// warp) walk the run, group j taking every (32/GL)-th piece.  A row of one
// piece is stored directly; a split row's pieces go to part[] and the group
// that finishes the row's last piece adds them in piece order, so the result
// does not depend on timing.  (A split row past the part[] capacity is done
// whole by its first piece's group.)  The last CTA out zeroes the counters
// for the next call on this stream, so no memset node is needed.
template <int TC, int GL>
__global__ void __launch_bounds__(256, 2) spmv_long(const int* __restrict__ rp, const int* __restrict__ col,
                                                     const double* __restrict__ val, const double* __restrict__ x,
                                                     int64_t col_base, double* __restrict__ y, LongRows lr) {
    static_assert(!TC || GL == 32, "the tensor-core block spans the whole warp (eight pieces, one per virtual row)");
    constexpr int NG = 32 / GL;
    const int tid = threadIdx.x, lane = tid & 31, grp = lane / GL, gl = lane & (GL - 1);
    const uint64_t pol = policy_evict_first(), polx = policy_evict_last();
    const unsigned long long c = *reinterpret_cast<volatile unsigned long long*>(lr.ctr);
    const unsigned nlong = (unsigned)(c >> kLongIndexShift);
    const uint64_t npieces = c & ((1ull << kLongIndexShift) - 1);
    const uint64_t W = (uint64_t)gridDim.x * (blockDim.x >> 5);
    const uint64_t w = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (tid >> 5);
    const uint64_t g0 = npieces * w / W, g1 = npieces * (w + 1) / W;
    if (g0 < g1) {
        // last list index i with base[i] <= g0: 32-ary search
        unsigned lo = 0, hi = nlong;  // answer in [lo, hi)
        while (hi - lo > 1) {
            const unsigned span = hi - lo, step = (span + 31) / 32;
            const unsigned probe = lo + lane * step;
            const bool le = probe < hi && __ldg(lr.base + probe) <= g0;
            const unsigned ball = __ballot_sync(0xffffffffu, le);
            const int k = 31 - __clz(ball);  // lane 0 always qualifies (base[lo] <= g0)
            lo = lo + (unsigned)k * step;
            hi = min(hi, lo + step);
        }
        unsigned i = lo;
        uint64_t b_i = __ldg(lr.base + i);
        uint64_t b_n = i + 1 < nlong ? __ldg(lr.base + i + 1) : npieces;
        // TC: virtual row r (lanes 4r..4r+3) takes piece gb + r of each batch
        // of 8; CC: group grp takes every NG-th piece.
        constexpr int STRIDE = TC ? 8 : NG;
        const int slot = TC ? (lane >> 2) : grp;
        const uint64_t gend = TC ? g0 + (g1 - g0 + 7) / 8 * 8 : g1;  // TC: whole batches (the warp stays converged)
        for (uint64_t g = g0 + slot; g < gend; g += STRIDE) {
            const bool live = g < g1;
            int row = 0;
            int64_t a = 0, bnd = 0;
            uint64_t np = 0;
            bool whole = true;
            if (live) {
                while (g >= b_n) {
                    ++i;
                    b_i = b_n;
                    b_n = i + 1 < nlong ? __ldg(lr.base + i + 1) : npieces;
                }
                row = lr.rows[i];
                const int64_t s = __ldg(rp + row), e = __ldg(rp + row + 1);
                np = b_n - b_i;
                const uint64_t q = g - b_i;
                whole = np == 1 || b_n > lr.pcap;  // unsplit, or past capacity: done by piece 0's lanes
                if (!whole || q == 0) {
                    a = whole ? s : s + (int64_t)q * lr.piece;
                    bnd = whole ? e : min(e, a + lr.piece);
                } else {
                    row = -1;  // a later piece of a row done whole: nothing to do
                }
            } else {
                row = -1;
            }
            if constexpr (!TC) {
                if (row < 0) continue;
            }
            double v;
            bool leader;
            if constexpr (TC) {
                v = warp_multi_tc(col, val, x, col_base, a, bnd, pol, polx, lr.vec);
                leader = lane == 4 * slot + (slot >> 1);
            } else {
                v = group_segment_cc<GL>(col, val, x, col_base, a, bnd, pol, polx, lr.vec);
                leader = gl == 0;
            }
            if (!leader || row < 0) continue;
            if (whole) {
                y[row] = v;
                continue;
            }
            lr.part[g] = v;
            __threadfence();
            if (atomicAdd(lr.done + i, 1u) == (unsigned)np - 1) {  // the row's last piece: sum in order
                __threadfence();
                double r = 0.0;
                for (uint64_t p = b_i; p < b_n; ++p) r += *reinterpret_cast<volatile double*>(lr.part + p);
                y[row] = r;
                lr.done[i] = 0;
            }
        }
    }
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        if (atomicAdd(lr.ctr + 2, 1u) == gridDim.x - 1) {
            *reinterpret_cast<unsigned long long*>(lr.ctr) = 0ull;
            lr.ctr[2] = 0;
        }
    }
}

// K3: CUDA core.  Row of warp-step u for group q: wbase + 8u + q.
// SCHED 0: warps stride over the whole row range (grid-stride);
// SCHED 1: each CTA owns one contiguous row range (x-window locality in L1).
template <int R, int SCHED, int XH, bool DIV>
__global__ void __launch_bounds__(1024) spmv_cc_v4(uint64_t r0, uint64_t r1,
                                                  const int* __restrict__ rp,
                                                  const int* __restrict__ col,
                                                  const double* __restrict__ val,
                                                  const double* __restrict__ x, int64_t col_base,
                                                  double* __restrict__ y, LongRows lr) {
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
        // rows past 16 nonzeros only: the diversion check stays off the
        // BASELINE path (16 per row), whose first 16 are loaded regardless
        bool skip[R];
#pragma unroll
        for (int u = 0; u < R; ++u)
            skip[u] = DIV && e[u] - s[u] > 16 && divert_long(lr, wbase + 8 * u + q, s[u], e[u], c == 0);
        Nz4 z[R];
#pragma unroll
        for (int u = 0; u < R; ++u) z[u] = load_nz4(col, val, s[u] + 4 * c, e[u], col_pad, pol, lr.vec);
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
                Nz4 t = load_nz4(col, val, j, e[u], col_pad, pol, lr.vec);
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
            if (c == 0 && row < rend && !skip[u]) y[row] = a;
        }
    }
}

// K4: tensor core.  A warp owns RB 8-row blocks per iteration (independent
// DMMA accumulator chains); SCHED as in K3.
template <int RB, int SCHED, bool DIV>
__global__ void __launch_bounds__(1024) spmv_tc(uint64_t r0, uint64_t r1,
                                                const int* __restrict__ rp,
                                                const int* __restrict__ col,
                                                const double* __restrict__ val,
                                                const double* __restrict__ x, int64_t col_base,
                                                double* __restrict__ y, LongRows lr) {
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
        bool skip[RB];
        int len = 0;
#pragma unroll
        for (int q = 0; q < RB; ++q) {
            const uint64_t row = base + 8 * q + r;
            const bool ok = row < last;
            s[q] = ok ? __ldg(rp + row) : 0;
            e[q] = ok ? __ldg(rp + row + 1) : 0;
            skip[q] = DIV && divert_long(lr, row, s[q], e[q], c == 0);  // long rows leave the 8-row block
            len = max(len, (int)(e[q] - s[q]));
        }
        const int maxlen = __reduce_max_sync(0xffffffffu, len);
        double d0[RB], d1[RB];
#pragma unroll
        for (int q = 0; q < RB; ++q) d0[q] = d1[q] = 0.0;
        for (int off = 0; off < maxlen; off += 16) {
            Nz4 z[RB];
#pragma unroll
            for (int q = 0; q < RB; ++q) z[q] = load_nz4(col, val, s[q] + off + 4 * c, e[q], col_pad, pol, lr.vec);
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
            if (c == (r >> 1) && row < last && !skip[q]) y[row] = (r & 1) ? d1[q] : d0[q];
        }
    }
}

}  // namespace

// Has the CSR row range rows the per-row kernels divert?  Probed once per
// (device, row_ptr, col, val, range): one small kernel and one stream
// synchronisation on the first call, then cached (the longest row; the
// answer follows the current spmv_long_min), so later calls stay fully
// asynchronous and pay nothing when there are none.  A stale entry (arrays
// rewritten in place at the same addresses) costs speed only: undiverted
// long rows are still computed by the per-row kernels, and a needless
// diversion pass finds an empty list.  Under stream capture the probe is
// skipped (-1: divert on the device).
static int row_profile(const int* rp, const int* col, const double* val, uint64_t r0, uint64_t r1,
                       cudaStream_t s) {
    struct Key {
        int dev;
        const void *rp, *col, *val;
        uint64_t r0, r1;
        bool operator<(const Key& o) const {
            return std::tie(dev, rp, col, val, r0, r1) < std::tie(o.dev, o.rp, o.col, o.val, o.r0, o.r1);
        }
    };
    static std::mutex mu;
    static std::map<Key, int> cache;   // longest row
    static std::map<int, int*> slots;  // per-device probe result
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return -1;
    const Key key{dev, rp, col, val, r0, r1};
    std::lock_guard<std::mutex> lock(mu);
    const auto it = cache.find(key);
    if (it != cache.end()) return it->second > tuning().spmv_long_min ? 1 : 0;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return -1;
    int*& slot = slots[dev];
    if (!slot && cudaMalloc(&slot, sizeof(int)) != cudaSuccess) {
        slot = nullptr;
        cudaGetLastError();
        return -1;
    }
    int h = 0;
    if (cudaMemsetAsync(slot, 0, sizeof(int), s) != cudaSuccess) return -1;
    spmv_maxlen<<<kNumSMs * 4, 256, 0, s>>>(r0, r1, rp, slot);
    note_launch();
    if (cudaMemcpyAsync(&h, slot, sizeof(int), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
        return -1;
    if (cache.size() >= 1024) cache.clear();
    cache[key] = h;
    return h > tuning().spmv_long_min ? 1 : 0;
}

int spmv_long_rows_probe(const int* rp, const int* col, const double* val, uint64_t r0, uint64_t r1,
                         cudaStream_t s) {
    return r1 > r0 ? row_profile(rp, col, val, r0, r1, s) : 0;
}

cudaError_t launch_spmv(int unit, uint64_t r0, uint64_t r1, const int* rp, const int* col,
                        const double* val, const double* x, int64_t col_base, double* y,
                        int long_rows, cudaStream_t s) {
    if (r1 <= r0) return cudaSuccess;
    const Tuning& t = tuning();
    if (long_rows < 0 && t.spmv_long_rows) long_rows = row_profile(rp, col, val, r0, r1, s);
    // long-row diversion (long_rows: -1 unknown, 0 none, 1 present)
    LongRows lr{};
    // 256-bit val / 128-bit col loads need 32- / 16-byte aligned base
    // pointers (a view at an offset may not be): else element loads only
    lr.vec = (reinterpret_cast<uintptr_t>(val) & 31) == 0 && (reinterpret_cast<uintptr_t>(col) & 15) == 0;
    if (long_rows != 0 && t.spmv_long_rows) {
        cudaError_t e = spmv_long_workspace(s, r1 - r0, lr);
        if (e != cudaSuccess) return e;
        lr.lmax = t.spmv_long_min;
        lr.piece = t.spmv_long_piece > 64 ? t.spmv_long_piece : 64;
    }
    cudaError_t err = launch_spmv_rows(unit, r0, r1, rp, col, val, x, col_base, y, lr, s);
    if (err != cudaSuccess || lr.ctr == nullptr) return err;
    if (unit == 1)
        spmv_long<1, 32><<<kNumSMs * 2, 256, 0, s>>>(rp, col, val, x, col_base, y, lr);
    else if (t.spmv_long_group == 32)
        spmv_long<0, 32><<<kNumSMs * 2, 256, 0, s>>>(rp, col, val, x, col_base, y, lr);
    else if (t.spmv_long_group == 16)
        spmv_long<0, 16><<<kNumSMs * 2, 256, 0, s>>>(rp, col, val, x, col_base, y, lr);
    else
        spmv_long<0, 8><<<kNumSMs * 2, 256, 0, s>>>(rp, col, val, x, col_base, y, lr);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_spmv_rows(int unit, uint64_t r0, uint64_t r1, const int* rp, const int* col,
                             const double* val, const double* x, int64_t col_base, double* y,
                             const LongRows& lr, cudaStream_t s) {
    const Tuning& t = tuning();
    const uint64_t rows = r1 - r0;
    if (unit == 1) {
        const int tthreads = t.spmv_tc_threads, RB = t.spmv_tc_rows;
        uint64_t blocks = (rows + (uint64_t)(tthreads / 32) * 8 * RB - 1) / ((uint64_t)(tthreads / 32) * 8 * RB);
        const uint64_t cap = (uint64_t)kNumSMs * (uint64_t)t.spmv_tc_blocks_per_sm;
        if (blocks > cap) blocks = cap;
#define RLB_TC(R, S)                                                                                        \
    do {                                                                                                    \
        if (lr.ctr) spmv_tc<R, S, true><<<(unsigned)blocks, tthreads, 0, s>>>(r0, r1, rp, col, val, x, col_base, y, lr); \
        else spmv_tc<R, S, false><<<(unsigned)blocks, tthreads, 0, s>>>(r0, r1, rp, col, val, x, col_base, y, lr); \
    } while (0)
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
#define RLB_SPMV2(RR, SS, XX, DV)                                                                      \
    do {                                                                                                \
        if (t.spmv_l1_carveout >= 0)                                                                    \
            cudaFuncSetAttribute(spmv_cc_v4<RR, SS, XX, DV>,                                            \
                                 cudaFuncAttributePreferredSharedMemoryCarveout, t.spmv_l1_carveout);   \
        spmv_cc_v4<RR, SS, XX, DV><<<(unsigned)blocks, cthreads, 0, s>>>(r0, r1, rp, col, val, x, col_base, y, lr); \
    } while (0)
#define RLB_SPMV(RR, SS, XX) \
    do { if (lr.ctr) RLB_SPMV2(RR, SS, XX, true); else RLB_SPMV2(RR, SS, XX, false); } while (0)
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
#undef RLB_SPMV2
    note_launch();
    return cudaGetLastError();
}

namespace {
struct LongWs {
    unsigned* ctr = nullptr;
    int* rows = nullptr;
    unsigned* base = nullptr;
    double* part = nullptr;
    unsigned* done = nullptr;
    uint64_t cap = 0;
};
}  // namespace

cudaError_t spmv_long_workspace(cudaStream_t s, uint64_t rows, LongRows& lr) {
    static std::mutex mu;
    static std::map<std::pair<int, cudaStream_t>, LongWs> table;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    LongWs& w = table[{dev, s}];
    if (w.cap < rows) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if ((e = cudaStreamIsCapturing(s, &cs)) != cudaSuccess) return e;
        if (cs != cudaStreamCaptureStatusNone) return cudaErrorStreamCaptureUnsupported;  // reserve first
        if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;  // old buffers may be in flight
        if (w.ctr) cudaFree(w.ctr);
        if (w.rows) cudaFree(w.rows);
        if (w.base) cudaFree(w.base);
        if (w.part) cudaFree(w.part);
        if (w.done) cudaFree(w.done);
        w = LongWs{};
        const uint64_t cap = rows < 65536 ? 65536 : rows;  // list entries and split pieces
        if ((e = cudaMalloc(&w.ctr, 8 * sizeof(unsigned))) != cudaSuccess) return e;
        if ((e = cudaMemset(w.ctr, 0, 8 * sizeof(unsigned))) != cudaSuccess) return e;
        if ((e = cudaMalloc(&w.rows, cap * sizeof(int))) != cudaSuccess) return e;
        if ((e = cudaMalloc(&w.base, cap * sizeof(unsigned))) != cudaSuccess) return e;
        if ((e = cudaMalloc(&w.part, cap * sizeof(double))) != cudaSuccess) return e;
        if ((e = cudaMalloc(&w.done, cap * sizeof(unsigned))) != cudaSuccess) return e;
        if ((e = cudaMemset(w.done, 0, cap * sizeof(unsigned))) != cudaSuccess) return e;
        w.cap = cap;
    }
    lr.ctr = w.ctr;
    lr.rows = w.rows;
    lr.base = w.base;
    lr.part = w.part;
    lr.done = w.done;
    lr.pcap = w.cap;
    return cudaSuccess;
}

}  // namespace rlb
