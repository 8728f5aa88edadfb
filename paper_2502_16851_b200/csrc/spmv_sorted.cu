// spmv_sorted.cu -- column-sorted block layout for the SpMV plan (K15).
//
// Why: CSR SpMV on the BASELINE band (16 random columns per row in a
// +-65,536 window) is bound by the L2 request rate of its x gathers, ~1
// random 8-byte gather per SM per cycle (profiles/README.md).  A warp
// instruction whose 32 gathers hit 32 different 128-byte lines costs 32 line
// lookups.  Visiting a block's nonzeros in COLUMN order packs them: a block of
// 16,384 nonzeros over ~132 K columns puts ~2 nonzeros in every line a warp
// touches, and tools/micro/sorted_gather.cu measures 539 G gathers/s against
// 281 G/s for the same columns unsorted.
//
// Layout (built once by rl_spmv_plan_create, host side below):
//   * rows are cut into blocks of <= 1024 rows whose "slot grid" maxlen x rows
//     fits CAP doubles of shared memory and whose column span is < 2^18;
//   * a block's nonzeros are stored sorted by column as (val f64, packed u32 =
//     (col - colbase) << 14 | slot) -- 12 B per nonzero, like CSR -- where
//     slot = j * rows + r for the j-th nonzero of block row r;
//   * the caller's row_ptr stays the row-length source.
// Kernel (one CTA per block, persistent over blocks):
//   phase 1: every thread takes nonzeros e = tid, tid + T, ... in column
//            order, gathers x, and stores val * x into prod[slot] (smem);
//   phase 2: thread r sums prod[j * rows + r], j = 0 .. len_r - 1, in row
//            order (deterministic, conflict-free: consecutive r, consecutive
//            slots) and stores y[r0 + r].
// Reference semantics: y[i] = sum_k val[k] x[col[k]] over row i's nonzeros
// (reference spmv_csr_model kernels.cpp:123-135 for the
// accounting) -- the same products, summed in CSR order per row.
#include <algorithm>
#include <thread>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace rlb {
namespace {

template <int CAP, int T>
__global__ void __launch_bounds__(T) spmv_sorted_kernel(const SpmvSBlock* __restrict__ blks, int b0, int b1,
                                                         const uint32_t* __restrict__ pk,
                                                         const double* __restrict__ sv,
                                                         const int32_t* __restrict__ rp,
                                                         const double* __restrict__ x, double* __restrict__ y) {
    extern __shared__ __align__(16) double prod[];
    const int tid = threadIdx.x;
    const uint64_t pol = policy_evict_first(), polx = policy_evict_last();
    for (int b = b0 + blockIdx.x; b < b1; b += gridDim.x) {
        const SpmvSBlock blk = blks[b];
        // phase-2 row bounds, loaded now so their latency hides under phase 1
        int rlo = 0, rhi = 0;
        if (tid < (int)blk.rows) {
            rlo = __ldg(rp + blk.r0 + tid);
            rhi = __ldg(rp + blk.r0 + tid + 1);
        }
        const uint32_t* p = pk + blk.kp;
        const double* v = sv + blk.kp;
        const double* xb = x + blk.colbase;
        constexpr int U = 8;
        int e = tid;
        for (; e + (U - 1) * T < blk.nent; e += U * T) {
            uint32_t q[U];
            double a[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
                    : "=r"(q[u]) : "l"(p + e + u * T), "l"(pol));
                asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
                    : "=d"(a[u]) : "l"(v + e + u * T), "l"(pol));
            }
            double g[U];
#pragma unroll
            for (int u = 0; u < U; ++u)
                asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(g[u]) : "l"(xb + (q[u] >> 14)), "l"(polx));
#pragma unroll
            for (int u = 0; u < U; ++u) prod[q[u] & 0x3fffu] = a[u] * g[u];
        }
        for (; e < blk.nent; e += T) {
            const uint32_t q = p[e];
            prod[q & 0x3fffu] = v[e] * __ldg(xb + (q >> 14));
        }
        __syncthreads();
        for (int r = tid; r < (int)blk.rows; r += T) {
            const uint32_t row = blk.r0 + (uint32_t)r;
            const int len = r == tid ? rhi - rlo : rp[row + 1] - rp[row];
            double s = 0.0;
            for (int j = 0; j < len; ++j) s += prod[j * (int)blk.rows + r];
            y[row] = s;
        }
        __syncthreads();
    }
}

// Software-pipelined variant: two product buffers; iteration i issues block
// i's streaming loads, then runs phase 2 of block i-1 from the other buffer
// while those loads are in flight, then gathers and scatters block i.  One
// barrier per block.  EPT = CAP / T entries per thread, all in flight at once.
template <int CAP, int T>
__global__ void __launch_bounds__(T, 1) spmv_sorted_pipe(const SpmvSBlock* __restrict__ blks, int b0, int b1,
                                                         const uint32_t* __restrict__ pk,
                                                         const double* __restrict__ sv,
                                                         const int32_t* __restrict__ rp,
                                                         const double* __restrict__ x, double* __restrict__ y) {
    constexpr int EPT = CAP / T;
    extern __shared__ __align__(16) double prod[];  // 2 x (CAP + 2)
    const int tid = threadIdx.x;
    const uint64_t pol = policy_evict_first(), polx = policy_evict_last();
    SpmvSBlock prev{};
    int plo = 0, phi = 0;
    bool have_prev = false;
    int it = 0;
    for (int b = b0 + blockIdx.x;; b += gridDim.x, ++it) {
        const bool have = b < b1;
        if (!have && !have_prev) break;
        SpmvSBlock blk{};
        uint32_t q[EPT];
        double a[EPT];
        int rlo = 0, rhi = 0;
        if (have) {
            blk = blks[b];
            if (tid < (int)blk.rows) {
                rlo = __ldg(rp + blk.r0 + tid);
                rhi = __ldg(rp + blk.r0 + tid + 1);
            }
#pragma unroll
            for (int u = 0; u < EPT; ++u) {
                const int e = tid + u * T;
                q[u] = 0;
                a[u] = 0.0;
                if (e < blk.nent) {
                    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
                        : "=r"(q[u]) : "l"(pk + blk.kp + e), "l"(pol));
                    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
                        : "=d"(a[u]) : "l"(sv + blk.kp + e), "l"(pol));
                }
            }
        }
        if (have_prev) {  // phase 2 of the previous block (other buffer)
            const double* pb = prod + ((it - 1) & 1) * (CAP + 2);
            if (tid < (int)prev.rows) {
                const int len = phi - plo;
                double sacc = 0.0;
                for (int j = 0; j < len; ++j) sacc += pb[j * (int)prev.rows + tid];
                y[prev.r0 + tid] = sacc;
            }
        }
        if (have) {
            double* pb = prod + (it & 1) * (CAP + 2);
            const double* xb = x + blk.colbase;
            double g[EPT];
#pragma unroll
            for (int u = 0; u < EPT; ++u)
                if (tid + u * T < blk.nent)
                    asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(g[u]) : "l"(xb + (q[u] >> 14)), "l"(polx));
#pragma unroll
            for (int u = 0; u < EPT; ++u)
                if (tid + u * T < blk.nent) pb[q[u] & 0x3fffu] = a[u] * g[u];
        }
        __syncthreads();
        prev = blk;
        plo = rlo;
        phi = rhi;
        have_prev = have;
    }
}

template <int CAP, int T>
cudaError_t launch_pipe(const SpmvSBlock* blks, int b0, int b1, const uint32_t* pk, const double* sv,
                        const int32_t* rp, const double* x, double* y, cudaStream_t s) {
    const size_t smem = (size_t)(CAP + 2) * 16;
    cudaError_t e = cudaFuncSetAttribute(spmv_sorted_pipe<CAP, T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    const int grid = std::max(1, std::min(b1 - b0, kNumSMs));
    spmv_sorted_pipe<CAP, T><<<grid, T, smem, s>>>(blks, b0, b1, pk, sv, rp, x, y);
    note_launch();
    return cudaGetLastError();
}

template <int CAP, int T>
cudaError_t launch_cfg(const SpmvSBlock* blks, int b0, int b1, const uint32_t* pk, const double* sv,
                       const int32_t* rp, const double* x, double* y, int ctas_per_sm, cudaStream_t s) {
    const size_t smem = (size_t)(CAP + 2) * 8;
    cudaError_t e = cudaFuncSetAttribute(spmv_sorted_kernel<CAP, T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    const int nb = b1 - b0;
    const int grid = std::max(1, std::min(nb, kNumSMs * ctas_per_sm));
    spmv_sorted_kernel<CAP, T><<<grid, T, smem, s>>>(blks, b0, b1, pk, sv, rp, x, y);
    note_launch();
    return cudaGetLastError();
}

}  // namespace

int spmv_sorted_cap() {
    const int c = tuning().spmv_sorted_cap;
    return c == 8192 || c == 12288 ? c : 16384;
}

bool spmv_sorted_build(uint64_t m, const int32_t* rp, const int32_t* col, const double* val, int cap,
                       std::vector<SpmvSBlock>& blks, std::vector<uint32_t>& pk, std::vector<double>& sv) {
    const uint64_t kMaxRows = cap == 12288 ? 768 : 1024, kSpan = 1u << 18;
    constexpr int kMaxLen = 64;
    blks.clear();
    // 1. blocks (sequential scan)
    uint64_t r = 0;
    while (r < m) {
        SpmvSBlock b{};
        b.r0 = (uint32_t)r;
        b.k0 = (uint64_t)rp[r];
        int maxlen = 0;
        int32_t lo = INT32_MAX, hi = INT32_MIN;
        uint64_t rows = 0;
        while (r + rows < m && rows < kMaxRows) {
            const uint64_t i = r + rows;
            const int len = rp[i + 1] - rp[i];
            if (len > kMaxLen) return false;  // long rows: the CSR kernels divert them; no sorted layout
            int32_t l2 = lo, h2 = hi;
            for (int32_t k = rp[i]; k < rp[i + 1]; ++k) {
                l2 = std::min(l2, col[k]);
                h2 = std::max(h2, col[k]);
            }
            const int ml = std::max(maxlen, len);
            if ((rows + 1) * (uint64_t)ml > (uint64_t)cap) break;
            if (h2 >= l2 && (uint64_t)((int64_t)h2 - l2) >= kSpan) break;
            maxlen = ml;
            lo = l2;
            hi = h2;
            ++rows;
        }
        if (rows == 0) return false;  // a single row that cannot fit (span >= 2^18)
        // a block padded to 32 entries needs the dummy slot cap - 1 outside its grid
        if (((rp[r + rows] - rp[r]) & 31) && rows * (uint64_t)maxlen >= (uint64_t)cap) {
            if (rows == 1) return false;
            --rows;
        }
        b.rows = (uint32_t)rows;
        b.colbase = hi >= lo ? lo : 0;
        b.nent = rp[r + rows] - rp[r];
        blks.push_back(b);
        r += rows;
    }
    // 2. padded offsets: every block starts on a 32-entry boundary (128-byte
    //    aligned packed columns, 256-byte aligned values);
    //    padding entries carry value 0 and the dummy slot cap - 1 (outside every slot grid)
    uint64_t kp = 0;
    for (auto& b : blks) {
        b.kp = kp;
        b.nent = (b.nent + 31) & ~31;
        kp += (uint64_t)b.nent;
    }
    // 3. per-block column sort (parallel over blocks)
    pk.assign(kp, (uint32_t)(cap - 1));
    sv.assign(kp, 0.0);
    const unsigned nth = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(), 64));
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < nth; ++t)
        pool.emplace_back([&, t] {
            std::vector<uint64_t> key;
            for (size_t bi = t; bi < blks.size(); bi += nth) {
                const SpmvSBlock& b = blks[bi];
                key.clear();
                for (uint32_t rr = 0; rr < b.rows; ++rr) {
                    const uint64_t i = b.r0 + rr;
                    for (int32_t k = rp[i]; k < rp[i + 1]; ++k) {
                        const uint64_t slot = (uint64_t)(k - rp[i]) * b.rows + rr;
                        // (column offset, slot, position in the block)
                        key.push_back(((uint64_t)(col[k] - b.colbase) << 46) | (slot << 32) |
                                      (uint64_t)(k - (int64_t)b.k0));
                    }
                }
                std::sort(key.begin(), key.end());
                for (size_t e = 0; e < key.size(); ++e) {
                    const uint64_t c = key[e] >> 46, slot = (key[e] >> 32) & 0x3fff, kk = key[e] & 0xffffffffu;
                    pk[b.kp + e] = (uint32_t)((c << 14) | slot);
                    sv[b.kp + e] = val[b.k0 + kk];
                }
            }
        });
    for (auto& th : pool) th.join();
    return true;
}

cudaError_t launch_spmv_sorted(const SpmvSBlock* blks, int b0, int b1, const uint32_t* pk, const double* sv,
                               const int32_t* rp, const double* x, double* y, int cap, cudaStream_t s) {
    if (b1 <= b0) return cudaSuccess;
    if (cap == 8192) return launch_cfg<8192, 512>(blks, b0, b1, pk, sv, rp, x, y, 3, s);
    if (cap == 12288) {
        if (tuning().spmv_sorted_pipe) return launch_pipe<12288, 768>(blks, b0, b1, pk, sv, rp, x, y, s);
        return launch_cfg<12288, 768>(blks, b0, b1, pk, sv, rp, x, y, 2, s);
    }
    return launch_cfg<16384, 1024>(blks, b0, b1, pk, sv, rp, x, y, 1, s);
}

}  // namespace rlb
