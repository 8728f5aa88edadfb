// spmv_colsort.cu -- K17: the SpMV plan's column-sorted row-block layout.
//
// Why: on the BASELINE band matrix the CSR kernels (spmv.cu) are bound by one
// L1 request per x gather (67.1 M random 8-byte gathers per call, ~1 per SM
// per cycle), not by HBM.  Here a block of R rows keeps its nonzeros sorted
// by COLUMN, so a warp instruction's 32 consecutive entries read x from a
// few L1 lines (~40 columns at R ~ 7000 and 16 nonzeros per row) instead of
// 32 random ones; the products are added into the block's y rows held in
// shared memory.
//
// Layout (built once on the host by rl_spmv_plan_create; bytes <= CSR's):
//   val  f64  per entry
//   meta u32  per entry = (col - block.col_lo) << rb | (row - block.row0)
//   blocks    {first entry, col_lo, row0, rows, entries}; entries padded to a
//             multiple of 32 with (val = 0, column col_lo, row = rows): the
//             padding adds into a scratch slot past the block's rows that is
//             never written back.
// Within each window of 128 sorted entries the host orders the entries so
// every aligned half-warp of 16 has distinct row % 16 where the window allows:
// the 64-bit shared-memory accesses of a half-warp then hit distinct bank
// pairs (tools/micro/spmv_colsort.cu: 0.2017 -> 0.1829 ms).
//
// CUDA core: 1024-thread CTAs, two per SM (y rows <= 8192 -> 64 KB each),
// persistent over the blocks; each thread streams entries e, e+1024, e+2048
// (val/meta evict_first, x gathers evict_last so x stays in L2), multiplies
// and adds into its row with a shared-memory FP64 atomicAdd (a CAS loop on
// sm_100a): FP64 arithmetic throughout, but the order of a row's additions is
// not fixed, so repeated calls may differ in the last bits (within the 1e-12
// norm-wise tolerance; the CSR kernels are the bit-reproducible path).
// Measured alternatives (profiles/spmv_colsort_r2.md): exact 96-bit
// fixed-point rows on native 32-bit shared atomics (bit-reproducible) ran
// 0.185-0.21 ms -- the three atomics per entry saturate the MIO queue -- and a
// 64-bit grid 0.154 ms but loses relative precision on rows far below their
// block's largest product.
// Tensor core: the same layout and accumulation; the 32 products of a warp
// step come out of 4 DMMA m8n8k4 (A and B masked to the k = j slot: lane
// 4c+j's product is D_j[c][c]; 8 of the 64 outputs of each MMA are useful,
// the most a K = 4 product of per-entry operands allows), shuffled back to
// their lanes for the same shared-memory add.
#include <algorithm>
#include <cstring>
#include <thread>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace rlb {

namespace {
constexpr int kThreads = 1024;
constexpr int kUnroll = 3;  // entry loads in flight per thread (measured: U2 0.183, U3 0.173, U4 0.193 ms)

__device__ __forceinline__ unsigned ld_meta(const unsigned* p, uint64_t pol) {
    unsigned v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}

template <bool TC>
__global__ void __launch_bounds__(kThreads, 2)
    spmv_colsort(const SpmvKBlock* __restrict__ blks, int b0, int b1, int rb, const double* __restrict__ val,
                 const unsigned* __restrict__ meta, const double* __restrict__ x, double* __restrict__ y) {
    extern __shared__ double ys[];
    const unsigned rmask = (1u << rb) - 1;
    const uint64_t pol = policy_evict_first(), polx = policy_evict_last();
    const int lane = threadIdx.x & 31;
    for (int b = b0 + blockIdx.x; b < b1; b += gridDim.x) {
        const SpmvKBlock blk = blks[b];
        for (unsigned i = threadIdx.x; i <= blk.rows; i += kThreads) ys[i] = 0.0;  // + the padding slot
        __syncthreads();
        const double* xb = x + blk.col_lo;
        const double* vb = val + blk.e0;
        const unsigned* mb = meta + blk.e0;
        auto step = [&](double v, unsigned mt, double xv) {
            if (!TC) {
                atomicAdd(&ys[mt & rmask], v * xv);
            } else {
                // product of lane 4c+j is D_j[c][c], held by lane 4c + (c >> 1) in slot c & 1;
                // one shuffle per MMA brings it back to lane 4c+j, then one full-warp add
                const int c = lane >> 2;
                const int home = 4 * c + (c >> 1);
                double p = 0.0;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    // both operands masked to the k = j slot, so an Inf/NaN of another
                    // entry never meets a zero of this one (Inf * 0 = NaN)
                    double d0, d1;
                    const bool mine = (lane & 3) == j;
                    dmma_m8n8k4(d0, d1, mine ? v : 0.0, mine ? xv : 0.0, 0.0, 0.0);
                    const double q = __shfl_sync(0xffffffffu, (c & 1) ? d1 : d0, home);
                    if (mine) p = q;
                }
                atomicAdd(&ys[mt & rmask], p);
            }
        };
        // nent is a multiple of 32: every warp step is full
        unsigned e = threadIdx.x;
        constexpr int U = TC ? 2 : kUnroll;  // the tensor-core step needs more registers
        for (; e + (U - 1) * kThreads < blk.nent; e += U * kThreads) {
            double v[U], xv[U];
            unsigned mt[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                v[u] = ld_stream(vb + e + u * kThreads, pol);
                mt[u] = ld_meta(mb + e + u * kThreads, pol);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) xv[u] = ld_policy(xb + (mt[u] >> rb), polx);
#pragma unroll
            for (int u = 0; u < U; ++u) step(v[u], mt[u], xv[u]);
        }
        // tail: whole warps only (nent is a multiple of 32), so the TC shuffles stay full
        for (; e - lane < blk.nent; e += kThreads) {
            const double v = ld_stream(vb + e, pol);
            const unsigned mt = ld_meta(mb + e, pol);
            step(v, mt, ld_policy(xb + (mt >> rb), polx));
        }
        __syncthreads();
        for (unsigned i = threadIdx.x; i < blk.rows; i += kThreads) y[blk.row0 + i] = ys[i];
        __syncthreads();
    }
}

// Order the entries of one window so that each aligned group of 16 (a
// half-warp of 64-bit shared accesses) takes one entry from as many distinct
// row % 16 classes (bank pairs) as the window has, largest classes first.
void bank_order(std::vector<std::pair<uint64_t, double>>& t, size_t w0, size_t w1, unsigned rmask,
                std::vector<std::pair<uint64_t, double>>& out) {
    std::vector<std::pair<uint64_t, double>> cls[16];
    for (size_t i = w0; i < w1; ++i) cls[(t[i].first & rmask) & 15].push_back(t[i]);
    size_t left = w1 - w0;
    out.clear();
    while (left) {
        int order[16];
        for (int c = 0; c < 16; ++c) order[c] = c;
        std::stable_sort(order, order + 16, [&](int a, int b) { return cls[a].size() > cls[b].size(); });
        int taken = 0;
        for (int oi = 0; oi < 16 && left; ++oi) {
            auto& c = cls[order[oi]];
            if (c.empty()) continue;
            out.push_back(c.back());
            c.pop_back();
            --left;
            ++taken;
        }
        while (taken < 16 && left) {  // fewer than 16 classes left: conflicts unavoidable
            int big = 0;
            for (int c = 1; c < 16; ++c)
                if (cls[c].size() > cls[big].size()) big = c;
            out.push_back(cls[big].back());
            cls[big].pop_back();
            --left;
            ++taken;
        }
    }
    std::copy(out.begin(), out.end(), t.begin() + w0);
}
}  // namespace

bool spmv_colsort_build(uint64_t m, uint64_t n, const int32_t* rp, const int32_t* col, const double* val,
                        SpmvColsortLayout& L, const std::vector<ColsortSegment>& segments_in) {
    (void)n;
    if (m == 0 || rp[m] == 0) return false;
    int64_t maxlen = 0;
    for (uint64_t i = 0; i < m; ++i) maxlen = std::max<int64_t>(maxlen, (int64_t)rp[i + 1] - rp[i]);
    if (maxlen > kColsortMaxRowLen) return false;  // one hot row would serialise its block's atomics
    // Default: one segment of two waves of two CTAs per SM (tools/micro/spmv_colsort.cu: 2 waves 0.173 ms,
    // 3 waves 0.191 ms at 2^22 rows).  Each segment's rows are cut into `blocks` equal blocks of at most
    // kColsortMaxRows (64 KB of y); all blocks are halved while a block's column span does not fit the
    // meta word.
    std::vector<ColsortSegment> segs = segments_in;
    if (segs.empty()) segs.push_back({m, 4 * (uint64_t)kNumSMsHost});
    for (int halve = 0;; ++halve) {
        std::vector<std::pair<uint64_t, uint64_t>> cut;  // (row0, rows)
        uint64_t seg0 = 0, Rmax = 1;
        for (const auto& sg : segs) {
            const uint64_t len = std::min(sg.row_end, m) - std::min(seg0, m);
            if (len) {
                uint64_t R = (len + sg.blocks - 1) / std::max<uint64_t>(1, sg.blocks);
                R = std::max<uint64_t>(32, std::min<uint64_t>(R, kColsortMaxRows)) >> halve;
                if (R < 1) return false;
                for (uint64_t r = seg0; r < seg0 + len; r += R) cut.push_back({r, std::min(R, seg0 + len - r)});
                Rmax = std::max(Rmax, R);
            }
            seg0 = std::max(seg0, std::min(sg.row_end, m));
        }
        if (seg0 < m || Rmax < 8) return false;
        int rb = 0;  // row field: 0..R (R = the padding's scratch slot)
        while ((1ull << rb) <= Rmax) ++rb;
        const uint64_t nb = cut.size();
        bool fits = true;
        for (uint64_t b = 0; b < nb && fits; ++b) {
            const uint64_t r0 = cut[b].first, r1 = r0 + cut[b].second;
            int32_t lo = INT32_MAX, hi = INT32_MIN;
            for (int64_t j = rp[r0]; j < rp[r1]; ++j) lo = std::min(lo, col[j]), hi = std::max(hi, col[j]);
            if (hi >= lo && (uint64_t)(hi - lo) >= (1ull << (32 - rb))) fits = false;
        }
        if (!fits) continue;
        L.rb = rb;
        L.rows = (int)Rmax;
        L.blocks.assign(nb, SpmvKBlock{});
        uint64_t e = 0;
        for (uint64_t b = 0; b < nb; ++b) {
            const uint64_t r0 = cut[b].first, r1 = r0 + cut[b].second;
            const uint64_t cnt = (uint64_t)(rp[r1] - rp[r0]);
            SpmvKBlock& k = L.blocks[b];
            k.e0 = e;
            k.row0 = (uint32_t)r0;
            k.rows = (uint32_t)(r1 - r0);
            k.nent = (uint32_t)((cnt + 31) / 32 * 32);
            int32_t lo = INT32_MAX;
            for (int64_t j = rp[r0]; j < rp[r1]; ++j) lo = std::min(lo, col[j]);
            k.col_lo = cnt ? lo : 0;
            e += k.nent;
        }
        L.val.assign(e, 0.0);
        L.meta.assign(e, 0u);
        const unsigned rmask = (1u << rb) - 1;
        auto work = [&](uint64_t bfirst, uint64_t bstep) {
            std::vector<std::pair<uint64_t, double>> t, scratch;
            for (uint64_t b = bfirst; b < nb; b += bstep) {
                const SpmvKBlock& k = L.blocks[b];
                const uint64_t r0 = k.row0, r1 = r0 + k.rows;
                t.clear();
                for (uint64_t r = r0; r < r1; ++r)
                    for (int64_t j = rp[r]; j < rp[r + 1]; ++j)
                        t.push_back({((uint64_t)(col[j] - k.col_lo) << rb) | (r - r0), val[j]});
                std::sort(t.begin(), t.end(), [](const auto& a, const auto& c) { return a.first < c.first; });
                const size_t win = (size_t)std::max(32, tuning().spmv_colsort_window);
                for (size_t w0 = 0; w0 < t.size(); w0 += win)
                    bank_order(t, w0, std::min(t.size(), w0 + win), rmask, scratch);
                for (size_t i = 0; i < t.size(); ++i) {
                    L.meta[k.e0 + i] = (uint32_t)t[i].first;
                    L.val[k.e0 + i] = t[i].second;
                }
                for (size_t i = t.size(); i < k.nent; ++i) L.meta[k.e0 + i] = k.rows;  // scratch slot
            }
        };
        const unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
        std::vector<std::thread> pool;
        for (unsigned i = 1; i < nt; ++i) pool.emplace_back(work, i, nt);
        work(0, nt);
        for (auto& th : pool) th.join();
        return true;
    }
}

cudaError_t launch_spmv_colsort(int unit, const SpmvKBlock* blks, int b0, int b1, int rb, int rows,
                                const double* val, const unsigned* meta, const double* x, double* y,
                                cudaStream_t s) {
    if (b1 <= b0) return cudaSuccess;
    const size_t smem = (size_t)(rows + 1) * 8;
    const int grid = std::min(b1 - b0, 2 * kNumSMs);
    cudaError_t e;
    if (unit) {
        e = cudaFuncSetAttribute(spmv_colsort<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        spmv_colsort<true><<<grid, kThreads, smem, s>>>(blks, b0, b1, rb, val, meta, x, y);
    } else {
        e = cudaFuncSetAttribute(spmv_colsort<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        spmv_colsort<false><<<grid, kThreads, smem, s>>>(blks, b0, b1, rb, val, meta, x, y);
    }
    note_launch();
    return cudaGetLastError();
}

}  // namespace rlb
