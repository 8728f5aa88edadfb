// spmv_chunked.cu -- K16: CSR SpMV through column chunks of x staged in
// shared memory (rl_spmv_plan's CUDA-core layout for banded / local matrices).
//
// Why: the CSR kernels (spmv.cu) gather every x value through L1/L2: one
// 32-byte L2 sector per 8-byte gather.  On the BASELINE matrix that is 67 M
// sectors = 2.1 GB of L2 traffic on top of the 0.86 GB streamed from HBM, at
// one distinct-line request per SM per cycle -- the gather roof the CSR
// kernels sit at.  Here each row block's x window is copied
// into shared memory once per block, densely, by cp.async.bulk (no per-value
// requests), and the gathers become shared-memory loads.
//
// Layout (built once on the host by spmv_chunked_build, like DASP's
// conversion or cusparseSpMV_preprocess; bytes <= the CSR's):
//   * rows are cut into blocks of R rows (the block count is a multiple of
//     the SM count, so the persistent grid has no tail); warp w of a block
//     owns rows [w RW, (w+1) RW), RW = R / 16 <= 512;
//   * a block's x window [min col, max col] is cut into chunks of kSpmvChunk
//     columns; chunks with no entry in the block are dropped;
//   * per (chunk, warp): the warp's entries whose column falls in the chunk,
//     ordered so that every aligned group of 32 entries holds 32 DIFFERENT
//     rows (rows' 1st entries, then 2nd entries, ..., with a greedy fix-up and,
//     when a group cannot be completed, padding entries that point at a
//     per-warp dummy row): val2 (f64), meta2 (u32 = row-in-warp << 16 |
//     column-in-chunk), wofs[chunk * 16 + w] = the segment start (segments
//     start 4-entry aligned; the alignment gap is dummy-row entries too).
// Kernel: one persistent CTA of 16 warps per SM; thread 0 streams the x
// chunks of the CTA's blocks through an S-stage ring (mbarrier full/empty,
// one arrive per warp), so the next block's chunks load while the current
// block finishes.  A warp walks its segments in batches of 4 groups (one
// entry per lane per group, coalesced loads), the loads running two batches
// ahead across chunk boundaries; per group each lane does one shared-memory
// x gather and one read-modify-write of its row's y in the warp's private y
// rows -- the 32 rows of a group are distinct, so a group's updates never
// collide and no reduction is needed.  After the block's last chunk the warp
// stores its y rows (coalesced).  Each row's sum follows a fixed entry order:
// deterministic, independent of timing.
#include <algorithm>
#include <thread>
#include <vector>

#include "common.cuh"
#include "kernels.h"
#include "tma.cuh"

namespace rlb {
namespace {

using namespace tmaop;

constexpr int kWarps = kSpmvChunkWarps;

template <int S>
__global__ void __launch_bounds__(32 * kSpmvChunkWarps, 1) spmv_chunked_kernel(
    const SpmvCBlock* __restrict__ blks, int nblk, const SpmvChunk* __restrict__ chunks,
    const unsigned* __restrict__ wofs, const double* __restrict__ val2, const unsigned* __restrict__ meta2,
    const double* __restrict__ x, double* __restrict__ y, int rw_max, int mode) {
    extern __shared__ __align__(128) double smem[];
    const int ystride = rw_max + 1;                  // + the warp's dummy row (padding entries)
    double* xs = smem;                               // S stages of kSpmvChunk doubles
    double* ys = smem + S * kSpmvChunk;              // kWarps x ystride rows
    uint64_t* full = reinterpret_cast<uint64_t*>(ys + kWarps * ystride);
    uint64_t* empty = full + S;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    double* yw = ys + w * ystride;
    const uint64_t pol = policy_evict_first(), polx = policy_evict_last();

    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, kWarps);
        }
        mbar_fence_init();
    }
    for (int i = lane; i < ystride; i += 32) yw[i] = 0.0;
    __syncthreads();

    // producer state (thread 0): next (block, chunk) to load, pk = its ring index
    int pb = blockIdx.x, pc = pb < nblk ? blks[pb].c0 : 0, pk = 0;
    auto produce = [&](int upto) {  // issue ring items pk .. upto-1
        while (pk < upto && pb < nblk) {
            if (pc >= blks[pb].c1) {
                pb += gridDim.x;
                if (pb >= nblk) break;
                pc = blks[pb].c0;
                continue;
            }
            if (pk >= S) mbar_wait(empty + (pk % S), (uint32_t)(((pk / S) - 1) & 1));
            const SpmvChunk ch = chunks[pc];
            uint64_t* bar = full + (pk % S);
            mbar_expect_tx(bar, (uint32_t)ch.ncols * 8u);
            bulk_g2s(xs + (pk % S) * kSpmvChunk, x + ch.col0, (uint32_t)ch.ncols * 8u, bar, polx);
            ++pc;
            ++pk;
        }
    };
    if (tid == 0 && mode != 3) produce(S);

    // A batch = 4 groups of 32 entries (entry j + 32 q + lane).  The loads of a
    // warp's batches run two batches ahead of the one being applied, across
    // chunk boundaries (they do not depend on the x stage).  Segment bounds of
    // 32 chunks at a time sit in the lanes (lane l: chunk g0 + l).
    struct Batch {
        int ci;         // chunk within the group of 32 (gn: no batch)
        unsigned j, e;  // first entry, end of the segment
        double v[4];
        unsigned m[4];
    };
    int k = 0;     // ring index of the chunk being consumed
    int turn = 0;  // which of the four batches is next
    for (int b = blockIdx.x; b < nblk; b += gridDim.x) {
        const SpmvCBlock blk = blks[b];
        for (int g0 = blk.c0; g0 < blk.c1; g0 += 32) {
            const int gn = min(32, blk.c1 - g0);
            const unsigned so = lane < gn ? __ldg(wofs + (size_t)(g0 + lane) * kWarps + w) : 0u;
            const unsigned eo = lane < gn ? __ldg(wofs + (size_t)(g0 + lane) * kWarps + w + 1) : 0u;
            int lc = 0;  // load cursor
            unsigned lj = __shfl_sync(0xffffffffu, so, 0), le = __shfl_sync(0xffffffffu, eo, 0);
            auto next = [&](Batch& bt) {
                while (lc < gn && lj >= le) {
                    ++lc;
                    lj = __shfl_sync(0xffffffffu, so, lc & 31);
                    le = __shfl_sync(0xffffffffu, eo, lc & 31);
                }
                bt.ci = lc;
                bt.j = lj;
                bt.e = le;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const unsigned jj = lj + 32 * q + lane;
                    if (lc < gn && jj < le && mode != 2) {
                        bt.v[q] = ld_stream(val2 + jj, pol);
                        bt.m[q] = (unsigned)ld_stream_i32(reinterpret_cast<const int*>(meta2) + jj, pol);
                    }
                }
                lj += 128;
            };
            // kSpmvChunkBatches (3 or 4) batches in flight per warp, rotated
            // without register copies (a copy of a batch whose loads are still in
            // flight would wait for them): the batch just applied is reloaded in
            // place, NB ahead.
            constexpr int NB = kSpmvChunkBatches;
            Batch A, B, C, D;
            turn = 0;
            next(A);
            next(B);
            next(C);
            if constexpr (NB == 4) next(D);
            auto apply = [&](const Batch& bt, const double* xc) {
                if (mode != 0) {  // diagnostic modes: data movement only
                    if (bt.v[0] == 12345.678) yw[0] += xc[0];
                    return;
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if (bt.j + 32 * q + lane < bt.e) {
                        const unsigned mm = bt.m[q];
                        double* yr = yw + (mm >> 16);
                        *yr = fma(bt.v[q], xc[mm & 0xFFFFu], *yr);
                    }
                }
            };
            for (int ci = 0; ci < gn; ++ci, ++k) {
                if (mode != 3) mbar_wait(full + (k % S), (uint32_t)((k / S) & 1));
                const double* xc = xs + (k % S) * kSpmvChunk;
                for (;;) {
                    bool more;
                    if constexpr (NB == 4)
                        more = turn == 0 ? (A.ci == ci) : turn == 1 ? (B.ci == ci)
                                                              : turn == 2 ? (C.ci == ci)
                                                                          : (D.ci == ci);
                    else
                        more = turn == 0 ? (A.ci == ci) : turn == 1 ? (B.ci == ci)
                                                                          : (C.ci == ci);
                    if (!more) break;
                    if (turn == 0) {
                        apply(A, xc);
                        next(A);
                    } else if (turn == 1) {
                        apply(B, xc);
                        next(B);
                    } else if (NB == 3 || turn == 2) {
                        apply(C, xc);
                        next(C);
                    } else {
                        apply(D, xc);
                        next(D);
                    }
                    turn = turn + 1 == NB ? 0 : turn + 1;
                }
                // release the stage (one arrive per warp); thread 0 refills it
                __syncwarp();
                if (lane == 0) mbar_arrive(empty + (k % S));
                if (tid == 0 && mode != 3) produce(k + 1 + S);
            }
        }
        // the block's y rows: coalesced store, then clear for the next block
        __syncwarp();
        const int rw = min(blk.rw, max(0, (int)blk.rows - w * blk.rw));
        double* yo = y + (uint64_t)blk.row0 + (uint64_t)w * blk.rw;
        for (int i = lane; i < rw; i += 32) yo[i] = yw[i];
        __syncwarp();
        for (int i = lane; i < ystride; i += 32) yw[i] = 0.0;
        __syncwarp();
    }
}

// One entry of the layout under construction.
struct Ent {
    uint32_t row;
    uint32_t col;
    double val;
};

// Order one (chunk, warp) segment so that every aligned group of 32 entries
// has 32 different rows.  `ent` holds (row, col, val) sorted by (row, col).
// Rows' k-th entries come in rounds k = 0, 1, ...; a greedy pass fills each
// group with the earliest pending entries whose rows the group lacks, and a
// group that cannot be completed while entries remain is padded with dummy
// entries (row = dummy, value 0).
void order_segment(const std::vector<Ent>& ent, uint32_t dummy, std::vector<Ent>& out, std::vector<uint32_t>& mark,
                   uint32_t& stamp) {
    out.clear();
    if (ent.empty()) return;
    std::vector<Ent> pending, rest;
    pending.reserve(ent.size());
    std::vector<uint32_t> start;  // index of each row's first entry
    for (size_t i = 0; i < ent.size(); ++i)
        if (i == 0 || ent[i].row != ent[i - 1].row) start.push_back((uint32_t)i);
    start.push_back((uint32_t)ent.size());
    for (size_t kk = 0;; ++kk) {
        bool any = false;
        for (size_t r = 0; r + 1 < start.size(); ++r)
            if (start[r] + kk < start[r + 1]) {
                pending.push_back(ent[start[r] + kk]);
                any = true;
            }
        if (!any) break;
    }
    while (!pending.empty()) {
        ++stamp;
        size_t taken = 0;
        rest.clear();
        for (const Ent& e : pending) {
            if (taken < 32 && mark[e.row] != stamp) {
                mark[e.row] = stamp;
                out.push_back(e);
                ++taken;
            } else {
                rest.push_back(e);
            }
        }
        if (taken < 32 && !rest.empty())
            for (; taken < 32; ++taken) out.push_back(Ent{dummy, 0u, 0.0});
        pending.swap(rest);
    }
}

}  // namespace

bool spmv_chunked_build(uint64_t m, uint64_t n, const int32_t* rp, const int32_t* col, const double* val,
                        SpmvChunkedLayout& L) {
    if (m == 0 || n == 0 || (n & 1) || n >= (1ull << 31)) return false;
    // blocks: a multiple of the SM count, R <= 8192 rows, R % kWarps == 0
    const uint64_t waves = (m + (uint64_t)kNumSMs * 8192 - 1) / ((uint64_t)kNumSMs * 8192);
    uint64_t nblk = (uint64_t)kNumSMs * waves;
    uint64_t R = (m + nblk - 1) / nblk;
    R = (R + kWarps - 1) / kWarps * kWarps;
    if (R < (uint64_t)kWarps) R = kWarps;
    nblk = (m + R - 1) / R;
    const int rw = (int)(R / kWarps);
    L.rw = rw;
    L.blocks.assign(nblk, SpmvCBlock{});
    std::vector<std::vector<SpmvChunk>> bchunks(nblk);
    std::vector<std::vector<std::vector<Ent>>> bseg(nblk);  // per block: per (chunk, warp) ordered entries
    const unsigned hw = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
    std::vector<char> bad(hw, 0);
    auto build_block = [&](unsigned tix) {
        std::vector<uint32_t> mark(rw + 1, 0);
        uint32_t stamp = 0;
        std::vector<Ent> ordered;
        std::vector<std::pair<int32_t, double>> rowbuf;
        for (uint64_t b = tix; b < nblk; b += hw) {
            const uint64_t r0 = b * R, r1 = std::min(m, r0 + R);
            SpmvCBlock& B = L.blocks[b];
            B.row0 = (uint32_t)r0;
            B.rows = (uint32_t)(r1 - r0);
            B.rw = rw;
            int64_t cmin = INT64_MAX, cmax = -1;
            for (uint64_t i = r0; i < r1; ++i)
                for (int64_t e = rp[i]; e < rp[i + 1]; ++e) {
                    const int64_t c = col[e];
                    if (c < 0 || (uint64_t)c >= n) {
                        bad[tix] = 1;
                        return;
                    }
                    cmin = std::min(cmin, c);
                    cmax = std::max(cmax, c);
                }
            if (cmax < 0) continue;  // no entries: the kernel writes zero rows
            const int64_t base = cmin & ~int64_t(1);
            const int64_t nch = (cmax - base) / kSpmvChunk + 1;
            // bucket the block's entries by (chunk, warp): rows ascending, columns sorted
            std::vector<std::vector<Ent>> bucket((size_t)nch * kWarps);
            for (uint64_t i = r0; i < r1; ++i) {
                const int wi = (int)((i - r0) / rw);
                const uint32_t rr = (uint32_t)((i - r0) % rw);
                rowbuf.clear();
                for (int64_t e = rp[i]; e < rp[i + 1]; ++e) rowbuf.emplace_back(col[e], val[e]);
                std::stable_sort(rowbuf.begin(), rowbuf.end(),
                                 [](const auto& a, const auto& b2) { return a.first < b2.first; });
                for (const auto& [c, v] : rowbuf) {
                    const int64_t ch = (c - base) / kSpmvChunk;
                    bucket[(size_t)ch * kWarps + wi].push_back(Ent{rr, (uint32_t)(c - (base + ch * kSpmvChunk)), v});
                }
            }
            for (int64_t ch = 0; ch < nch; ++ch) {
                size_t tot = 0;
                for (int wi = 0; wi < kWarps; ++wi) tot += bucket[(size_t)ch * kWarps + wi].size();
                if (!tot) continue;
                SpmvChunk C;
                C.col0 = (int32_t)(base + ch * kSpmvChunk);
                // only the columns the block reads (its window ends at cmax)
                C.ncols = (int32_t)std::min<int64_t>(kSpmvChunk, cmax + 1 - C.col0);
                C.ncols = (C.ncols + 1) & ~1;  // n is even: stays inside x
                bchunks[b].push_back(C);
                for (int wi = 0; wi < kWarps; ++wi) {
                    order_segment(bucket[(size_t)ch * kWarps + wi], (uint32_t)rw, ordered, mark, stamp);
                    bseg[b].push_back(ordered);
                }
            }
        }
    };
    {
        std::vector<std::thread> th;
        for (unsigned t = 0; t < hw; ++t) th.emplace_back(build_block, t);
        for (auto& t : th) t.join();
    }
    if (std::any_of(bad.begin(), bad.end(), [](char c) { return c != 0; })) return false;
    uint64_t nchunks = 0, E = 0;
    std::vector<uint64_t> bofs(nblk + 1, 0);
    for (uint64_t b = 0; b < nblk; ++b) {
        L.blocks[b].c0 = (int)nchunks;
        nchunks += bchunks[b].size();
        L.blocks[b].c1 = (int)nchunks;
        bofs[b] = E;
        for (const auto& sg : bseg[b]) E += (sg.size() + 3) & ~size_t(3);  // segments start 32-byte aligned
    }
    if (E >= (1ull << 32) || nchunks >= (1ull << 31)) return false;
    L.chunks.resize(nchunks);
    L.wofs.assign(nchunks * kWarps + 1, 0);
    L.val.assign(E, 0.0);
    L.meta.assign(E, (uint32_t)rw << 16);  // alignment gaps: dummy-row entries, value 0
    auto place = [&](unsigned tix) {
        for (uint64_t b = tix; b < nblk; b += hw) {
            std::copy(bchunks[b].begin(), bchunks[b].end(), L.chunks.begin() + L.blocks[b].c0);
            uint64_t o = bofs[b];
            for (size_t q = 0; q < bseg[b].size(); ++q) {
                const auto& sg = bseg[b][q];
                L.wofs[(size_t)L.blocks[b].c0 * kWarps + q] = (unsigned)o;
                for (size_t i = 0; i < sg.size(); ++i) {
                    L.val[o + i] = sg[i].val;
                    L.meta[o + i] = (sg[i].row << 16) | sg[i].col;
                }
                o += (sg.size() + 3) & ~size_t(3);
            }
            bseg[b].clear();
            bseg[b].shrink_to_fit();
        }
    };
    {
        std::vector<std::thread> th;
        for (unsigned t = 0; t < hw; ++t) th.emplace_back(place, t);
        for (auto& t : th) t.join();
    }
    L.wofs[nchunks * kWarps] = (unsigned)E;
    L.x_bytes = 0;
    for (const auto& c : L.chunks) L.x_bytes += (uint64_t)c.ncols * 8;
    return true;
}

size_t spmv_chunked_smem(int rw) {
    return (size_t)kSpmvChunkStages * kSpmvChunk * 8 + (size_t)kWarps * (rw + 1) * 8 + 2 * kSpmvChunkStages * 8;
}

cudaError_t launch_spmv_chunked(const SpmvCBlock* blks, int nblk, const SpmvChunk* chunks, const unsigned* wofs,
                                const double* val2, const unsigned* meta2, const double* x, double* y, int rw,
                                cudaStream_t s) {
    if (nblk <= 0) return cudaSuccess;
    const size_t smem = spmv_chunked_smem(rw);
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(spmv_chunked_kernel<kSpmvChunkStages>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(227 * 1024));
        if (e != cudaSuccess) return e;
        attr = true;
    }
    const int grid = std::min(nblk, kNumSMs);
    spmv_chunked_kernel<kSpmvChunkStages><<<grid, 32 * kWarps, smem, s>>>(blks, nblk, chunks, wofs, val2, meta2, x, y,
                                                                        rw, tuning().spmv_chunked_mode);
    note_launch();
    return cudaGetLastError();
}

}  // namespace rlb
