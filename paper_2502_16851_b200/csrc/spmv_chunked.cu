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
//   * rows are cut into blocks of R rows (a multiple of 32; the block count
//     is a multiple of the SM count so the persistent grid has no tail);
//     warp w of a block owns rows [w RW, (w+1) RW), RW = R / 32 <= 256;
//   * a block's x window [min col, max col] is cut into chunks of kChunk
//     columns; chunks with no entry in the block are dropped;
//   * per (chunk, warp), the warp's entries whose column falls in the chunk,
//     row-major (row, then column), padded to a multiple of 4:
//     val2 (f64) and meta2 (u32 = row-in-warp << 16 | column-in-chunk;
//     column 0xFFFF marks padding), and wofs[(chunk) * 32 + w] the start of
//     that segment (monotone, u32).
// Kernel: one persistent CTA of 32 warps per SM; thread 0 streams the x
// chunks of the CTA's blocks through an S-stage ring (mbarrier full/empty,
// one arrive per warp), so the next block's chunks load while the current
// block finishes.  A warp walks its segment 128 entries per step: one 256-bit
// val and one 128-bit meta load per lane (HBM, evict_first), 4 shared-memory
// x gathers, then a row-run reduction -- runs inside the lane, a segmented
// shuffle scan across lanes for runs that span lanes -- and one
// read-modify-write of the warp's private y rows in shared memory per run.
// After the block's last chunk the warp stores its y rows (coalesced).
// The sums per row follow the entries' column order within each chunk and
// chunk order across chunks: deterministic, independent of timing.
#include <algorithm>
#include <thread>
#include <vector>

#include "common.cuh"
#include "kernels.h"
#include "tma.cuh"

namespace rlb {
namespace {

using namespace tmaop;

constexpr int kWarps = 32;
constexpr unsigned kPadCol = 0xFFFFu;

__device__ __forceinline__ int4 ld4_i32_stream(const unsigned* p, uint64_t pol) {
    int4 v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
        : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
        : "l"(p), "l"(pol));
    return v;
}

template <int S>
__global__ void __launch_bounds__(1024, 1) spmv_chunked_kernel(const SpmvCBlock* __restrict__ blks, int nblk,
                                                               const SpmvChunk* __restrict__ chunks,
                                                               const unsigned* __restrict__ wofs,
                                                               const double* __restrict__ val2,
                                                               const unsigned* __restrict__ meta2,
                                                               const double* __restrict__ x, double* __restrict__ y,
                                                               int rw_max) {
    extern __shared__ __align__(128) double smem[];
    double* xs = smem;                               // S stages of kChunk doubles
    double* ys = smem + S * kSpmvChunk;              // 32 warps x rw_max rows
    uint64_t* full = reinterpret_cast<uint64_t*>(ys + kWarps * rw_max);
    uint64_t* empty = full + S;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    double* yw = ys + w * rw_max;
    const uint64_t pol = policy_evict_first(), polx = policy_evict_last();

    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, kWarps);
        }
        mbar_fence_init();
    }
    for (int i = lane; i < rw_max; i += 32) yw[i] = 0.0;
    __syncthreads();

    // producer state (thread 0): next (block, chunk) to load, k = its ring index
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
    if (tid == 0) produce(S);

    int k = 0;  // ring index of the chunk being consumed
    for (int b = blockIdx.x; b < nblk; b += gridDim.x) {
        const SpmvCBlock blk = blks[b];
        for (int c = blk.c0; c < blk.c1; ++c, ++k) {
            mbar_wait(full + (k % S), (uint32_t)((k / S) & 1));
            const double* xc = xs + (k % S) * kSpmvChunk;
            const unsigned s0 = __ldg(wofs + (size_t)c * kWarps + w), s1 = __ldg(wofs + (size_t)c * kWarps + w + 1);
            for (unsigned j0 = s0; j0 < s1; j0 += 128) {
                const unsigned j = j0 + 4 * lane;
                const bool act = j < s1;
                double p[4];
                int r[4];
                if (act) {
                    const d4 v = ld4_stream(val2 + j, pol);
                    const int4 m = ld4_i32_stream(meta2 + j, pol);
                    const unsigned mm[4] = {(unsigned)m.x, (unsigned)m.y, (unsigned)m.z, (unsigned)m.w};
                    const double vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        r[q] = (int)(mm[q] >> 16);
                        const unsigned cc = mm[q] & 0xFFFFu;
                        p[q] = cc == kPadCol ? 0.0 : vv[q] * xc[cc];
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        r[q] = -1 - lane;  // distinct from every real row and from each other lane
                        p[q] = 0.0;
                    }
                }
                // runs inside the lane: s[q] = sum of the run up to entry q
                double s[4];
                s[0] = p[0];
#pragma unroll
                for (int q = 1; q < 4; ++q) s[q] = r[q] == r[q - 1] ? s[q - 1] + p[q] : p[q];
                const int h = r[0], t = r[3];
                // segmented inclusive scan of the tail runs across lanes: lane l's
                // tail chain continues lane l-1's when the whole lane is one row
                // equal to lane l-1's tail row
                const int t_prev = __shfl_up_sync(0xffffffffu, t, 1);
                double T = s[3];
                int F = (lane == 0 || h != t || h != t_prev) ? 1 : 0;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const double Tu = __shfl_up_sync(0xffffffffu, T, d);
                    const int Fu = __shfl_up_sync(0xffffffffu, F, d);
                    if (lane >= d && !F) {
                        T += Tu;
                        F |= Fu;
                    }
                }
                const double T_prev = __shfl_up_sync(0xffffffffu, T, 1);
                const int h_next = __shfl_down_sync(0xffffffffu, h, 1);
                const double cin = (lane > 0 && h == t_prev) ? T_prev : 0.0;
                if (act) {
                    // runs that end inside the lane (entries 0..2)
#pragma unroll
                    for (int q = 0; q < 3; ++q) {
                        if (r[q] != r[q + 1]) {
                            const double add = s[q] + (r[q] == h ? cin : 0.0);
                            yw[r[q]] += add;
                        }
                    }
                    // the tail run, written by the last lane of its chain
                    if (lane == 31 || h_next != t) yw[t] += T;
                }
                __syncwarp();  // the next step's lanes read what this step's lanes wrote
            }
            // release the stage (one arrive per warp); thread 0 refills it
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + (k % S));
            if (tid == 0) produce(k + 1 + S);
        }
        // the block's y rows: coalesced store, then clear for the next block
        __syncwarp();
        const int rw = min(blk.rw, max(0, (int)blk.rows - w * blk.rw));
        double* yo = y + (uint64_t)blk.row0 + (uint64_t)w * blk.rw;
        for (int i = lane; i < rw; i += 32) {
            yo[i] = yw[i];
            yw[i] = 0.0;
        }
        for (int i = rw + lane; i < blk.rw; i += 32) yw[i] = 0.0;
        __syncwarp();
    }
}

}  // namespace

bool spmv_chunked_build(uint64_t m, uint64_t n, const int32_t* rp, const int32_t* col, const double* val,
                        SpmvChunkedLayout& L) {
    if (m == 0 || n == 0 || (n & 1) || n >= (1ull << 31)) return false;
    const uint64_t nnz = (uint64_t)rp[m];
    // blocks: a multiple of the SM count, R <= 8192 rows, R % 32 == 0
    uint64_t waves = (m + (uint64_t)kNumSMs * 8192 - 1) / ((uint64_t)kNumSMs * 8192);
    uint64_t nblk = (uint64_t)kNumSMs * waves;
    uint64_t R = (m + nblk - 1) / nblk;
    R = (R + 31) / 32 * 32;
    if (R < 32) R = 32;
    nblk = (m + R - 1) / R;
    const int rw = (int)(R / 32);
    L.rw = rw;
    L.blocks.assign(nblk, SpmvCBlock{});
    std::vector<std::vector<SpmvChunk>> bchunks(nblk);
    std::vector<std::vector<unsigned>> bcount(nblk);  // per block: per (chunk, warp) padded counts
    const unsigned hw = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
    std::vector<char> bad(hw, 0);
    auto pass1 = [&](unsigned tix) {
        for (uint64_t b = tix; b < nblk; b += hw) {
            const uint64_t r0 = b * R, r1 = std::min(m, r0 + R);
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
            SpmvCBlock& B = L.blocks[b];
            B.row0 = (uint32_t)r0;
            B.rows = (uint32_t)(r1 - r0);
            B.rw = rw;
            if (cmax < 0) continue;  // no entries: y rows are zero (written by the kernel)
            const int64_t base = cmin & ~int64_t(1);
            const int64_t nch = (cmax - base) / kSpmvChunk + 1;
            std::vector<unsigned> cnt((size_t)nch * kWarps, 0);
            for (uint64_t i = r0; i < r1; ++i) {
                const int wi = (int)((i - r0) / rw);
                for (int64_t e = rp[i]; e < rp[i + 1]; ++e) ++cnt[(size_t)((col[e] - base) / kSpmvChunk) * kWarps + wi];
            }
            for (int64_t ch = 0; ch < nch; ++ch) {
                unsigned tot = 0;
                for (int wi = 0; wi < kWarps; ++wi) tot += cnt[(size_t)ch * kWarps + wi];
                if (!tot) continue;
                SpmvChunk C;
                C.col0 = (int32_t)(base + ch * kSpmvChunk);
                C.ncols = (int32_t)std::min<int64_t>(kSpmvChunk, (int64_t)n - C.col0);
                C.ncols = (C.ncols + 1) & ~1;  // n is even: stays inside x
                bchunks[b].push_back(C);
                for (int wi = 0; wi < kWarps; ++wi) bcount[b].push_back((cnt[(size_t)ch * kWarps + wi] + 3u) & ~3u);
            }
        }
    };
    {
        std::vector<std::thread> th;
        for (unsigned t = 0; t < hw; ++t) th.emplace_back(pass1, t);
        for (auto& t : th) t.join();
    }
    if (std::any_of(bad.begin(), bad.end(), [](char c) { return c != 0; })) return false;
    // global chunk table and segment offsets
    uint64_t nchunks = 0, E = 0;
    std::vector<uint64_t> bofs(nblk + 1, 0);  // first entry of each block
    for (uint64_t b = 0; b < nblk; ++b) {
        L.blocks[b].c0 = (int)nchunks;
        nchunks += bchunks[b].size();
        L.blocks[b].c1 = (int)nchunks;
        bofs[b] = E;
        for (unsigned c : bcount[b]) E += c;
    }
    bofs[nblk] = E;
    if (E >= (1ull << 32) || nchunks >= (1ull << 31)) return false;
    L.chunks.resize(nchunks);
    L.wofs.assign(nchunks * kWarps + 1, 0);
    L.val.assign(E, 0.0);
    L.meta.assign(E, 0u);
    for (uint64_t b = 0; b < nblk; ++b) {
        std::copy(bchunks[b].begin(), bchunks[b].end(), L.chunks.begin() + L.blocks[b].c0);
        uint64_t o = bofs[b];
        for (size_t q = 0; q < bcount[b].size(); ++q) {
            L.wofs[(size_t)L.blocks[b].c0 * kWarps + q] = (unsigned)o;
            o += bcount[b][q];
        }
    }
    L.wofs[nchunks * kWarps] = (unsigned)E;
    auto pass2 = [&](unsigned tix) {
        std::vector<unsigned> fill;
        for (uint64_t b = tix; b < nblk; b += hw) {
            const SpmvCBlock& B = L.blocks[b];
            const int nc = B.c1 - B.c0;
            if (!nc) continue;
            const uint64_t r0 = B.row0, r1 = r0 + B.rows;
            fill.assign((size_t)nc * kWarps, 0);
            // rows in order, and each row's entries in column order (sorted
            // here if the CSR row is not), keep every segment row-major
            std::vector<std::pair<int32_t, double>> rowbuf;
            for (uint64_t i = r0; i < r1; ++i) {
                const int wi = (int)((i - r0) / B.rw);
                const unsigned rr = (unsigned)((i - r0) % B.rw);
                rowbuf.clear();
                for (int64_t e = rp[i]; e < rp[i + 1]; ++e) rowbuf.emplace_back(col[e], val[e]);
                std::stable_sort(rowbuf.begin(), rowbuf.end(),
                                 [](const auto& a, const auto& b2) { return a.first < b2.first; });
                int ci = 0;
                for (const auto& [c, v] : rowbuf) {
                    while (L.chunks[B.c0 + ci].col0 + kSpmvChunk <= c) ++ci;
                    const size_t seg = (size_t)ci * kWarps + wi;
                    const uint64_t pos = L.wofs[(size_t)B.c0 * kWarps + seg] + fill[seg]++;
                    L.val[pos] = v;
                    L.meta[pos] = (rr << 16) | (unsigned)(c - L.chunks[B.c0 + ci].col0);
                }
            }
            // padding: repeat the segment's last row, column marked as padding
            for (size_t seg = 0; seg < fill.size(); ++seg) {
                const uint64_t s0 = L.wofs[(size_t)B.c0 * kWarps + seg], s1 = L.wofs[(size_t)B.c0 * kWarps + seg + 1];
                for (uint64_t pos = s0 + fill[seg]; pos < s1; ++pos) {
                    L.val[pos] = 0.0;
                    L.meta[pos] = (L.meta[pos - 1] & 0xFFFF0000u) | kPadCol;
                }
            }
        }
    };
    {
        std::vector<std::thread> th;
        for (unsigned t = 0; t < hw; ++t) th.emplace_back(pass2, t);
        for (auto& t : th) t.join();
    }
    L.x_bytes = 0;
    for (const auto& c : L.chunks) L.x_bytes += (uint64_t)c.ncols * 8;
    (void)nnz;
    return true;
}

size_t spmv_chunked_smem(int rw) { return (size_t)kSpmvChunkStages * kSpmvChunk * 8 + (size_t)kWarps * rw * 8 + 2 * kSpmvChunkStages * 8; }

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
    spmv_chunked_kernel<kSpmvChunkStages><<<grid, 1024, smem, s>>>(blks, nblk, chunks, wofs, val2, meta2, x, y, rw);
    note_launch();
    return cudaGetLastError();
}

}  // namespace rlb
