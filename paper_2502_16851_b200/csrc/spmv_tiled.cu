// spmv_tiled.cu -- column-tiled SpMV behind rl_spmv_plan (CUDA core).
//
// Why: a CSR row of the BASELINE matrix gathers 16 random x values from a
// +-65,536-column band.  Measured on this B200, random 8-byte gathers from
// L2 sustain ~1 per SM per cycle, so the plain CSR kernel is capped near
// 3.3 TB/s whatever its schedule (profiles/README.md).  A plan can pay a
// one-time layout change (the role of cusparseSpMV_preprocess, or DASP's
// format conversion in the paper) so that every x value a
// row needs comes from shared memory:
//
//   * rows are cut into blocks of RB = 8192 (one CTA of 32 warps; warp w owns
//     rows 256w .. 256w+255 of the block and their sums in shared memory);
//   * a block's nonzeros, in column order, are cut into tiles of at most
//     kEMax entries spanning at most kT = 2048 columns;
//   * a tile is one contiguous segment in HBM: 33 per-warp entry offsets,
//     the values (f64) and one u32 of metadata per entry (column in tile |
//     row in warp | segment depth | segment end), entries sorted by row;
//   * one pipeline thread bulk-copies (cp.async.bulk + mbarrier transaction
//     count) the x slice and the segment into a 4-stage shared-memory ring;
//     the last warp to release a stage refills it, so no warp waits on
//     another except through the data itself;
//   * each warp walks its entries 32 at a time: lane product val*x (x from
//     shared memory), a segmented inclusive scan over the lanes (depth from
//     the metadata, shuffles only as deep as the warp's longest run), and the
//     run's last lane adds the row's partial sum to shared y.  Rows never
//     span warps and runs of a row are added in a fixed order, so the result
//     is deterministic.
//
// Traffic per call is the segments (12 B per nonzero + 80 B per tile) plus
// y; x slices are served from L2.  The algorithmic accounting stays the CSR
// model's (kernels.cpp:125-136 of the reference).
#include <algorithm>
#include <atomic>
#include <cstring>
#include <thread>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace rlb {

namespace {
constexpr int kRB = kSpmvTiledRows;  // rows per block
constexpr int kWarps = 32;
constexpr int kThreads = kWarps * 32;
constexpr int kRowsPerWarp = kRB / kWarps;  // 256 -> 8-bit row field
constexpr int kT = 2048;                    // max tile width (columns) -> 11-bit column field
constexpr int kEMax = 2048;                 // max entries per tile
constexpr int kStages = 4;

__host__ __device__ constexpr size_t pad16(size_t b) { return (b + 15) & ~size_t(15); }
constexpr size_t kOffBytes = pad16((kWarps + 1) * 2);  // 80
constexpr size_t kSegMax = kOffBytes + pad16((size_t)kEMax * 12);
constexpr size_t kXBytes = (size_t)kT * 8;
constexpr size_t kStageBytes = kXBytes + kSegMax;
constexpr size_t kYBytes = (size_t)kRB * 8;
constexpr size_t kSmem = kStages * kStageBytes + kYBytes + kStages * 8 + kStages * 4;
static_assert(kSmem <= 227 * 1024, "tiled SpMV shared memory");

// metadata word
constexpr int kColBits = 11, kRowShift = 11, kDepthShift = 19, kEndShift = 24;

__device__ __forceinline__ uint32_t sptr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
            "r"(sptr(dst)),
        "l"(src), "r"(bytes), "r"(sptr(bar)), "l"(pol)
        : "memory");
}

__global__ void __launch_bounds__(kThreads, 1) spmv_tiled_kernel(uint64_t m, uint64_t b_first,
                                                                 const uint8_t* __restrict__ segs,
                                                                 const SpmvTile* __restrict__ tiles,
                                                                 const int* __restrict__ blk_tiles,
                                                                 const double* __restrict__ x,
                                                                 double* __restrict__ y) {
    extern __shared__ __align__(128) uint8_t smem[];
    double* ysm = reinterpret_cast<double*>(smem + kStages * kStageBytes);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes + kYBytes);
    uint32_t* cnt = reinterpret_cast<uint32_t*>(full + kStages);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t b = b_first + blockIdx.x;
    const int t0 = blk_tiles[b], t1 = blk_tiles[b + 1];
    const int nt = t1 - t0;
    double* yw = ysm + warp * kRowsPerWarp;
#pragma unroll
    for (int i = 0; i < kRowsPerWarp / 32; ++i) yw[lane + 32 * i] = 0.0;
    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sptr(full + s)) : "memory");
            cnt[s] = 0;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int k) {
        const SpmvTile t = tiles[t0 + k];
        uint8_t* st = smem + (k % kStages) * kStageBytes;
        const uint32_t xb = (uint32_t)(t.width * 8);
        const uint32_t sb = (uint32_t)t.seg_bytes;
        uint64_t* bar = full + (k % kStages);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sptr(bar)), "r"(xb + sb)
                     : "memory");
        bulk_g2s(st, x + t.col_base, xb, bar, policy_evict_last());
        bulk_g2s(st + kXBytes, segs + t.seg_offset, sb, bar, policy_evict_first());
    };
    if (tid == 0)
        for (int k = 0; k < kStages && k < nt; ++k) issue(k);
    for (int k = 0; k < nt; ++k) {
        const int s = k % kStages;
        const uint32_t parity = (uint32_t)((k / kStages) & 1);
        asm volatile(
            "{\n .reg .pred P;\nRLB_TW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1, %2;\n"
            " @!P bra RLB_TW_%=;\n}" ::"r"(sptr(full + s)),
            "r"(parity), "r"(1000000u)
            : "memory");
        const uint8_t* st = smem + s * kStageBytes;
        const double* xs = reinterpret_cast<const double*>(st);
        const uint8_t* seg = st + kXBytes;
        const uint16_t* offs = reinterpret_cast<const uint16_t*>(seg);
        const int E = offs[kWarps], e0 = offs[warp], e1 = offs[warp + 1];
        const double* vals = reinterpret_cast<const double*>(seg + kOffBytes);
        const uint32_t* meta = reinterpret_cast<const uint32_t*>(seg + kOffBytes + (size_t)E * 8);
        // two 32-entry rounds per pass: both rounds' loads in flight together
        for (int base = e0; base < e1; base += 64) {
            const int ea = base + lane, eb = ea + 32;
            double pa = 0.0, pb = 0.0;
            uint32_t ma = 0, mb = 0;
            if (ea < e1) ma = meta[ea];
            if (eb < e1) mb = meta[eb];
            if (ea < e1) pa = vals[ea] * xs[ma & ((1u << kColBits) - 1)];
            if (eb < e1) pb = vals[eb] * xs[mb & ((1u << kColBits) - 1)];
            const int da = (int)((ma >> kDepthShift) & 31), db = (int)((mb >> kDepthShift) & 31);
            const int maxd = (int)__reduce_max_sync(0xffffffffu, (unsigned)max(da, db));
            for (int o = 1; o <= maxd; o <<= 1) {
                const double qa = __shfl_up_sync(0xffffffffu, pa, o);
                const double qb = __shfl_up_sync(0xffffffffu, pb, o);
                if (o <= da) pa += qa;
                if (o <= db) pb += qb;
            }
            if ((ma >> kEndShift) & 1) yw[(ma >> kRowShift) & (kRowsPerWarp - 1)] += pa;
            __syncwarp();
            if ((mb >> kEndShift) & 1) yw[(mb >> kRowShift) & (kRowsPerWarp - 1)] += pb;
            __syncwarp();
        }
        // release the stage; the last warp out refills it
        if (lane == 0) {
            __threadfence_block();
            if (atomicAdd(&cnt[s], 1u) == kWarps - 1) {
                __threadfence_block();
                cnt[s] = 0;
                if (k + kStages < nt) issue(k + kStages);
            }
        }
    }
    __syncwarp();
    const uint64_t r0 = b * kRB + (uint64_t)warp * kRowsPerWarp;
    if (r0 + kRowsPerWarp <= m && ((reinterpret_cast<uintptr_t>(y + r0) & 31) == 0)) {
#pragma unroll
        for (int i = 0; i < kRowsPerWarp / 128; ++i) {
            const int r = 4 * lane + 128 * i;
            st4(y + r0 + r, d4{yw[r], yw[r + 1], yw[r + 2], yw[r + 3]});
        }
    } else {
        for (int r = lane; r < kRowsPerWarp; r += 32)
            if (r0 + r < m) y[r0 + r] = yw[r];
    }
}

struct HostEntry {
    int32_t col;
    int32_t row;  // row within the block
    double val;
};

// Tiles of one row block, appended to (segs, tiles) with segment offsets
// relative to the block's first byte.
void build_block(uint64_t r0, uint64_t r1, uint64_t n, const int32_t* rp, const int32_t* col, const double* val,
                 std::vector<uint8_t>& segs, std::vector<SpmvTile>& tiles) {
    std::vector<HostEntry> es;
    es.reserve((size_t)(rp[r1] - rp[r0]));
    for (uint64_t i = r0; i < r1; ++i)
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) es.push_back({col[k], (int32_t)(i - r0), val[k]});
    if (es.empty()) return;
    std::stable_sort(es.begin(), es.end(), [](const HostEntry& a, const HostEntry& c) { return a.col < c.col; });
    size_t p = 0;
    while (p < es.size()) {
        const int32_t c0 = es[p].col & ~1;
        const int64_t lim = std::min<int64_t>((int64_t)c0 + kT, (int64_t)n);
        size_t q = p;
        while (q < es.size() && es[q].col < lim && q - p < (size_t)kEMax) ++q;
        int32_t width = ((es[q - 1].col - c0) + 2) & ~1;
        if ((uint64_t)c0 + width > n) width = (int32_t)(n - c0);
        // entries by (row, column): warps' runs are contiguous, rows sorted
        std::stable_sort(es.begin() + p, es.begin() + q,
                         [](const HostEntry& a, const HostEntry& c) { return a.row < c.row; });
        const int E = (int)(q - p);
        SpmvTile t{};
        t.seg_offset = segs.size();
        t.col_base = c0;
        t.width = width;
        t.entries = E;
        t.seg_bytes = (int)(kOffBytes + pad16((size_t)E * 12));
        segs.resize(segs.size() + t.seg_bytes, 0);
        uint8_t* sb = segs.data() + t.seg_offset;
        uint16_t* off = reinterpret_cast<uint16_t*>(sb);
        double* v = reinterpret_cast<double*>(sb + kOffBytes);
        uint32_t* mt = reinterpret_cast<uint32_t*>(sb + kOffBytes + (size_t)E * 8);
        const HostEntry* te = es.data() + p;
        int cur = 0;
        for (int w = 0; w <= kWarps; ++w) {
            while (cur < E && te[cur].row / kRowsPerWarp < w) ++cur;
            off[w] = (uint16_t)cur;
        }
        int seg_start = 0;
        for (int i = 0; i < E; ++i) {
            const int w = te[i].row / kRowsPerWarp;
            if (i == 0 || te[i].row != te[i - 1].row) seg_start = i;
            const int round_start = off[w] + ((i - off[w]) / 32) * 32;
            const int depth = i - std::max(seg_start, round_start);
            const bool end = i + 1 == E || te[i + 1].row != te[i].row || (i + 1 - off[w]) % 32 == 0;
            v[i] = te[i].val;
            mt[i] = (uint32_t)(te[i].col - c0) | ((uint32_t)(te[i].row % kRowsPerWarp) << kRowShift) |
                    ((uint32_t)depth << kDepthShift) | ((end ? 1u : 0u) << kEndShift);
        }
        tiles.push_back(t);
        p = q;
    }
}

}  // namespace

// Host-side layout build from a host CSR (called once by rl_spmv_plan_create).
// Row blocks are built in parallel on the host's cores, then concatenated.
void spmv_tiled_build(uint64_t m, uint64_t n, const int32_t* rp, const int32_t* col, const double* val,
                      std::vector<uint8_t>& segs, std::vector<SpmvTile>& tiles, std::vector<int>& blk_tiles) {
    segs.clear();
    tiles.clear();
    blk_tiles.clear();
    const uint64_t nblocks = (m + kRB - 1) / kRB;
    std::vector<std::vector<uint8_t>> bsegs(nblocks);
    std::vector<std::vector<SpmvTile>> btiles(nblocks);
    std::atomic<uint64_t> next{0};
    auto work = [&]() {
        for (uint64_t b; (b = next.fetch_add(1)) < nblocks;)
            build_block(b * kRB, std::min<uint64_t>(m, (b + 1) * kRB), n, rp, col, val, bsegs[b], btiles[b]);
    };
    const unsigned nth = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(), 64));
    std::vector<std::thread> pool;
    for (unsigned i = 1; i < nth && i < nblocks; ++i) pool.emplace_back(work);
    work();
    for (auto& t : pool) t.join();
    size_t total = 0, ntiles = 0;
    for (uint64_t b = 0; b < nblocks; ++b) {
        total += bsegs[b].size();
        ntiles += btiles[b].size();
    }
    segs.resize(total);
    tiles.reserve(ntiles);
    size_t off = 0;
    for (uint64_t b = 0; b < nblocks; ++b) {
        blk_tiles.push_back((int)tiles.size());
        if (!bsegs[b].empty()) std::memcpy(segs.data() + off, bsegs[b].data(), bsegs[b].size());
        for (SpmvTile t : btiles[b]) {
            t.seg_offset += off;
            tiles.push_back(t);
        }
        off += bsegs[b].size();
        std::vector<uint8_t>().swap(bsegs[b]);
    }
    blk_tiles.push_back((int)tiles.size());
}

size_t spmv_tiled_smem() { return kSmem; }

cudaError_t launch_spmv_tiled(uint64_t m, const uint8_t* segs, const SpmvTile* tiles, const int* blk_tiles,
                              uint64_t b0, uint64_t b1, const double* x, double* y, cudaStream_t s) {
    if (b1 <= b0) return cudaSuccess;
    static bool attr = false;
    if (!attr) {
        cudaError_t e =
            cudaFuncSetAttribute(spmv_tiled_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    spmv_tiled_kernel<<<(unsigned)(b1 - b0), kThreads, kSmem, s>>>(m, b0, segs, tiles, blk_tiles, x, y);
    note_launch();
    return cudaGetLastError();
}

}  // namespace rlb
