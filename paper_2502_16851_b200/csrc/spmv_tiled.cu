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
//   * rows are cut into blocks of RB = 8192 (one CTA of 16 warps; warp w owns
//     rows 512w .. 512w+511 of the block and their sums in shared memory);
//   * a block's nonzeros, in column order, are cut into tiles of at most
//     kEMax entries spanning at most kT = 2048 columns;
//   * a tile is one contiguous segment in HBM: 17 per-warp chunk offsets,
//     the values (f64) and one u32 of metadata per entry (column in tile |
//     row in warp | run start / end | lane carry depth), entries sorted by
//     row, each warp's chunk padded to a multiple of 4;
//   * one pipeline thread bulk-copies (cp.async.bulk + mbarrier transaction
//     count) the x slice and the segment into a 4-stage shared-memory ring;
//     the last warp to release a stage refills it, so no warp waits on
//     another except through the data itself;
//   * each warp walks its chunk 128 entries at a time, 4 consecutive entries
//     per lane (128-bit shared loads of values and metadata, x gathered from
//     the shared slice); runs of a row are summed inside the lane, a run that
//     crosses lanes takes its carry from one shuffle (a segmented scan only
//     when a run spans more than two lanes), and the entry that ends a run
//     adds it to shared y.  Rows never span warps and runs are added in a
//     fixed order, so the result is deterministic.
//
// Traffic per call is the segments (12 B per nonzero + 64 B per tile) plus
// y; x slices are served from L2.  The algorithmic accounting stays the CSR
// model's (kernels.cpp:125-136 of the reference).
#include <algorithm>
#include <atomic>
#include <cstring>
#include <thread>
#include <vector>

#include "common.cuh"
#include "kernels.h"
#include "tma.cuh"

namespace rlb {

namespace {
constexpr int kRB = kSpmvTiledRows;         // rows per block (one CTA)
constexpr int kWarps = 16;
constexpr int kThreads = kWarps * 32;
constexpr int kRowsPerWarp = kRB / kWarps;  // 512 -> 9-bit row field
#ifndef RLB_TILED_T
#define RLB_TILED_T 2048
#endif
#ifndef RLB_TILED_EMAX
#define RLB_TILED_EMAX 2048
#endif
#ifndef RLB_TILED_STAGES
#define RLB_TILED_STAGES 3
#endif
constexpr int kT = RLB_TILED_T;             // max tile width (columns, <= 2048: 11-bit column field)
constexpr int kEMax = RLB_TILED_EMAX;       // max nonzeros per tile
constexpr int kPerLane = 4;                 // consecutive entries a lane owns in a round
constexpr int kRound = 32 * kPerLane;       // entries a warp consumes per round
constexpr int kEPad = kEMax + (kPerLane - 1) * kWarps;  // warp chunks padded to multiples of 4
constexpr int kStages = RLB_TILED_STAGES;

__host__ __device__ constexpr size_t pad16(size_t b) { return (b + 15) & ~size_t(15); }
constexpr size_t kOffBytes = 64;  // kWarps + 1 u16 chunk offsets
constexpr size_t kSegMax = kOffBytes + (size_t)kEPad * 12;
constexpr size_t kXBytes = (size_t)kT * 8;
constexpr size_t kStageBytes = kXBytes + kSegMax;
constexpr size_t kYBytes = (size_t)kRB * 8;
constexpr int kDescCache = 512;  // tile descriptors staged in shared memory (later ones read from global)
constexpr size_t kSmem = kStages * kStageBytes + kYBytes + kDescCache * sizeof(SpmvTile) + kStages * 8 + kStages * 4;
static_assert(kSmem <= 227 * 1024, "tiled SpMV shared memory");
static_assert(kStageBytes % 128 == 0 && kSegMax % 16 == 0, "stage alignment");

// metadata word of one entry
constexpr uint32_t kColMask = (1u << 11) - 1;  // bits 0-10: column in the tile
constexpr int kRowShift = 11;                  // bits 11-19: row in the warp's 512
constexpr uint32_t kValid = 1u << 20;          // real nonzero (0 = padding)
constexpr uint32_t kStart = 1u << 21;          // first entry of its row's run in this round
constexpr uint32_t kEnd = 1u << 22;            // last entry of its row's run in this round
constexpr int kDepthShift = 23;                // bits 23-27 (lane's first entry): lanes the carry spans
constexpr uint32_t kLaneStart = 1u << 28;      // (lane's first entry) a run starts in this lane

using namespace tmaop;  // mbarrier / bulk-copy primitives (tma.cuh)

__global__ void __launch_bounds__(kThreads, 1) spmv_tiled_kernel(uint64_t m, uint64_t b_first,
                                                                 const uint8_t* __restrict__ segs,
                                                                 const SpmvTile* __restrict__ tiles,
                                                                 const int* __restrict__ blk_tiles,
                                                                 const double* __restrict__ x,
                                                                 double* __restrict__ y) {
    extern __shared__ __align__(128) uint8_t smem[];
    double* ysm = reinterpret_cast<double*>(smem + kStages * kStageBytes);
    SpmvTile* desc = reinterpret_cast<SpmvTile*>(smem + kStages * kStageBytes + kYBytes);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes + kYBytes +
                                                 kDescCache * sizeof(SpmvTile));
    uint32_t* cnt = reinterpret_cast<uint32_t*>(full + kStages);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t b = b_first + blockIdx.x;
    const int t0 = blk_tiles[b], t1 = blk_tiles[b + 1];
    const int nt = t1 - t0;
    double* yw = ysm + warp * kRowsPerWarp;
#pragma unroll
    for (int i = 0; i < kRowsPerWarp / 32; ++i) yw[lane + 32 * i] = 0.0;
    for (int i = tid; i < nt && i < kDescCache; i += kThreads) desc[i] = tiles[t0 + i];
    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(full + s, 1);
            cnt[s] = 0;
        }
        mbar_fence_init();
    }
    __syncthreads();
    auto issue = [&](int k) {
        const SpmvTile t = k < kDescCache ? desc[k] : tiles[t0 + k];
        uint8_t* st = smem + (k % kStages) * kStageBytes;
        const uint32_t xb = (uint32_t)(t.width * 8);
        const uint32_t sb = (uint32_t)t.seg_bytes;
        uint64_t* bar = full + (k % kStages);
        mbar_expect_tx(bar, xb + sb);
        bulk_g2s(st, x + t.col_base, xb, bar, policy_evict_last());
        bulk_g2s(st + kXBytes, segs + t.seg_offset, sb, bar, policy_evict_first());
    };
    if (tid == 0)
        for (int k = 0; k < kStages && k < nt; ++k) issue(k);
    for (int k = 0; k < nt; ++k) {
        const int s = k % kStages;
        const uint32_t parity = (uint32_t)((k / kStages) & 1);
        mbar_wait_hint(full + s, parity, 1000000u);
        const uint8_t* st = smem + s * kStageBytes;
        const double* xs = reinterpret_cast<const double*>(st);
        const uint8_t* seg = st + kXBytes;
        const uint16_t* offs = reinterpret_cast<const uint16_t*>(seg);
        const int E = offs[kWarps], e0 = offs[warp], e1 = offs[warp + 1];
        const double* vals = reinterpret_cast<const double*>(seg + kOffBytes);
        const uint32_t* meta = reinterpret_cast<const uint32_t*>(seg + kOffBytes + (size_t)E * 8);
        for (int base = e0; base < e1; base += kRound) {
            const int e = base + kPerLane * lane;  // chunk lengths are multiples of 4
            double p[kPerLane] = {0.0, 0.0, 0.0, 0.0};
            uint32_t mt[kPerLane] = {0u, 0u, 0u, 0u};
            if (e < e1) {
                const uint4 m4 = *reinterpret_cast<const uint4*>(meta + e);
                const double2 va = *reinterpret_cast<const double2*>(vals + e);
                const double2 vb = *reinterpret_cast<const double2*>(vals + e + 2);
                mt[0] = m4.x, mt[1] = m4.y, mt[2] = m4.z, mt[3] = m4.w;
                const double v[kPerLane] = {va.x, va.y, vb.x, vb.y};
#pragma unroll
                for (int j = 0; j < kPerLane; ++j)
                    if (mt[j] & kValid) p[j] = v[j] * xs[mt[j] & kColMask];
            }
            // lane tail: the running sum since the lane's last run start
            double t = 0.0;
#pragma unroll
            for (int j = 0; j < kPerLane; ++j) t = (mt[j] & kStart) ? p[j] : t + p[j];
            const int d = (int)((mt[0] >> kDepthShift) & 31);
            const int maxd = (int)__reduce_max_sync(0xffffffffu, (unsigned)d);
            double carry = 0.0;
            if (maxd > 0) {
                // segmented inclusive scan of the tails over lanes, only as
                // deep as the longest run crossing lane boundaries
                double T = t;
                bool f = (mt[0] & kLaneStart) || !(mt[0] & kValid);
                for (int o = 1; o < maxd; o <<= 1) {
                    const double q = __shfl_up_sync(0xffffffffu, T, o);
                    const bool fq = __shfl_up_sync(0xffffffffu, (int)f, o) != 0;
                    if (lane >= o && !f) {
                        T += q;
                        f = fq;
                    }
                }
                const double c = __shfl_up_sync(0xffffffffu, T, 1);
                if (d > 0) carry = c;
            }
            double run = carry;
#pragma unroll
            for (int j = 0; j < kPerLane; ++j) {
                run = (mt[j] & kStart) ? p[j] : run + p[j];
                if (mt[j] & kEnd) yw[(mt[j] >> kRowShift) & (kRowsPerWarp - 1)] += run;
            }
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
    std::vector<int> slot_row;       // per padded slot: row (-1 = padding)
    std::vector<const HostEntry*> slot_src;
    size_t p = 0;
    while (p < es.size()) {
        const int32_t c0 = es[p].col & ~1;
        const int64_t lim = std::min<int64_t>((int64_t)c0 + kT, (int64_t)n);
        size_t q = p;
        while (q < es.size() && es[q].col < lim && q - p < (size_t)kEMax) ++q;
        int32_t width = ((es[q - 1].col - c0) + 2) & ~1;
        if ((uint64_t)c0 + width > n) width = (int32_t)(n - c0);
        // entries by (row, column): each warp's chunk is contiguous, rows sorted
        std::stable_sort(es.begin() + p, es.begin() + q,
                         [](const HostEntry& a, const HostEntry& c) { return a.row < c.row; });
        const HostEntry* te = es.data() + p;
        const int E = (int)(q - p);
        // per-warp chunks padded to multiples of kPerLane
        int off[kWarps + 1];
        slot_row.clear();
        slot_src.clear();
        int cur = 0;
        for (int w = 0; w < kWarps; ++w) {
            off[w] = (int)slot_row.size();
            while (cur < E && te[cur].row / kRowsPerWarp == w) {
                slot_row.push_back(te[cur].row);
                slot_src.push_back(te + cur);
                ++cur;
            }
            while (slot_row.size() % kPerLane) {
                slot_row.push_back(-1);
                slot_src.push_back(nullptr);
            }
        }
        off[kWarps] = (int)slot_row.size();
        const int EP = off[kWarps];
        SpmvTile t{};
        t.seg_offset = segs.size();
        t.col_base = c0;
        t.width = width;
        t.entries = E;
        t.seg_bytes = (int)(kOffBytes + pad16((size_t)EP * 12));
        segs.resize(segs.size() + t.seg_bytes, 0);
        uint8_t* sb = segs.data() + t.seg_offset;
        uint16_t* o16 = reinterpret_cast<uint16_t*>(sb);
        double* v = reinterpret_cast<double*>(sb + kOffBytes);
        uint32_t* mt = reinterpret_cast<uint32_t*>(sb + kOffBytes + (size_t)EP * 8);
        for (int w = 0; w <= kWarps; ++w) o16[w] = (uint16_t)off[w];
        for (int w = 0; w < kWarps; ++w) {
            for (int rs = off[w]; rs < off[w + 1]; rs += kRound) {  // rounds
                const int re = std::min(rs + kRound, off[w + 1]);
                auto valid = [&](int i) { return i < re && slot_row[i] >= 0; };
                bool lane_start[32] = {};
                for (int i = rs; i < re; ++i) {
                    const bool st = valid(i) && (i == rs || slot_row[i] != slot_row[i - 1]);
                    const bool en = valid(i) && (!valid(i + 1) || slot_row[i + 1] != slot_row[i]);
                    uint32_t word = 0;
                    if (valid(i)) {
                        const HostEntry* h = slot_src[i];
                        v[i] = h->val;
                        word = (uint32_t)(h->col - c0) | ((uint32_t)(h->row % kRowsPerWarp) << kRowShift) | kValid;
                    }
                    if (st) {
                        word |= kStart;
                        lane_start[(i - rs) / kPerLane] = true;
                    }
                    if (en) word |= kEnd;
                    mt[i] = word;
                }
                // lane's first entry: does a run start in the lane, and how many
                // lanes back does its carried-in run begin
                for (int l = 0; l * kPerLane < re - rs; ++l) {
                    const int i = rs + l * kPerLane;
                    if (lane_start[l]) mt[i] |= kLaneStart;
                    if (!valid(i) || (mt[i] & kStart)) continue;
                    int dd = 1;
                    while (l - dd >= 0 && !lane_start[l - dd]) ++dd;
                    mt[i] |= (uint32_t)dd << kDepthShift;
                }
            }
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
