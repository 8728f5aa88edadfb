// stencil_r.cu -- TMA-pipelined 2D stencils of the other presets (SURVEY.md
// §8f next #4): 2d9pt (3x3 box), 2d13pt (radius-3 star) and 2d49pt (7x7
// box), the reference's stencil_presets() (kernels.cpp:54-58).  At B200
// balance 2d9pt and 2d13pt are HBM-bound (1.125 and 1.625 flop/B) and 2d49pt
// sits at the FP64 ridge (6.125 flop/B against ~5.6): its CUDA-core form is
// bound by the DFMA pipe, which is the case PAPER.md:592 calls compute-bound
// on A100.
//
// Layout and pipeline as in stencil_tma.cu: a CTA owns a 64-column strip and
// marches a row segment; one elected thread streams 32-row stages with their
// R-row / LP-column halos (LP = R rounded up to even, so the 16-byte-aligned
// TMA box starts at x0 - LP) through an S-stage mbarrier ring.
//
// CUDA core: thread = 2 adjacent columns x 8 rows.  Each input row is read
//   once per thread with 128-bit shared loads (LP+1 column pairs) and feeds
//   every output row within +-R of it, DFMA with the weights straight from
//   the kernel's parameter bank.  Per stage a warp issues 49*8*2 DFMA per
//   thread against 14*5 LDS.128 (2d49pt), so the FP64 pipe, not shared
//   memory, is the limit.  When the box weights are mirror-symmetric in x
//   (the presets' defaults are), u[x-b] + u[x+b] is formed once per input
//   row and reused by all 2R+1 output rows: 4 DFMA + 3/8*... DADD per
//   (input row, output row) instead of 7 DFMA, ~33 FP64 ops per 2d49pt
//   point instead of 49.
// Tensor core (DMMA m8n8k4): an 8x8 output tile is a sum of banded products
//   D += U_dy (8 x K) * B_dy (K x 8) with B_dy[k][n] = w(dy, k - n - R), K =
//   8 + 2R padded to a multiple of 4 (box: one product per row offset dy;
//   star: the dy = 0 product plus one transposed product Band_y (8 x K) * U
//   for the vertical arms).  The band fragments are built once per thread;
//   the U fragments come from the stage, whose row pitch is 4 mod 16 doubles
//   so each fragment load is two conflict-free wavefronts.  Per 8x8 tile:
//   2d9pt 9, 2d13pt 8, 2d49pt 28 DMMA; with y-mirror-symmetric box weights
//   (the defaults) the rows y-dy and y+dy are added before one shared
//   product, so 2d9pt takes 6 and 2d49pt 16.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <utility>

#include "common.cuh"
#include "kernels.h"
#include "tma.cuh"

namespace rlb {
namespace {

constexpr int kTXr = 64;   // columns per strip
constexpr int kTYr = 32;   // output rows per stage
constexpr int kRYr = 8;    // output rows per thread (CC) / per DMMA tile

using namespace tmaop;  // mbarrier / TMA primitives and the stage Ring (tma.cuh)

template <int R>
struct Geo {
    static constexpr int LP = (R + 1) & ~1;      // left pad: box starts at x0 - LP (16-byte aligned)
    static constexpr int ROWS = kTYr + 2 * R;    // stage rows
};
template <int R>
__host__ __device__ constexpr int ksteps() { return (8 + 2 * R + 3) / 4; }  // k-steps of a banded product (K = 8 + 2R)
// Stage pitch (doubles): CC needs 64 + 2 LP; TC needs the padded band
// columns in bounds (LP + 56 - R + 4 KS) and pads to 4 mod 16 for
// conflict-free 8x4 fragment loads.
template <int R, bool TC>
__host__ __device__ constexpr int pitch() {
    int p = kTXr + 2 * Geo<R>::LP;
    if (TC || R == 1) {  // the CUDA-core 2d9pt stage measured ~2.5 % faster with the wider box too
        const int need = Geo<R>::LP + 56 - R + 4 * ksteps<R>();
        if (p < need) p = need;
        while (p % 16 != 4) ++p;
    }
    return p;
}
// Stage rows allocated: the star's vertical product reads rows 8 ti + k for
// k < 4 KS, past the TMA box; those rows stay zero.
template <int R, bool TC>
__host__ __device__ constexpr int alloc_rows() {
    return (TC && Geo<R>::ROWS < 24 + 4 * ksteps<R>()) ? 24 + 4 * ksteps<R>() : Geo<R>::ROWS;
}
template <int R, bool TC>
__host__ __device__ constexpr int stage_doubles() {
    return ((alloc_rows<R, TC>() * pitch<R, TC>() * 8 + 127) / 128) * 128 / 8;
}
template <int R, bool TC, int S>
constexpr size_t ring_bytes() {
    return (size_t)S * stage_doubles<R, TC>() * 8 + 2 * S * 8;
}

// Canonical weight index (oracle/oracle.c preset_offsets) of offset (dy, dx).
template <int R, bool BOX>
__host__ __device__ constexpr int widx(int dy, int dx) {
    if (BOX) return (dy + R) * (2 * R + 1) + (dx + R);
    if (dy == 0 && dx == 0) return 0;
    if (dx == 0) return 1 + 4 * ((dy < 0 ? -dy : dy) - 1) + (dy < 0 ? 0 : 1);
    return 1 + 4 * ((dx < 0 ? -dx : dx) - 1) + (dx < 0 ? 2 : 3);
}
template <bool BOX>
__host__ __device__ constexpr bool has_tap(int dy, int dx) {
    return BOX || dy == 0 || dx == 0;
}

// Shared ring + producer for both units.

// Store two adjacent outputs (x, x+1) of row y when interior.
__device__ __forceinline__ void store_pair(double* v, uint64_t nx, int R, int64_t x, uint64_t y, double a,
                                           double b) {
    double* p = v + y * nx + x;
    const bool i0 = x >= R && x <= (int64_t)nx - 1 - R;
    const bool i1 = x + 1 >= R && x + 1 <= (int64_t)nx - 1 - R;
    if (i0 && i1)
        asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(a), "d"(b) : "memory");
    else {
        if (i0) p[0] = a;
        if (i1) p[1] = b;
    }
}

// ===========================================================================
// CUDA core
// ===========================================================================
// One input row (stage row IR of the thread's group) into every output row
// within +-R of it.
template <int R, bool BOX, bool SYM, int P, int IR>
__device__ __forceinline__ void cc_row(const double* T, const StencilDesc& d, double (&acc)[kRYr][2]) {
    constexpr int LP = Geo<R>::LP, NP = LP + 1;
    constexpr bool wide = BOX || (IR >= R && IR < R + kRYr);  // star: arms need only the centre
    double vv[2 * NP];
    const double* rowp = T + IR * P;
    if constexpr (wide) {
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            const double2 t = *reinterpret_cast<const double2*>(rowp + 2 * q);
            vv[2 * q] = t.x;
            vv[2 * q + 1] = t.y;
        }
    } else {
        const double2 t = *reinterpret_cast<const double2*>(rowp + LP);
        vv[LP] = t.x;
        vv[LP + 1] = t.y;
    }
    if constexpr (SYM && BOX) {
        // w(dy, dx) == w(dy, -dx): pair the columns once per input row (R DADD
        // per column), then R+1 DFMA per (input row, output row) instead of 2R+1
        double h[2][R + 1];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            h[c][0] = vv[LP + c];
#pragma unroll
            for (int b = 1; b <= R; ++b) h[c][b] = vv[LP + c - b] + vv[LP + c + b];
        }
#pragma unroll
        for (int b = 0; b <= R; ++b) {
#pragma unroll
            for (int j = 0; j < kRYr; ++j) {
                const int dy = IR - R - j;
                if (dy >= -R && dy <= R) {
                    const double w = d.w[widx<R, BOX>(dy, b)];
                    acc[j][0] = fma(w, h[0][b], acc[j][0]);
                    acc[j][1] = fma(w, h[1][b], acc[j][1]);
                }
            }
        }
    } else {
        // dx outer: consecutive DFMAs go to different accumulators
#pragma unroll
        for (int dx = -R; dx <= R; ++dx) {
#pragma unroll
            for (int j = 0; j < kRYr; ++j) {
                const int dy = IR - R - j;
                if (dy >= -R && dy <= R && has_tap<BOX>(dy, dx)) {
                    const double w = d.w[widx<R, BOX>(dy, dx)];
                    acc[j][0] = fma(w, vv[LP + dx], acc[j][0]);
                    acc[j][1] = fma(w, vv[LP + 1 + dx], acc[j][1]);
                }
            }
        }
    }
}
template <int R, bool BOX, bool SYM, int P, int... IR>
__device__ __forceinline__ void cc_rows(const double* T, const StencilDesc& d, double (&acc)[kRYr][2],
                                        std::integer_sequence<int, IR...>) {
    (cc_row<R, BOX, SYM, P, IR>(T, d, acc), ...);
}

template <int R, bool BOX, bool SYM, int S>
__global__ void __launch_bounds__(128) st2dr_tma_cc(const __grid_constant__ CUtensorMap tm, double* __restrict__ v,
                                                    uint64_t nx, uint64_t y_begin, uint64_t y_end, int seg_rows,
                                                    int strips, const __grid_constant__ StencilDesc d) {
    constexpr int LP = Geo<R>::LP, P = pitch<R, false>(), STAGE = stage_doubles<R, false>();
    extern __shared__ __align__(128) double smem[];
    Ring<S, STAGE> ring(smem);
    const int tid = threadIdx.x, lane = tid & 31, g = tid >> 5;
    const int64_t x0 = (int64_t)(blockIdx.x % strips) * kTXr;
    const uint64_t ya = y_begin + (uint64_t)(blockIdx.x / strips) * seg_rows;
    if (ya >= y_end) return;
    const uint64_t yb = min(ya + (uint64_t)seg_rows, y_end);
    const int nblk = (int)((yb - ya + kTYr - 1) / kTYr);
    ring.init(4);
    constexpr uint32_t kBytes = Geo<R>::ROWS * P * 8;
    if (tid == 0)
        for (int k = 0; k < S && k < nblk; ++k)
            ring.issue2d(k, &tm, (int)(x0 - LP), (int)(ya + (uint64_t)k * kTYr) - R, kBytes);
    const int64_t x = x0 + 2 * lane;
    for (int k = 0; k < nblk; ++k) {
        ring.wait_full(k);
        const double* T = ring.stage(k) + (kRYr * g) * P + 2 * lane;
        double acc[kRYr][2];
#pragma unroll
        for (int j = 0; j < kRYr; ++j) acc[j][0] = acc[j][1] = 0.0;
        // input rows as a compile-time sequence (dy, tap and weight index fold to constants)
        cc_rows<R, BOX, SYM, P>(T, d, acc, std::make_integer_sequence<int, kRYr + 2 * R>{});
        ring.release(k);
        if (tid == 0 && k + S < nblk) {
            ring.wait_empty(k);
            ring.issue2d(k + S, &tm, (int)(x0 - LP), (int)(ya + (uint64_t)(k + S) * kTYr) - R, kBytes);
        }
        const uint64_t yr = ya + (uint64_t)k * kTYr + kRYr * g;
#pragma unroll
        for (int j = 0; j < kRYr; ++j)
            if (yr + j < yb) store_pair(v, nx, R, x, yr + j, acc[j][0], acc[j][1]);
    }
}

// ===========================================================================
// Tensor core
// ===========================================================================
template <int R, bool BOX, bool SYMY, int S>
__global__ void __launch_bounds__(128) st2dr_tma_tc(const __grid_constant__ CUtensorMap tm, double* __restrict__ v,
                                                    uint64_t nx, uint64_t y_begin, uint64_t y_end, int seg_rows,
                                                    int strips, const __grid_constant__ StencilDesc d) {
    constexpr int LP = Geo<R>::LP, P = pitch<R, true>(), STAGE = stage_doubles<R, true>();
    constexpr int KS = ksteps<R>();
    // x-band products: one per row offset (box), or one per |dy| when the box
    // weights are mirror-symmetric in y (U[y-dy] + U[y+dy] share a band)
    constexpr int NDY = BOX ? (SYMY ? R + 1 : 2 * R + 1) : 1;
    extern __shared__ __align__(128) double smem[];
    Ring<S, STAGE> ring(smem);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int fr = lane >> 2, fc = lane & 3;   // fragment row / column
    const int64_t x0 = (int64_t)(blockIdx.x % strips) * kTXr;
    const uint64_t ya = y_begin + (uint64_t)(blockIdx.x / strips) * seg_rows;
    if (ya >= y_end) return;
    const uint64_t yb = min(ya + (uint64_t)seg_rows, y_end);
    const int nblk = (int)((yb - ya + kTYr - 1) / kTYr);
    // band fragments: x-band B_dy[k][n] = w(dy, k - n - R) (lane: k = 4s + fc, n = fr)
    double bx[NDY][KS];
#pragma unroll
    for (int i = 0; i < NDY; ++i) {
        const int dy = BOX ? (SYMY ? i : i - R) : 0;
#pragma unroll
        for (int s = 0; s < KS; ++s) {
            const int dx = 4 * s + fc - fr - R;
            double w = 0.0;
#pragma unroll
            for (int t = -R; t <= R; ++t)
                if (dx == t) w = d.w[widx<R, BOX>(dy, t)];
            bx[i][s] = w;
        }
    }
    // star: vertical band A[i][k] = w(k - i - R, 0), k != i + R (lane: i = fr, k = 4s + fc)
    double by[BOX ? 1 : KS];
    if (!BOX) {
#pragma unroll
        for (int s = 0; s < KS; ++s) {
            const int dy = 4 * s + fc - fr - R;
            double w = 0.0;
#pragma unroll
            for (int t = -R; t <= R; ++t)
                if (t != 0 && dy == t) w = d.w[widx<R, BOX>(t, 0)];
            by[s] = w;
        }
    }
    constexpr int XR = alloc_rows<R, true>() - Geo<R>::ROWS;  // zero rows past the box
    if (XR > 0)
        for (int i = tid; i < S * XR * P; i += blockDim.x)
            smem[(i / (XR * P)) * STAGE + Geo<R>::ROWS * P + i % (XR * P)] = 0.0;
    ring.init(4);
    constexpr uint32_t kBytes = Geo<R>::ROWS * P * 8;
    if (tid == 0)
        for (int k = 0; k < S && k < nblk; ++k)
            ring.issue2d(k, &tm, (int)(x0 - LP), (int)(ya + (uint64_t)k * kTYr) - R, kBytes);
    for (int k = 0; k < nblk; ++k) {
        ring.wait_full(k);
        const double* T = ring.stage(k);
        // warp: column tiles 2*warp, 2*warp+1; all four row tiles
        double acc[4][2][2];
#pragma unroll
        for (int ti = 0; ti < 4; ++ti)
#pragma unroll
            for (int c = 0; c < 2; ++c) acc[ti][c][0] = acc[ti][c][1] = 0.0;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const int tj = 2 * warp + c;
#pragma unroll
            for (int ti = 0; ti < 4; ++ti) {
                // x-band products: A = U[8ti + R + dy + fr][LP + 8tj - R + 4s + fc]
#pragma unroll
                for (int i = 0; i < NDY; ++i) {
                    const int dy = BOX ? (SYMY ? i : i - R) : 0;
                    const double* ap = T + (8 * ti + R + dy + fr) * P + (LP + 8 * tj - R + fc);
                    const double* am = T + (8 * ti + R - dy + fr) * P + (LP + 8 * tj - R + fc);
#pragma unroll
                    for (int s = 0; s < KS; ++s) {
                        const double a = (SYMY && dy > 0) ? ap[4 * s] + am[4 * s] : ap[4 * s];
                        dmma_m8n8k4(acc[ti][c][0], acc[ti][c][1], a, bx[i][s], acc[ti][c][0], acc[ti][c][1]);
                    }
                }
                if (!BOX) {
                    // vertical arms: D += Band_y (8 x K) * U[8ti + 4s + fc][LP + 8tj + fr]
                    const double* bp = T + (8 * ti + fc) * P + (LP + 8 * tj + fr);
#pragma unroll
                    for (int s = 0; s < KS; ++s)
                        dmma_m8n8k4(acc[ti][c][0], acc[ti][c][1], by[s], bp[4 * s * P], acc[ti][c][0],
                                    acc[ti][c][1]);
                }
            }
        }
        ring.release(k);
        if (tid == 0 && k + S < nblk) {
            ring.wait_empty(k);
            ring.issue2d(k + S, &tm, (int)(x0 - LP), (int)(ya + (uint64_t)(k + S) * kTYr) - R, kBytes);
        }
        const uint64_t ys = ya + (uint64_t)k * kTYr;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const int64_t x = x0 + 8 * (2 * warp + c) + 2 * fc;
#pragma unroll
            for (int ti = 0; ti < 4; ++ti) {
                const uint64_t y = ys + 8 * ti + fr;
                if (y < yb) store_pair(v, nx, R, x, y, acc[ti][c][0], acc[ti][c][1]);
            }
        }
    }
}

template <class K>
cudaError_t prep(K kernel, size_t smem) {
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

// Box weights mirror-symmetric in x (w(dy, dx) == w(dy, -dx), exactly)?
template <int R>
bool x_symmetric(const StencilDesc& d) {
    for (int dy = -R; dy <= R; ++dy)
        for (int dx = 1; dx <= R; ++dx)
            if (d.w[widx<R, true>(dy, dx)] != d.w[widx<R, true>(dy, -dx)]) return false;
    return true;
}

// Box weights mirror-symmetric in y (w(dy, dx) == w(-dy, dx), exactly)?
template <int R>
bool y_symmetric(const StencilDesc& d) {
    for (int dy = 1; dy <= R; ++dy)
        for (int dx = -R; dx <= R; ++dx)
            if (d.w[widx<R, true>(dy, dx)] != d.w[widx<R, true>(-dy, dx)]) return false;
    return true;
}

template <int R, bool BOX>
cudaError_t launch_r(int unit, const StencilDesc& d, uint64_t o0, uint64_t o1, const double* u, double* v,
                     cudaStream_t s) {
    constexpr int S = 4;
    CUtensorMap m;
    const uint32_t bx = (uint32_t)(unit == 1 ? pitch<R, true>() : pitch<R, false>());
    if (!encode_map_2d(&m, u, d.nx, d.ny, bx, (uint32_t)Geo<R>::ROWS, tuning().stencil_r_l2promo))
        return cudaErrorInvalidValue;
    const uint64_t strips = (d.nx + kTXr - 1) / kTXr;
    // split the rows so the grid is many waves deep (balance across 148 SMs)
    const uint64_t want = (uint64_t)kNumSMs * (uint64_t)(tuning().stencil_r_ctas_per_sm);
    uint64_t nseg = strips >= want ? 1 : (want + strips - 1) / strips;
    const uint64_t cap = (o1 - o0 + 63) / 64;
    if (nseg > cap) nseg = cap;
    if (nseg < 1) nseg = 1;
    const int seg_rows = (int)(((o1 - o0 + nseg - 1) / nseg + kTYr - 1) / kTYr * kTYr);
    const uint64_t segs = (o1 - o0 + seg_rows - 1) / seg_rows;
    const unsigned grid = (unsigned)(strips * segs);
    cudaError_t e;
    if (unit == 1) {
        // stages: radius 3's DMMA chains need warps more than ring depth (4
        // stages leave 2 CTAs = 8 warps per SM, `wait`-stalled).  Measured
        // 16384^2 GB/s at 2 / 4 stages: 2d49pt 3650 / 3105, 2d13pt 5950 / 5690,
        // 2d9pt 5870 / 6220.
        int st = tuning().stencil_r_tc_stages;
        if (st == 0) st = R == 3 ? 2 : S;
#define RLB_RTC(SY, SS)                                                                                     \
    do {                                                                                                    \
        const size_t sm = ring_bytes<R, true, SS>();                                                        \
        if ((e = prep(st2dr_tma_tc<R, BOX, SY, SS>, sm)) != cudaSuccess) return e;                         \
        st2dr_tma_tc<R, BOX, SY, SS><<<grid, 128, sm, s>>>(m, v, d.nx, o0, o1, seg_rows, (int)strips, d); \
    } while (0)
        if (BOX && y_symmetric<R>(d) && tuning().stencil_r_sym) {
            if (st == 2) RLB_RTC(true, 2); else if (st == 3) RLB_RTC(true, 3); else RLB_RTC(true, 4);
        } else {
            if (st == 2) RLB_RTC(false, 2); else if (st == 3) RLB_RTC(false, 3); else RLB_RTC(false, 4);
        }
#undef RLB_RTC
    } else {
        int st = tuning().stencil_r_cc_stages;
        if (st == 0) st = (R == 3 && BOX) ? 2 : 4;  // 2d49pt: compute-bound, more CTAs beat a deeper ring
#define RLB_RCC(SY, SS)                                                                                     \
    do {                                                                                                    \
        const size_t sm = ring_bytes<R, false, SS>();                                                       \
        if ((e = prep(st2dr_tma_cc<R, BOX, SY, SS>, sm)) != cudaSuccess) return e;                         \
        st2dr_tma_cc<R, BOX, SY, SS><<<grid, 128, sm, s>>>(m, v, d.nx, o0, o1, seg_rows, (int)strips, d); \
    } while (0)
        if (BOX && x_symmetric<R>(d) && tuning().stencil_r_sym) {
            if (st == 2) RLB_RCC(true, 2); else if (st == 3) RLB_RCC(true, 3); else RLB_RCC(true, 4);
        } else {
            if (st == 2) RLB_RCC(false, 2); else if (st == 3) RLB_RCC(false, 3); else RLB_RCC(false, 4);
        }
#undef RLB_RCC
    }
    note_launch();
    return cudaGetLastError();
}

}  // namespace

bool stencil_r_eligible(const StencilDesc& d, const double* u, const double* v) {
    if (d.preset != kP2d9 && d.preset != kP2d13 && d.preset != kP2d49) return false;
    if (d.nx % 2 != 0) return false;  // row pitch must be a multiple of 16 bytes
    if ((reinterpret_cast<uintptr_t>(u) & 15) || (reinterpret_cast<uintptr_t>(v) & 15)) return false;
    if (d.nx > (1ull << 31) || d.ny > (1ull << 31)) return false;
    return tma_encode_available();
}

cudaError_t launch_stencil_r(int unit, const StencilDesc& d, uint64_t o0, uint64_t o1, const double* u, double* v,
                             cudaStream_t s) {
    switch (d.preset) {
        case kP2d9: return launch_r<1, true>(unit, d, o0, o1, u, v, s);
        case kP2d13: return launch_r<3, false>(unit, d, o0, o1, u, v, s);
        case kP2d49: return launch_r<3, true>(unit, d, o0, o1, u, v, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace rlb
