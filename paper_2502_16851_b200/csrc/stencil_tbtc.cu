// stencil_tbtc.cu -- 2d5pt temporal blocking of depth T on the tensor core
// (SURVEY.md §8f "next" #1, where temporal blocking is
// what could lift a stencil's intensity to the point where the matrix engine
// might matter; stencil_model(shape, P, t), kernels.cpp:137-155).
//
// Overlapped tiles in shared memory: a persistent CTA takes 64 x 64 output
// tiles in turn.  One 2D TMA box brings the tile plus a T-deep halo (out of
// grid: zeros) into the input buffer; T levels then sweep the buffer,
// ping-ponging between two more buffers, each level as the tensor-core form
// the single-step kernels use (stencil_tma.cu, st2d_tma_tch):
//     D = U . band(w_x-, 0, w_x+) + C,   C = w_c u + w_y- u[y-1] + w_y+ u[y+1]
// with the x-band on DMMA m8n8k4 (3 per 8 x 8 tile, K = 12) and C formed by
// DFMA at the accumulator positions.  Each level computes the whole 9 x 9
// tile grid of the buffer; the valid region shrinks by one point per level
// and after T levels is exactly the 64 x 64 output.  The next tile's box is
// issued as soon as level 1 has read the input buffer, so its load overlaps
// levels 2..T and the stores.  HBM sees one read of the (64 + 2T + ...)^2
// box and one write of the 64^2 tile per T timesteps.
//
// Dirichlet points (first or last row/column of the grid) keep their value
// at every level; out-of-grid cells hold zeros and only feed boundary points
// or points outside a stored output's dependency cone.
#include <cuda.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "tma.cuh"

namespace rlb {
namespace {
using namespace tmaop;

constexpr int kTile = 64;
constexpr int kWarps = 32;
constexpr int kTilesPerWarp = 3;  // 81 compute tiles per level over 32 warps, all three in flight

template <int T>
struct TbtcGeom {
    static constexpr int NT = (kTile + 2 * T + 7) / 8;   // 8 x 8 compute tiles per dimension
    static constexpr int BH = 8 * NT + 2;                // buffer rows: one guard row each side
    // buffer columns: two guard columns each side, pitch = 4 mod 16 doubles so
    // the fragment loads are conflict-free with the row permutation below
    static constexpr int BW = ((8 * NT + 4 + 11) / 16) * 16 + 4;
    static constexpr int XO = T + 2 + ((T & 1) ? 0 : 1); // buffer column of the tile's first output (odd: the
                                                         // box starts on an even global column, 16-byte aligned)
    static constexpr int YO = T + 1;                     // buffer row of the tile's first output
    static constexpr int BUF = BH * BW;
    static_assert(XO + kTile <= 2 + 8 * NT - (T - 1) && YO + kTile <= 1 + 8 * NT - (T - 1),
                  "the compute tiles must cover level 1's region");
};

template <int T>
constexpr size_t tbtc_smem() {
    return (size_t)3 * TbtcGeom<T>::BUF * 8 + 16;
}

// MMA row m <-> tile row with bits 0 and 1 swapped: with a 4 (mod 16) double
// pitch, the 16 lanes of an 8-byte load phase (rows 0-3 or 4-7) and the 8
// lanes of a 16-byte phase (rows 2k, 2k+1) then hit distinct banks.
__device__ __forceinline__ int frag_row(int r) { return (r & 4) | ((r & 1) << 1) | ((r >> 1) & 1); }

__device__ __forceinline__ double band(int k, int n, double wm, double wp) {
    return k == n + 1 ? wm : (k == n + 3 ? wp : 0.0);
}

template <int T>
__global__ void __launch_bounds__(kWarps * 32, 1)
    st2d5_tb_tc(const __grid_constant__ CUtensorMap tm, double* __restrict__ v, int nx, int ny, int tiles_x,
                int tiles, const __grid_constant__ StencilDesc d) {
    using G = TbtcGeom<T>;
    extern __shared__ __align__(128) double smem[];
    double* buf[3] = {smem, smem + G::BUF, smem + 2 * G::BUF};  // input box, two level buffers
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + 3 * G::BUF);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int r = lane >> 2, c = lane & 3, fr = frag_row(r);
    for (int i = tid; i < 3 * G::BUF; i += kWarps * 32) smem[i] = 0.0;  // finite guards for every level
    if (tid == 0) {
        mbar_init(full, 1);
        mbar_fence_init();
    }
    __syncthreads();
    const double w0 = d.w[0], wym = d.w[1], wyp = d.w[2];
    double bx[3];
#pragma unroll
    for (int kb = 0; kb < 3; ++kb) bx[kb] = band(4 * kb + c, r, d.w[3], d.w[4]);
    auto origin = [&](int k, int& x0, int& y0) {
        x0 = 1 + (k % tiles_x) * kTile;
        y0 = 1 + (k / tiles_x) * kTile;
    };
    auto issue = [&](int k) {
        int x0, y0;
        origin(k, x0, y0);
        mbar_expect_tx(full, G::BUF * 8);
        tma2d(buf[0], &tm, full, x0 - G::XO, y0 - G::YO);
    };
    if (tid == 0 && (int)blockIdx.x < tiles) issue(blockIdx.x);
    int it = 0;
    for (int k = blockIdx.x; k < tiles; k += gridDim.x, ++it) {
        int x0, y0;
        origin(k, x0, y0);
        mbar_wait(full, (uint32_t)(it & 1));
        // each warp computes the same compute tiles at every level, so a lane's
        // level-l output pair is its centre value at level l + 1 (registers)
        // (T = 4: the extra registers spill, the centre comes from shared memory)
        constexpr bool kRegCentre = T <= 3;
        double2 ct[kTilesPerWarp];
        for (int l = 1; l <= T; ++l) {
            const double* src = buf[l == 1 ? 0 : (l & 1 ? 2 : 1)];
            double* dst = buf[l & 1 ? 1 : 2];
            static_assert(kTilesPerWarp * kWarps >= G::NT * G::NT, "every compute tile has a warp");
            double a[kTilesPerWarp][3], d0[kTilesPerWarp], d1[kTilesPerWarp];
#pragma unroll
            for (int q = 0; q < kTilesPerWarp; ++q) {  // loads of all the warp's tiles first
                const int tt = min(warp + q * kWarps, G::NT * G::NT - 1);
                const int ti = tt / G::NT, tj = tt % G::NT;
                const double* pr = src + (1 + 8 * ti + fr) * G::BW;
                const int col = 2 + 8 * tj + 2 * c;
#pragma unroll
                for (int kb = 0; kb < 3; ++kb) a[q][kb] = pr[8 * tj + 4 * kb + c];
                if (l == 1 || !kRegCentre) ct[q] = *reinterpret_cast<const double2*>(pr + col);
                const double2 up = *reinterpret_cast<const double2*>(pr - G::BW + col);
                const double2 dn = *reinterpret_cast<const double2*>(pr + G::BW + col);
                d0[q] = fma(wyp, dn.x, fma(wym, up.x, w0 * ct[q].x));
                d1[q] = fma(wyp, dn.y, fma(wym, up.y, w0 * ct[q].y));
            }
#pragma unroll
            for (int kb = 0; kb < 3; ++kb)
#pragma unroll
                for (int q = 0; q < kTilesPerWarp; ++q) dmma_m8n8k4(d0[q], d1[q], a[q][kb], bx[kb], d0[q], d1[q]);
#pragma unroll
            for (int q = 0; q < kTilesPerWarp; ++q) {
                const int tt = warp + q * kWarps;
                if (tt >= G::NT * G::NT) break;
                const int ti = tt / G::NT, tj = tt % G::NT;
                const int row = 1 + 8 * ti + fr, col = 2 + 8 * tj + 2 * c;
                // Dirichlet and out-of-grid points keep their value
                const int gy = y0 - G::YO + row, gx = x0 - G::XO + col;
                const bool by = gy <= 0 || gy >= ny - 1;
                const double o0 = (by || gx <= 0 || gx >= nx - 1) ? ct[q].x : d0[q];
                const double o1 = (by || gx + 1 <= 0 || gx + 1 >= nx - 1) ? ct[q].y : d1[q];
                *reinterpret_cast<double2*>(dst + row * G::BW + col) = make_double2(o0, o1);
                ct[q] = make_double2(o0, o1);
            }
            __syncthreads();
            if (l == 1 && tid == 0 && k + (int)gridDim.x < tiles) issue(k + gridDim.x);  // input buffer is free
        }
        // the 64 x 64 output (interior points only; the Dirichlet ring is never written)
        const double* fin = buf[T & 1 ? 1 : 2];
        for (int i = tid; i < kTile * kTile; i += kWarps * 32) {
            const int oy = i / kTile, ox = i % kTile;
            const int gy = y0 + oy, gx = x0 + ox;
            if (gy < ny - 1 && gx < nx - 1) v[(int64_t)gy * nx + gx] = fin[(G::YO + oy) * G::BW + G::XO + ox];
        }
        __syncthreads();
    }
}

template <int T>
cudaError_t launch_tbtc(const StencilDesc& d, const double* u, double* v, cudaStream_t s) {
    using G = TbtcGeom<T>;
    alignas(64) CUtensorMap m;
    if (!encode_map_2d(&m, u, d.nx, d.ny, G::BW, G::BH, 1)) return cudaErrorInvalidValue;
    const int tiles_x = (int)((d.nx - 2 + kTile - 1) / kTile), tiles_y = (int)((d.ny - 2 + kTile - 1) / kTile);
    const int tiles = tiles_x * tiles_y;
    const size_t sm = tbtc_smem<T>();
    cudaError_t e = cudaFuncSetAttribute(st2d5_tb_tc<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    st2d5_tb_tc<T><<<std::min(tiles, kNumSMs), kWarps * 32, sm, s>>>(m, v, (int)d.nx, (int)d.ny, tiles_x, tiles, d);
    note_launch();
    return cudaGetLastError();
}

}  // namespace

bool stencil_tbtc_supported(const StencilDesc& d, int t, const double* u, const double* v) {
    if (d.preset != kP2d5 || t < 2 || t > 4) return false;
    if (d.nx < 3 || d.ny < 3 || d.nx % 2 != 0) return false;  // 16-byte row pitch for the TMA box
    if ((reinterpret_cast<uintptr_t>(u) & 15) || (reinterpret_cast<uintptr_t>(v) & 15)) return false;
    if (d.nx >= (1u << 30) || d.ny >= (1u << 30)) return false;
    return tma_encode_available();
}

// One fused sweep of t timesteps over the whole grid (interior rows 1..ny-2).
cudaError_t launch_stencil_tbtc(const StencilDesc& d, int t, const double* u, double* v, cudaStream_t s) {
    if (!stencil_tbtc_supported(d, t, u, v)) return cudaErrorInvalidValue;
    switch (t) {
        case 2: return launch_tbtc<2>(d, u, v, s);
        case 3: return launch_tbtc<3>(d, u, v, s);
        default: return launch_tbtc<4>(d, u, v, s);
    }
}

}  // namespace rlb
