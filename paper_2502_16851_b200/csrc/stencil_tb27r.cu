// stencil_tb27r.cu -- 3d27pt temporal blocking of depth 2, register-blocked
// (SURVEY.md §8f "next" #1; at B200's balance a 3d27pt
// sweep fused over t = 2 timesteps is already compute-bound,
// min_temporal_depth = 2; stencil_model(shape, P, t), kernels.cpp:137-155).
//
// The march of stencil_tb3r.cu (3d7pt) with the 27-point box in class form,
// w(dx, dy, dz) = g(|dx| + |dy| + |dz|):
//   * A CTA of NW warps owns a 64-column x NW*H-row tile (plus the halo) and
//     marches z; one thread streams the input planes into a ring of TMA
//     stages.  Warp w owns rows [w H, w H + H), lane l columns 2l and 2l+1.
//   * In-plane class sums of a plane at every point: E (the 4 edge
//     neighbours) and K (the 4 corners), with the left / right neighbours one
//     shuffle away and the rows above / below the warp from the stage (level
//     1) or from the edge-row slots (level 2).  A plane contributes
//         s1 = g1 c + g2 E + g3 K   to the planes above and below,
//         s0 = g0 c + g1 E + g2 K   to its own plane.
//   * Each level keeps two partial-sum planes: when plane q arrives (a raw
//     plane from its stage for level 1, level 1's output for level 2) it
//     finishes q-1 (A + s1(q)), A <- B + s0(q), B <- s1(q), so every plane's
//     in-plane sums are formed once per level.  The levels are
//     skewed by one input plane, so the only cross-warp data -- level 1's
//     first / last rows -- goes through a double-buffered shared slot: one
//     barrier per input plane.
// Dirichlet points (any coordinate on the first or last index) keep their
// value at both levels.  Class weights only (the BASELINE form; general 27
// weights take the z-column kernel, stencil_tb3.cu).
#include <cuda.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "tma.cuh"

namespace rlb {
namespace {
using namespace tmaop;

constexpr int kT = 2;

template <int H, int NW>
struct Tb27Geom {
    static constexpr int LX = 64;
    static constexpr int TL = 2;                 // x halo (even: 16-byte aligned boxes)
    static constexpr int LY = NW * H;
    static constexpr int TYO = LY - 2 * kT;
    static constexpr int STAGE = LX * LY;
    static constexpr int SLOT = NW * 2 * LX;     // level 1's edge rows: [warp][first, last][LX]
    static constexpr int XCH = 2 * SLOT;         // [parity]
};

template <int S, int H, int NW>
constexpr size_t tb27_smem() {
    using G = Tb27Geom<H, NW>;
    return (size_t)(S * G::STAGE + G::XCH) * 8 + S * 8;
}

struct G4 {
    double g0, g1, g2, g3;
};

__device__ __forceinline__ void ld2(double (&r)[2], const double* p) {
    const double2 t = *reinterpret_cast<const double2*>(p);
    r[0] = t.x;
    r[1] = t.y;
}
__device__ __forceinline__ void st2(double* p, double a, double b) {
    *reinterpret_cast<double2*>(p) = make_double2(a, b);
}

// s1 / s0 of one plane at the thread's H x 2 points: rows a[0..H-1], the row
// above (up) and below (dn) the warp.  Left / right neighbours by shuffle
// (lane 0's left and lane 31's right are outside every stored output's cone).
template <int H>
__device__ __forceinline__ void plane_sums(const double (&a)[H][2], const double (&up)[2], const double (&dn)[2],
                                           const G4& g, double (&s1)[H][2], double (&s0)[H][2]) {
    double lf[H + 2], rt[H + 2];  // row index + 1: 0 = up, H + 1 = dn
    lf[0] = __shfl_up_sync(0xffffffffu, up[1], 1);
    rt[0] = __shfl_down_sync(0xffffffffu, up[0], 1);
#pragma unroll
    for (int h = 0; h < H; ++h) {
        lf[h + 1] = __shfl_up_sync(0xffffffffu, a[h][1], 1);
        rt[h + 1] = __shfl_down_sync(0xffffffffu, a[h][0], 1);
    }
    lf[H + 1] = __shfl_up_sync(0xffffffffu, dn[1], 1);
    rt[H + 1] = __shfl_down_sync(0xffffffffu, dn[0], 1);
#pragma unroll
    for (int h = 0; h < H; ++h) {
        const double n0 = h > 0 ? a[h - 1][0] : up[0], n1 = h > 0 ? a[h - 1][1] : up[1];
        const double d0 = h < H - 1 ? a[h + 1][0] : dn[0], d1 = h < H - 1 ? a[h + 1][1] : dn[1];
        const double e0 = (n0 + d0) + (lf[h + 1] + a[h][1]);
        const double e1 = (n1 + d1) + (a[h][0] + rt[h + 1]);
        const double k0 = (lf[h] + n1) + (lf[h + 2] + d1);
        const double k1 = (n0 + rt[h]) + (d0 + rt[h + 2]);
        s1[h][0] = fma(g.g3, k0, fma(g.g2, e0, g.g1 * a[h][0]));
        s1[h][1] = fma(g.g3, k1, fma(g.g2, e1, g.g1 * a[h][1]));
        s0[h][0] = fma(g.g2, k0, fma(g.g1, e0, g.g0 * a[h][0]));
        s0[h][1] = fma(g.g2, k1, fma(g.g1, e1, g.g0 * a[h][1]));
    }
}

template <int H, int NW>
struct Tb27Ctx {
    const double* sg0;  // this thread's first row in stage 0
    const double* xr0;  // edge slot read: the warp above's last row
    const double* xd0;  //                 the warp below's first row
    double* xw0;        // edge slot write: this warp's first / last row
    double* dst;        // output of the plane level 2 emits at k = 0
    int64_t pstride;
    int oru, ord, nx, nz, i0, za, zb, nin, K;
    uint32_t bnd, stm;
};

template <int H, int NW, int S, bool EDGE>
__device__ __forceinline__ void tb27_march(const Tb27Ctx<H, NW>& cx, const G4& g, const CUtensorMap* tm,
                                           double* stage, uint64_t* full, int bx0, int by0) {
    using G = Tb27Geom<H, NW>;
    constexpr int LX = G::LX;
    static_assert(S % 2 == 0 && S >= 4, "the march is unrolled by S");
    // level 2: ring[par] = arrival (level 1's plane q), ring[par ^ 1] = q - 1;
    // A = the plane q - 1 waiting for its dz = +1 term, B = plane q's dz = -1 term
    // level 1: A1 / B1 likewise, pv1 = the previous raw plane (Dirichlet values)
    double ring[2][H][2], A[H][2], B[H][2], A1[H][2], B1[H][2], pv1[H][2];
#pragma unroll
    for (int h = 0; h < H; ++h)
#pragma unroll
        for (int c = 0; c < 2; ++c)
            ring[0][h][c] = ring[1][h][c] = A[h][c] = B[h][c] = A1[h][c] = B1[h][c] = pv1[h][c] = 0.0;
    const int tid = threadIdx.x;
    double* dst = cx.dst;
    for (int k0 = 0; k0 < cx.K; k0 += S) {
        const uint32_t ph = (uint32_t)((k0 / S) & 1);
#pragma unroll
        for (int j = 0; j < S; ++j) {
            const int k = k0 + j;
            if (k >= cx.K) break;
            const int par = j & 1;
            if (k < cx.nin) mbar_wait(full + j, ph);
            // level 2: consumes level 1's plane from the last iteration, emits r
            {
                const double(&a)[H][2] = ring[par];
                const double(&pv)[H][2] = ring[par ^ 1];
                const int so = (par ^ 1) * G::SLOT;
                double up[2], dn[2], s1[H][2], s0[H][2];
                ld2(up, cx.xr0 + so);
                ld2(dn, cx.xd0 + so);
                plane_sums<H>(a, up, dn, g, s1, s0);
                const int r = cx.i0 + k - 3;
                const bool zbd = r <= 0 || r >= cx.nz - 1;
                double out[H][2];
#pragma unroll
                for (int h = 0; h < H; ++h)
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        double o = A[h][c] + s1[h][c];
                        if (zbd) o = pv[h][c];
                        if constexpr (EDGE) {
                            if ((cx.bnd >> (2 * h + c)) & 1u) o = pv[h][c];
                        }
                        out[h][c] = o;
                        A[h][c] = B[h][c] + s0[h][c];
                        B[h][c] = s1[h][c];
                    }
                if (r >= cx.za && r < cx.zb) {
#pragma unroll
                    for (int h = 0; h < H; ++h) {
                        const uint32_t m = (cx.stm >> (2 * h)) & 3u;
                        double* p = dst + (int64_t)h * cx.nx;
                        if (m == 3u) __stcs(reinterpret_cast<double2*>(p), make_double2(out[h][0], out[h][1]));
                        if constexpr (EDGE) {
                            if (m == 1u) __stcs(p, out[h][0]);
                            if (m == 2u) __stcs(p + 1, out[h][1]);
                        }
                    }
                }
            }
            dst += cx.pstride;
            // level 1: the raw plane i0 + k arrives from its stage and finishes
            // plane p = i0 + k - 1 (the same partial-sum scheme as level 2, so
            // every plane's in-plane sums are formed once)
            if (k < cx.nin) {
                const double* sq = cx.sg0 + j * G::STAGE;
                double a[H][2], up[2], dn[2], s1[H][2], s0[H][2];
                ld2(up, sq + cx.oru);
#pragma unroll
                for (int h = 0; h < H; ++h) ld2(a[h], sq + h * LX);
                ld2(dn, sq + cx.ord);
                plane_sums<H>(a, up, dn, g, s1, s0);
                double(&out)[H][2] = ring[par ^ 1];
                const int p = cx.i0 + k - 1;
                const bool zbd = p <= 0 || p >= cx.nz - 1;
#pragma unroll
                for (int h = 0; h < H; ++h)
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        double o = A1[h][c] + s1[h][c];
                        if (zbd) o = pv1[h][c];
                        if constexpr (EDGE) {
                            if ((cx.bnd >> (2 * h + c)) & 1u) o = pv1[h][c];
                        }
                        out[h][c] = o;
                        A1[h][c] = B1[h][c] + s0[h][c];
                        B1[h][c] = s1[h][c];
                        pv1[h][c] = a[h][c];
                    }
                double* cs = cx.xw0 + par * G::SLOT;
                st2(cs, out[0][0], out[0][1]);
                st2(cs + LX, out[H - 1][0], out[H - 1][1]);
            }
            __syncthreads();  // edge slots of parity `par` published; plane k's stage consumed
            if (tid == 0 && k + S < cx.nin) {
                mbar_expect_tx(full + j, G::STAGE * 8);
                tma3d(stage + j * G::STAGE, tm, full + j, bx0, by0, cx.i0 + k + S);
            }
        }
    }
}

template <int H, int NW, int S>
__global__ void __launch_bounds__(NW * 32, 1)
    st3d27_tbr(const __grid_constant__ CUtensorMap tm, double* __restrict__ v, int nx, int ny, int nz, int z_begin,
               int z_end, int zchunk, int tiles_x, int tiles_y, const __grid_constant__ StencilDesc d) {
    using G = Tb27Geom<H, NW>;
    constexpr int LX = G::LX;
    extern __shared__ __align__(128) double smem[];
    double* stage = smem;
    double* xch = smem + S * G::STAGE;
    uint64_t* full = reinterpret_cast<uint64_t*>(xch + G::XCH);

    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int tiles = tiles_x * tiles_y;
    const int tile = blockIdx.x % tiles;
    const int za = z_begin + (int)(blockIdx.x / tiles) * zchunk;
    if (za >= z_end) return;
    const int zb = min(za + zchunk, z_end);
    const int bx0 = (tile % tiles_x) * (LX - 2 * G::TL) - G::TL;
    const int by0 = (tile / tiles_x) * G::TYO - kT;

    Tb27Ctx<H, NW> cx;
    cx.i0 = za - kT;
    cx.nin = zb - za + 2 * kT;
    cx.K = zb - za + 3 * kT - 1;
    cx.za = za;
    cx.zb = zb;
    cx.nx = nx;
    cx.nz = nz;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) mbar_init(full + s, 1);
        mbar_fence_init();
    }
    for (int i = tid; i < G::XCH; i += NW * 32) xch[i] = 0.0;
    __syncthreads();
    if (tid == 0) {
        for (int j = 0; j < S && j < cx.nin; ++j) {
            mbar_expect_tx(full + j, G::STAGE * 8);
            tma3d(stage + j * G::STAGE, &tm, full + j, bx0, by0, cx.i0 + j);
        }
    }
    const G4 g{d.w[13], d.w[12], d.w[9], d.w[0]};
    const int gx = bx0 + 2 * lane, gy0 = by0 + w * H;
    cx.bnd = 0;
    cx.stm = 0;
#pragma unroll
    for (int h = 0; h < H; ++h)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const int x = gx + c, y = gy0 + h, lx = 2 * lane + c, ly = w * H + h;
            const bool in = x >= 0 && x < nx && y >= 0 && y < ny;
            const bool b = x <= 0 || x >= nx - 1 || y <= 0 || y >= ny - 1;
            const bool o = lx >= G::TL && lx < LX - G::TL && ly >= kT && ly < G::LY - kT;
            if (b) cx.bnd |= 1u << (2 * h + c);
            if (o && in && !b) cx.stm |= 1u << (2 * h + c);
        }
    cx.pstride = (int64_t)nx * ny;
    const int wu = w > 0 ? w - 1 : w, wd = w < NW - 1 ? w + 1 : w;
    const int ru = max(w * H - 1, 0), rd = min(w * H + H, G::LY - 1);
    cx.sg0 = stage + (w * H) * LX + 2 * lane;
    cx.oru = (ru - w * H) * LX;
    cx.ord = (rd - w * H) * LX;
    cx.xr0 = xch + (wu * 2 + 1) * LX + 2 * lane;
    cx.xd0 = xch + (wd * 2 + 0) * LX + 2 * lane;
    cx.xw0 = xch + w * 2 * LX + 2 * lane;
    cx.dst = v + (int64_t)(cx.i0 - 3) * cx.pstride + (int64_t)gy0 * nx + gx;
    const bool edge = bx0 <= 0 || bx0 + LX >= nx || by0 <= 0 || by0 + G::LY >= ny;
    if (edge)
        tb27_march<H, NW, S, true>(cx, g, &tm, stage, full, bx0, by0);
    else
        tb27_march<H, NW, S, false>(cx, g, &tm, stage, full, bx0, by0);
}

template <int H, int NW, int S>
cudaError_t launch_tb27(const StencilDesc& d, uint64_t o0, uint64_t o1, const double* u, double* v, cudaStream_t s) {
    using G = Tb27Geom<H, NW>;
    alignas(64) CUtensorMap m;
    if (!encode_map_3d(&m, u, d.nx, d.ny, d.nz, G::LX, G::LY, tuning().stencil_tb3_l2promo)) return cudaErrorInvalidValue;
    auto kern = st3d27_tbr<H, NW, S>;
    constexpr size_t smem = tb27_smem<S, H, NW>();
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NW * 32, smem) != cudaSuccess || occ < 1) occ = 1;
    const int tiles_x = (int)((d.nx + (G::LX - 2 * G::TL) - 1) / (G::LX - 2 * G::TL));
    const int tiles_y = (int)((d.ny + G::TYO - 1) / G::TYO);
    const long tiles = (long)tiles_x * tiles_y;
    const int planes = (int)(o1 - o0);
    // z chunks: minimise waves x (chunk + pipeline fill) over the resident slots
    int nch = tuning().stencil_tb3_chunks;
    if (nch <= 0) {
        const long slots = (long)kNumSMs * occ;
        double best = 1e300;
        const int cap = std::max(1, planes / (4 * kT));
        for (int c = 1; c <= cap; ++c) {
            const int zc = (planes + c - 1) / c;
            const long ctas = tiles * ((planes + zc - 1) / zc);
            const double waves = (double)((ctas + slots - 1) / slots);
            const double cost = waves * (zc + 3 * kT - 1);
            if (cost < best * 0.999) {
                best = cost;
                nch = c;
            }
        }
    }
    nch = std::max(1, std::min(nch, planes));
    const int zchunk = (planes + nch - 1) / nch;
    const int zch = (planes + zchunk - 1) / zchunk;
    kern<<<(unsigned)(tiles * zch), NW * 32, smem, s>>>(m, v, (int)d.nx, (int)d.ny, (int)d.nz, (int)o0, (int)o1,
                                                         zchunk, tiles_x, tiles_y, d);
    note_launch();
    return cudaGetLastError();
}

// Weights that depend only on |dx| + |dy| + |dz|.
bool class27(const StencilDesc& d) {
    const double g[4] = {d.w[13], d.w[12], d.w[9], d.w[0]};
    for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx)
                if (d.w[(dz + 1) * 9 + (dy + 1) * 3 + (dx + 1)] != g[std::abs(dx) + std::abs(dy) + std::abs(dz)])
                    return false;
    return true;
}

}  // namespace

bool stencil_tb27r_supported(const StencilDesc& d, int t, const double* u, const double* v) {
    if (d.preset != kP3d27 || t != 2 || !class27(d)) return false;
    if (d.nx % 2 != 0) return false;  // 16-byte row pitch for TMA and the paired stores
    if ((reinterpret_cast<uintptr_t>(u) & 15) || (reinterpret_cast<uintptr_t>(v) & 15)) return false;
    if (d.nx >= (1u << 30) || d.ny >= (1u << 30) || d.nz >= (1u << 30)) return false;
    return tma_encode_available();
}

cudaError_t launch_stencil_tb27r(const StencilDesc& d, int t, uint64_t o0, uint64_t o1, const double* u, double* v,
                                 cudaStream_t s) {
    if (!stencil_tb27r_supported(d, t, u, v)) return cudaErrorInvalidValue;
    // rows per warp x warps: 2 x 8 (256 threads, 118 registers, two CTAs per SM) measured 0.315 ms per
    // timestep; 2 x 16 0.335, 4 x 8 0.331, 1 x 32 0.409 (tools/micro/tb27_shapes.py)
    if (tuning().stencil_tb3_shape == 3) return launch_tb27<2, 16, 6>(d, o0, o1, u, v, s);
    return launch_tb27<2, 8, 6>(d, o0, o1, u, v, s);
}

}  // namespace rlb
