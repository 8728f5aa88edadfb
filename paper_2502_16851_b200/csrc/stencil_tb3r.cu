// stencil_tb3r.cu -- 3d7pt temporal blocking of depth T, register-blocked
// and skewed (SURVEY.md §8f "next" #1 for 3D; PAPER.md:223-236;
// stencil_model(shape, P, t), kernels.cpp:137-155).
//
// A CTA owns a 64-column x LY-row tile (plus the shrinking T-halo) and
// marches z through a chunk.  One elected thread streams the input planes
// into a ring of shared-memory stages with 3D TMA boxes (OOB cells arrive as
// zeros).  Warp w owns rows [w H, w H + H) of the tile, lane l owns columns
// 2l and 2l + 1, so every in-plane neighbour except the warp's first/last
// row is in the thread's own registers or one shuffle away.
//
// Each level keeps two planes per thread: the previous input plane `pv` and
// the partial sum `ac` of the plane waiting for its z+1 term.  When plane p
// of level l-1 arrives:
//     out_l(p-1) = ac + w_z+ a_p        (the finished plane, emitted)
//     ac         = w_0 a_p + w_z- pv + w_y-+ a(y-+1) + w_x-+ a(x-+1)
//     pv         = a_p
// The levels are skewed by one input plane: level l consumes in iteration k
// what level l-1 emitted in iteration k-1, so the only cross-warp data (the
// first/last row of each warp's emitted plane) goes through a double-buffered
// shared-memory slot and the CTA needs ONE barrier per input plane.  Level 1
// reads its input (and the rows above/below each warp) straight from the TMA
// stage.
//
// Dirichlet points (any coordinate on the first or last index of the grid)
// keep their value at every level; out-of-grid cells only feed boundary
// points or points outside the stored tile's dependency cone.
#include <cuda.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "tma.cuh"

namespace rlb {
namespace {
using namespace tmaop;

template <int T, int H, int NW>
struct Tb3rGeom {
    static constexpr int LX = 64;               // loaded columns (2 per lane)
    static constexpr int TL = T + (T & 1);      // x halo, even so boxes start 16-byte aligned
    static constexpr int TXO = LX - 2 * TL;     // output columns per tile
    static constexpr int LY = NW * H;           // loaded rows
    static constexpr int TYO = LY - 2 * T;      // output rows per tile
    static constexpr int STAGE = LX * LY;       // doubles per TMA stage
    static constexpr int SLOT = NW * 2 * LX;    // one level's edge rows: [warp][first, last][LX]
    static constexpr int XCH = 2 * (T - 1) * SLOT;  // [parity][level][...]
    static_assert(TYO > 0 && TXO > 0, "tile smaller than its halo");
};

template <int S, int T, int H, int NW>
constexpr size_t tb3r_smem() {
    using G = Tb3rGeom<T, H, NW>;
    return (size_t)(S * G::STAGE + G::XCH) * 8 + S * 8;
}

struct W7 {
    double c, zm, zp, ym, yp, xm, xp;
};

__device__ __forceinline__ void ld2(double (&r)[2], const double* p) {
    const double2 t = *reinterpret_cast<const double2*>(p);
    r[0] = t.x;
    r[1] = t.y;
}
__device__ __forceinline__ void st2(double* p, double a, double b) {
    *reinterpret_cast<double2*>(p) = make_double2(a, b);
}

// One level's step for the thread's H x 2 points: finish the pending plane
// with the arriving plane `a` (out) and start the partial sum of `a`; `pv`
// is the previous arrival.  Dirichlet points (bit 2h + c of `bnd`, or the
// whole plane when `zbd`) emit their previous value instead.
template <int H, bool EDGE>
__device__ __forceinline__ void level_step(const double (&a)[H][2], const double (&pv)[H][2], const double (&up)[2],
                                           const double (&dn)[2], const double (&lf)[H], const double (&rt)[H],
                                           double (&ac)[H][2], double (&out)[H][2], bool zbd, uint32_t bnd,
                                           const W7& w) {
#pragma unroll
    for (int h = 0; h < H; ++h)
#pragma unroll
        for (int c = 0; c < 2; ++c) out[h][c] = fma(w.zp, a[h][c], ac[h][c]);
    if (zbd) {
#pragma unroll
        for (int h = 0; h < H; ++h)
#pragma unroll
            for (int c = 0; c < 2; ++c) out[h][c] = pv[h][c];
    }
    if constexpr (EDGE) {
#pragma unroll
        for (int h = 0; h < H; ++h)
#pragma unroll
            for (int c = 0; c < 2; ++c)
                if ((bnd >> (2 * h + c)) & 1u) out[h][c] = pv[h][c];
    }
#pragma unroll
    for (int h = 0; h < H; ++h) {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const double ym = h > 0 ? a[h - 1][c] : up[c];
            const double yp = h < H - 1 ? a[h + 1][c] : dn[c];
            const double xm = c == 0 ? lf[h] : a[h][0];
            const double xp = c == 1 ? rt[h] : a[h][1];
            double n = w.c * a[h][c];
            n = fma(w.zm, pv[h][c], n);
            n = fma(w.ym, ym, n);
            n = fma(w.yp, yp, n);
            n = fma(w.xm, xm, n);
            n = fma(w.xp, xp, n);
            ac[h][c] = n;
        }
    }
}

// Per-CTA context of the march (everything loop-invariant).
template <int T, int H, int NW>
struct Tb3rCtx {
    const double* sg0;  // this thread's first row in stage 0
    const double* xr0;  // edge slot read: the warp above's last row
    const double* xd0;  //                 the warp below's first row
    double* xw0;        // edge slot write: this warp's first / last row
    double* dst;        // output of the plane level T emits at k = 0
    int64_t pstride;
    int oru, ord, nx, nz, i0, za, zb, nin, K;
    uint32_t bnd, stm;
};

// The z march.  EDGE = the tile touches the grid's x / y boundary (per-point
// Dirichlet masks, partial pair stores); interior tiles compile without them.
template <int T, int H, int NW, int S, bool EDGE>
__device__ __forceinline__ void tbr_march(const Tb3rCtx<T, H, NW>& cx, const W7& wt, const CUtensorMap* tm,
                                          double* stage, uint64_t* full, int bx0, int by0) {
    using G = Tb3rGeom<T, H, NW>;
    constexpr int LX = G::LX;
    static_assert(S % 2 == 0 && S >= 4, "the march is unrolled by S (stage and slot parity compile-time)");
    // Level l >= 2 keeps a 2-ring of its input planes: at iteration k it
    // consumes ring[l][k & 1] (emitted by level l-1 last iteration) with
    // ring[l][(k+1) & 1] as the previous plane; level l-1 then overwrites
    // the latter with its next emission.  ac[l] is the pending partial sum.
    double ring[T + 1][2][H][2], ac[T + 1][H][2];
#pragma unroll
    for (int l = 0; l <= T; ++l)
#pragma unroll
        for (int h = 0; h < H; ++h)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                ring[l][0][h][c] = ring[l][1][h][c] = 0.0;
                ac[l][h][c] = 0.0;
            }
    const int tid = threadIdx.x;
    double* dst = cx.dst;
    for (int k0 = 0; k0 < cx.K; k0 += S) {
        const uint32_t ph = (uint32_t)((k0 / S) & 1);
#pragma unroll
        for (int j = 0; j < S; ++j) {
            const int k = k0 + j;
            if (k >= cx.K) break;
            const int par = j & 1;
            if (k < cx.nin) mbar_wait(full + j, ph);  // input plane k (issued S - 2 iterations ago)
            // Levels T..2 (descending: level l reads ring[l] before level l-1 refills it).
#pragma unroll
            for (int l = T; l >= 2; --l) {
                const double(&a)[H][2] = ring[l][par];
                const double(&pv)[H][2] = ring[l][par ^ 1];
                const int so = ((par ^ 1) * (T - 1) + (l - 2)) * G::SLOT;
                double up[2], dn[2], lf[H], rt[H], out[H][2];
                ld2(up, cx.xr0 + so);
                ld2(dn, cx.xd0 + so);
#pragma unroll
                for (int h = 0; h < H; ++h) {
                    lf[h] = __shfl_up_sync(0xffffffffu, a[h][1], 1);
                    rt[h] = __shfl_down_sync(0xffffffffu, a[h][0], 1);
                }
                const int r = cx.i0 + k - (2 * l - 1);  // the plane level l emits now
                level_step<H, EDGE>(a, pv, up, dn, lf, rt, ac[l], out, r <= 0 || r >= cx.nz - 1, cx.bnd, wt);
                if (l < T) {
#pragma unroll
                    for (int h = 0; h < H; ++h) {
                        ring[l + 1][par ^ 1][h][0] = out[h][0];
                        ring[l + 1][par ^ 1][h][1] = out[h][1];
                    }
                    double* cs = cx.xw0 + (par * (T - 1) + (l - 1)) * G::SLOT;
                    st2(cs, out[0][0], out[0][1]);
                    st2(cs + LX, out[H - 1][0], out[H - 1][1]);
                } else if (r >= cx.za && r < cx.zb) {
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
            // Level 1 straight from the stages: plane p = i0 + k - 1 from the
            // resident input planes p - 1, p, p + 1 (no per-level state).
            if (k >= 2 && k < cx.nin) {
                const double* sm = cx.sg0 + ((j + S - 2) % S) * G::STAGE;
                const double* sc = cx.sg0 + ((j + S - 1) % S) * G::STAGE;
                const double* sp = cx.sg0 + j * G::STAGE;
                double cr[H + 2][2];
                double(&out)[H][2] = ring[2][par ^ 1];
                ld2(cr[0], sc + cx.oru);
#pragma unroll
                for (int h = 0; h < H; ++h) ld2(cr[h + 1], sc + h * LX);
                ld2(cr[H + 1], sc + cx.ord);
#pragma unroll
                for (int h = 0; h < H; ++h) {
                    double zm[2], zp[2];
                    ld2(zm, sm + h * LX);
                    ld2(zp, sp + h * LX);
                    const double xl = __shfl_up_sync(0xffffffffu, cr[h + 1][1], 1);
                    const double xr = __shfl_down_sync(0xffffffffu, cr[h + 1][0], 1);
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        double n = wt.c * cr[h + 1][c];
                        n = fma(wt.zm, zm[c], n);
                        n = fma(wt.zp, zp[c], n);
                        n = fma(wt.ym, cr[h][c], n);
                        n = fma(wt.yp, cr[h + 2][c], n);
                        n = fma(wt.xm, c == 0 ? xl : cr[h + 1][0], n);
                        n = fma(wt.xp, c == 1 ? xr : cr[h + 1][1], n);
                        out[h][c] = n;
                    }
                }
                const int r = cx.i0 + k - 1;
                if (r <= 0 || r >= cx.nz - 1) {
#pragma unroll
                    for (int h = 0; h < H; ++h) {
                        out[h][0] = cr[h + 1][0];
                        out[h][1] = cr[h + 1][1];
                    }
                }
                if constexpr (EDGE) {
#pragma unroll
                    for (int h = 0; h < H; ++h)
#pragma unroll
                        for (int c = 0; c < 2; ++c)
                            if ((cx.bnd >> (2 * h + c)) & 1u) out[h][c] = cr[h + 1][c];
                }
                double* cs = cx.xw0 + (par * (T - 1)) * G::SLOT;
                st2(cs, out[0][0], out[0][1]);
                st2(cs + LX, out[H - 1][0], out[H - 1][1]);
            }
            __syncthreads();  // edge slots of parity `par` published; plane k - 2's stage consumed
            if (tid == 0 && k >= 2 && k - 2 + S < cx.nin) {
                const int sj = (j + S - 2) % S;
                mbar_expect_tx(full + sj, G::STAGE * 8);
                tma3d(stage + sj * G::STAGE, tm, full + sj, bx0, by0, cx.i0 + k - 2 + S);
            }
        }
    }
}

template <int T, int H, int NW, int S>
__global__ void __launch_bounds__(NW * 32, NW * 32 <= 256 && T == 2 ? 2 : 1)
    st3d7_tbr(const __grid_constant__ CUtensorMap tm, double* __restrict__ v, int nx, int ny, int nz, int z_begin,
              int z_end, int zchunk, int tiles_x, int tiles_y, const __grid_constant__ StencilDesc d) {
    static_assert(T >= 2, "depth 1 is the plain sweep");
    using G = Tb3rGeom<T, H, NW>;
    constexpr int LX = G::LX;
    extern __shared__ __align__(128) double smem[];
    double* stage = smem;
    double* xch = smem + S * G::STAGE;
    uint64_t* full = reinterpret_cast<uint64_t*>(xch + G::XCH);

    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int tiles = tiles_x * tiles_y;
    const int tile = blockIdx.x % tiles;
    const int za = z_begin + (int)(blockIdx.x / tiles) * zchunk;
    if (za >= z_end) return;  // uniform per CTA
    const int zb = min(za + zchunk, z_end);
    const int bx0 = (tile % tiles_x) * G::TXO - G::TL;  // loaded region origin, even
    const int by0 = (tile / tiles_x) * G::TYO - T;

    Tb3rCtx<T, H, NW> cx;
    cx.i0 = za - T;                // first input plane
    cx.nin = zb - za + 2 * T;      // input planes za-T .. zb-1+T
    cx.K = zb - za + 3 * T - 1;    // iterations: level T emits plane i0 + k - (2T-1)
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

    const W7 wt{d.w[0], d.w[1], d.w[2], d.w[3], d.w[4], d.w[5], d.w[6]};
    const int gx = bx0 + 2 * lane, gy0 = by0 + w * H;
    cx.bnd = 0;
    cx.stm = 0;  // bit 2h + c: Dirichlet point / stored output point
#pragma unroll
    for (int h = 0; h < H; ++h)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const int x = gx + c, y = gy0 + h, lx = 2 * lane + c, ly = w * H + h;
            const bool in = x >= 0 && x < nx && y >= 0 && y < ny;
            const bool b = x <= 0 || x >= nx - 1 || y <= 0 || y >= ny - 1;
            const bool o = lx >= G::TL && lx < LX - G::TL && ly >= T && ly < G::LY - T;
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
    cx.dst = v + (int64_t)(cx.i0 - (2 * T - 1)) * cx.pstride + (int64_t)gy0 * nx + gx;
    // The tile's loaded region [bx0, bx0 + 64) x [by0, by0 + LY) holds no
    // boundary or out-of-grid point: no masks needed.
    const bool edge = bx0 <= 0 || bx0 + LX >= nx || by0 <= 0 || by0 + G::LY >= ny;
    if (edge)
        tbr_march<T, H, NW, S, true>(cx, wt, &tm, stage, full, bx0, by0);
    else
        tbr_march<T, H, NW, S, false>(cx, wt, &tm, stage, full, bx0, by0);
}

template <class K>
int occupancy(K kernel, int threads, size_t smem) {
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, smem) != cudaSuccess) n = 1;
    return std::max(n, 1);
}

template <int T, int H, int NW, int S>
cudaError_t launch_tbr(const StencilDesc& d, uint64_t o0, uint64_t o1, const double* u, double* v, cudaStream_t s) {
    using G = Tb3rGeom<T, H, NW>;
    alignas(64) CUtensorMap m;
    if (!encode_map_3d(&m, u, d.nx, d.ny, d.nz, G::LX, G::LY, tuning().stencil_tb3_l2promo)) return cudaErrorInvalidValue;
    auto kern = st3d7_tbr<T, H, NW, S>;
    constexpr size_t smem = tb3r_smem<S, T, H, NW>();
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    static const int occ = occupancy(kern, NW * 32, smem);  // per instantiation (same on every B200)
    const int tiles_x = (int)((d.nx + G::TXO - 1) / G::TXO), tiles_y = (int)((d.ny + G::TYO - 1) / G::TYO);
    const long tiles = (long)tiles_x * tiles_y;
    const int planes = (int)(o1 - o0);
    // z chunks: minimise waves x (chunk + pipeline fill) over the resident slots
    int nch = tuning().stencil_tb3_chunks;
    if (nch <= 0) {
        const long slots = (long)kNumSMs * occ;
        double best = 1e300;
        const int cap = std::max(1, planes / (4 * T));
        for (int c = 1; c <= cap; ++c) {
            const int zc = (planes + c - 1) / c;
            const long ctas = tiles * ((planes + zc - 1) / zc);
            const double waves = (double)((ctas + slots - 1) / slots);
            const double cost = waves * (zc + 3 * T - 1);
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

}  // namespace

bool stencil_tb3r_supported(const StencilDesc& d, int t, const double* u, const double* v) {
    if (d.preset != kP3d7 || t < 2 || t > 4) return false;
    if (d.nx % 2 != 0) return false;  // 16-byte row pitch for TMA and the paired stores
    if ((reinterpret_cast<uintptr_t>(u) & 15) || (reinterpret_cast<uintptr_t>(v) & 15)) return false;
    if (d.nx >= (1u << 30) || d.ny >= (1u << 30) || d.nz >= (1u << 30)) return false;
    return tma_encode_available();
}

cudaError_t launch_stencil_tb3r(const StencilDesc& d, int t, uint64_t o0, uint64_t o1, const double* u, double* v,
                                cudaStream_t s) {
    if (!stencil_tb3r_supported(d, t, u, v)) return cudaErrorInvalidValue;
    // shape: rows per warp x warps (tuning stencil_tb3_shape; 0 = the measured default per depth)
    const int shape = tuning().stencil_tb3_shape;
    switch (t) {
        case 2:
            if (shape == 2) return launch_tbr<2, 2, 16, 6>(d, o0, o1, u, v, s);
            if (shape == 3) return launch_tbr<2, 4, 16, 6>(d, o0, o1, u, v, s);
            return launch_tbr<2, 4, 8, 6>(d, o0, o1, u, v, s);
        case 3:
            return shape == 2 ? launch_tbr<3, 2, 16, 6>(d, o0, o1, u, v, s)
                              : launch_tbr<3, 4, 8, 6>(d, o0, o1, u, v, s);
        default:
            return shape == 2 ? launch_tbr<4, 2, 16, 6>(d, o0, o1, u, v, s)
                              : launch_tbr<4, 4, 8, 6>(d, o0, o1, u, v, s);
    }
}

}  // namespace rlb
