// stencil_tma.cu -- TMA-pipelined Jacobi stencils (K5-K10, the default path
// on sm_100a when rows are 16-byte aligned).
//
// Every CTA (4 warps) owns a 64-column x 16-row tile and marches the slowest
// axis (y in 2D, z in 3D) through a chunk of it.  One elected thread streams
// the input through a ring of shared-memory stages with
// cp.async.bulk.tensor (TMA) and mbarrier transaction counts: a stage is the
// tile with its one-cell halo (18 rows x 68 columns; OOB cells arrive as
// zeros).  Measured on this B200/driver: the innermost start coordinate of
// a box must be 16-byte aligned (an odd FP64 x start raises "illegal
// instruction"; negative or past-the-end boxes are fine and zero-filled), so
// boxes start at x0 - 2 and are 68 wide (x0-2 .. x0+65): the stage column of
// x is x - x0 + 2.  Consumers read neighbours from the stage, release it with an
// mbarrier arrive, and the producer refills it S planes ahead, so 3-4 stages
// (~30 KB) are always in flight per CTA and ~150 KB per SM -- enough to cover
// HBM latency with no register prefetch queues.  Each u value crosses HBM
// once per sweep; halo rows/columns are L2 hits of the neighbouring tiles.
//
// CUDA core (DFMA):
//   2D: a stage holds 16 output rows + halo; thread = 1 column x 8 rows.
//   3D: a stage holds one plane of the tile; plane p contributes
//       P_{-1}(p) to output plane p+1, P_0(p) to p and P_{+1}(p) to p-1, so
//       one stage at a time suffices (7pt: P_{+-1} = w_z+- u; 27pt: 3x3 sums,
//       through class sums when w depends only on |dx|+|dy|+|dz|).
// Tensor core (DMMA m8n8k4, banded products as in stencil_tc.cu):
//   2D: 16 8x8 output tiles per stage, 4 per warp, 6 DMMA each.
//   3D: three consecutive planes stay resident (5-stage ring) and each output
//       plane is formed directly: 7pt 6 DMMA + DFMA z terms, 27pt class 9 DMMA,
//       27pt general 27 DMMA per 8x8 tile.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "common.cuh"
#include "kernels.h"
#include "tma.cuh"

namespace rlb {
namespace {

constexpr int kTX = 64, kTY = 16, kBY = kTY + 2;
constexpr int kBX = 68;   // box / stage row width (doubles)
constexpr int kCofs = 2;  // stage column of the tile's first x

using namespace tmaop;  // mbarrier / TMA primitives and the stage Ring (tma.cuh)

__host__ __device__ constexpr int stage_doubles(int bx) { return ((kBY * bx * 8 + 127) / 128) * 128 / 8; }
template <int S, int BX>
constexpr size_t ring_bytes() {
    return (size_t)S * stage_doubles(BX) * 8 + 2 * S * 8;
}

// Element (k, n) of band(a, b, c) (see stencil_tc.cu).
__device__ __forceinline__ double bandv(int k, int n, double a, double b, double c) {
    return k == n ? a : (k == n + 1 ? b : (k == n + 2 ? c : 0.0));
}

// ===========================================================================
// CUDA core, 2d5pt.  w: centre, y-1, y+1, x-1, x+1.
// ===========================================================================
template <int S, int RYT>
__global__ void __launch_bounds__(64 * kTY / RYT) st2d_tma_cc(const __grid_constant__ CUtensorMap tm,
                                                   double* __restrict__ v, uint64_t nx, uint64_t y_begin,
                                                   uint64_t y_end, int seg_rows, int strips, StencilDesc d) {
    constexpr int BX = kBX, STAGE = stage_doubles(BX);
    extern __shared__ __align__(128) double smem[];
    Ring<S, STAGE> ring(smem);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wx = warp & 1, wy = warp >> 1;
    const int64_t x0 = (int64_t)(blockIdx.x % strips) * kTX;
    const uint64_t ya = y_begin + (uint64_t)(blockIdx.x / strips) * seg_rows;
    if (ya >= y_end) return;
    const uint64_t yb = min(ya + (uint64_t)seg_rows, y_end);
    const int nblk = (int)((yb - ya + kTY - 1) / kTY);
    const int64_t xs = x0 - kCofs;
    const int cofs = kCofs;
    ring.init(2 * kTY / RYT);
    auto issue = [&](int k) {
        mbar_expect_tx(ring.full + (k % S), kBY * BX * 8);
        tma2d(ring.stage(k), &tm, ring.full + (k % S), (int)xs, (int)(ya + (uint64_t)k * kTY) - 1);
    };
    if (tid == 0)
        for (int k = 0; k < S && k < nblk; ++k) issue(k);
    const double w0 = d.w[0], w1 = d.w[1], w2 = d.w[2], w3 = d.w[3], w4 = d.w[4];
    const int col = 32 * wx + lane + cofs;
    const int cl = col > 0 ? col - 1 : 0;  // x-1 (clamped: only x = 0, a boundary column)
    const int64_t x = x0 + 32 * wx + lane;
    const bool xin = x >= 1 && x <= (int64_t)nx - 2;
    for (int k = 0; k < nblk; ++k) {
        ring.wait_full(k);
        const double* T = ring.stage(k);
        double o[RYT];
        double cp = T[(RYT * wy) * BX + col], c = T[(RYT * wy + 1) * BX + col];
#pragma unroll
        for (int j = 0; j < RYT; ++j) {
            const int r = RYT * wy + j + 1;
            const double cn = T[(r + 1) * BX + col];
            double a = w0 * c;
            a = fma(w1, cp, a);
            a = fma(w2, cn, a);
            a = fma(w3, T[r * BX + cl], a);
            a = fma(w4, T[r * BX + col + 1], a);
            o[j] = a;
            cp = c;
            c = cn;
        }
        ring.release(k);
        if (tid == 0 && k + S < nblk) {
            ring.wait_empty(k);
            issue(k + S);
        }
        const uint64_t yr = ya + (uint64_t)k * kTY + RYT * wy;
        if (xin) {
#pragma unroll
            for (int j = 0; j < RYT; ++j)
                if (yr + j < yb) v[(yr + j) * nx + x] = o[j];
        }
    }
}

// ===========================================================================
// CUDA core, 3D.  KIND 0: 3d7pt (c, z-, z+, y-, y+, x-, x+); 1: 3d27pt
// general; 2: 3d27pt class weights g0..g3 in w[0..3].
// ===========================================================================
template <int KIND, int S, int RYT>
__global__ void __launch_bounds__(64 * kTY / RYT) st3d_tma_cc(const __grid_constant__ CUtensorMap tm,
                                                   double* __restrict__ v, StencilDesc d, uint64_t z_begin,
                                                   uint64_t z_end, int zchunk, int tiles_x, int tiles_xy) {
    constexpr int BX = kBX, STAGE = stage_doubles(BX);
    extern __shared__ __align__(128) double smem[];
    Ring<S, STAGE> ring(smem);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wx = warp & 1, wy = warp >> 1;
    const int tile = blockIdx.x % tiles_xy;
    const uint64_t za = z_begin + (uint64_t)(blockIdx.x / tiles_xy) * zchunk;
    if (za >= z_end) return;
    const uint64_t zb = min(za + (uint64_t)zchunk, z_end);
    const int np = (int)(zb - za) + 2;  // planes za-1 .. zb
    const int64_t x0 = (int64_t)(tile % tiles_x) * kTX;
    const uint64_t nty = (uint64_t)(tiles_xy / tiles_x), ty = (uint64_t)(tile / tiles_x);
    const int64_t y0 = (int64_t)(ty * d.ny / nty), yhi = (int64_t)((ty + 1) * d.ny / nty);  // rows [y0, yhi)
    const uint64_t nx = d.nx, ny = d.ny;
    const int64_t xs = x0 - kCofs;
    const int cofs = kCofs, rofs = 1;  // stage column/row of (x0, y0); boxes may start OOB
    ring.init(2 * kTY / RYT);
    auto issue = [&](int k) {
        mbar_expect_tx(ring.full + (k % S), kBY * BX * 8);
        tma3d(ring.stage(k), &tm, ring.full + (k % S), (int)xs, (int)(y0 - rofs), (int)(za - 1 + k));
    };
    if (tid == 0)
        for (int k = 0; k < S && k < np; ++k) issue(k);
    const int col = 32 * wx + lane + cofs;
    const int cl = col > 0 ? col - 1 : 0;
    const int rbase = RYT * wy + rofs;  // stage row of this thread's first output row
    const int64_t x = x0 + 32 * wx + lane;
    const bool xin = x >= 1 && x <= (int64_t)nx - 2;
    const int64_t yr0 = y0 + RYT * wy;
    double acc_a[RYT], acc_b[RYT];
#pragma unroll
    for (int j = 0; j < RYT; ++j) acc_a[j] = acc_b[j] = 0.0;
    const double* w = d.w;
    for (int k = 0; k < np; ++k) {
        ring.wait_full(k);
        const double* T = ring.stage(k);
        double pm[RYT], p0[RYT], pp[RYT];
        if (KIND == 0) {
            // rows rbase-1 .. rbase+RYT; rbase-1 < 0 only at y0 == 0, where
            // output row 0 is boundary and never stored
            double cp = T[max(rbase - 1, 0) * BX + col], c = T[rbase * BX + col];
#pragma unroll
            for (int j = 0; j < RYT; ++j) {
                const int r = rbase + j;
                const double cn = T[(r + 1) * BX + col];
                double a = w[0] * c;
                a = fma(w[3], cp, a);
                a = fma(w[4], cn, a);
                a = fma(w[5], T[r * BX + cl], a);
                a = fma(w[6], T[r * BX + col + 1], a);
                p0[j] = a;
                pm[j] = w[1] * c;  // u(p) is the z-1 neighbour of plane p+1
                pp[j] = w[2] * c;  // ... and the z+1 neighbour of plane p-1
                cp = c;
                c = cn;
            }
        } else {
            // rolling 3x3 window: A = row above, B = centre row, C = row below
            const double* ra = T + max(rbase - 1, 0) * BX;
            const double* rb0 = T + rbase * BX;
            double al = ra[cl], ac = ra[col], ar = ra[col + 1];
            double bl = rb0[cl], bc = rb0[col], br = rb0[col + 1];
#pragma unroll
            for (int j = 0; j < RYT; ++j) {
                const double* rc = T + (rbase + j + 1) * BX;
                const double cL = rc[cl], cc = rc[col], cr = rc[col + 1];
                if (KIND == 2) {
                    const double s0 = bc;
                    const double s1 = (ac + cc) + (bl + br);
                    const double s2 = (al + ar) + (cL + cr);
                    p0[j] = fma(w[2], s2, fma(w[1], s1, w[0] * s0));
                    pm[j] = fma(w[3], s2, fma(w[2], s1, w[1] * s0));
                    pp[j] = pm[j];
                } else {
                    const double nb[9] = {al, ac, ar, bl, bc, br, cL, cc, cr};
                    double a = 0.0, b = 0.0, c = 0.0;
#pragma unroll
                    for (int q = 0; q < 9; ++q) {
                        a = fma(w[q], nb[q], a);        // dz = -1 weights -> output p+1
                        b = fma(w[9 + q], nb[q], b);    // dz =  0
                        c = fma(w[18 + q], nb[q], c);   // dz = +1 weights -> output p-1
                    }
                    pm[j] = a;
                    p0[j] = b;
                    pp[j] = c;
                }
                al = bl; ac = bc; ar = br;
                bl = cL; bc = cc; br = cr;
            }
        }
        ring.release(k);
        if (tid == 0 && k + S < np) {
            ring.wait_empty(k);
            issue(k + S);
        }
        double o[RYT];
#pragma unroll
        for (int j = 0; j < RYT; ++j) {
            o[j] = acc_a[j] + pp[j];
            acc_a[j] = acc_b[j] + p0[j];
            acc_b[j] = pm[j];
        }
        if (k >= 2 && xin) {
            const uint64_t p = za - 2 + (uint64_t)k;
#pragma unroll
            for (int j = 0; j < RYT; ++j) {
                const int64_t y = yr0 + j;
                if (y >= 1 && y <= (int64_t)ny - 2 && y < yhi) v[(p * ny + (uint64_t)y) * nx + x] = o[j];
            }
        }
    }
}

// ===========================================================================
// CUDA core, 3d27pt with class weights, two columns per thread.  A warp owns
// the tile's 64 columns (lane: columns 2 lane, 2 lane + 1) and RYT rows; each
// staged row is read as three 128-bit pairs (columns 2 lane - 1 .. 2 lane + 2
// of the tile plus alignment), and the vertical sums u[y-1] + u[y+1] of the
// four columns are shared between the two outputs' face and corner classes:
// 10 DADD + 12 DFMA/DMUL per two points per plane, half the shared loads of
// the one-column kernel.  Partial sums across planes as in st3d_tma_cc.
// ===========================================================================
template <int S, int RYT>
__global__ void __launch_bounds__(32 * kTY / RYT) st3d_tma_cc27x2(const __grid_constant__ CUtensorMap tm,
                                                         double* __restrict__ v, StencilDesc d,
                                                         uint64_t z_begin, uint64_t z_end, int zchunk,
                                                         int tiles_x, int tiles_xy) {
    constexpr int BX = kBX, STAGE = stage_doubles(BX);
    extern __shared__ __align__(128) double smem[];
    Ring<S, STAGE> ring(smem);
    const int tid = threadIdx.x, lane = tid & 31, wy = tid >> 5;
    const int tile = blockIdx.x % tiles_xy;
    const uint64_t za = z_begin + (uint64_t)(blockIdx.x / tiles_xy) * zchunk;
    if (za >= z_end) return;
    const uint64_t zb = min(za + (uint64_t)zchunk, z_end);
    const int np = (int)(zb - za) + 2;  // planes za-1 .. zb
    const int64_t x0 = (int64_t)(tile % tiles_x) * kTX;
    const uint64_t nty = (uint64_t)(tiles_xy / tiles_x), ty = (uint64_t)(tile / tiles_x);
    const int64_t y0 = (int64_t)(ty * d.ny / nty), yhi = (int64_t)((ty + 1) * d.ny / nty);  // rows [y0, yhi)
    const uint64_t nx = d.nx, ny = d.ny;
    ring.init(kTY / RYT);
    auto issue = [&](int k) {
        mbar_expect_tx(ring.full + (k % S), kBY * BX * 8);
        tma3d(ring.stage(k), &tm, ring.full + (k % S), (int)(x0 - kCofs), (int)(y0 - 1), (int)(za - 1 + k));
    };
    if (tid == 0)
        for (int k = 0; k < S && k < np; ++k) issue(k);
    const double g0 = d.w[0], g1 = d.w[1], g2 = d.w[2], g3 = d.w[3];
    const int cb = 2 * lane;            // stage column of the pair (cb, cb+1) = x0 - 2 + cb
    const int rbase = RYT * wy + 1;     // stage row of this warp's first output row
    const int64_t x = x0 + 2 * lane;    // output columns x (stage cb + 2) and x + 1
    const bool in0 = x >= 1 && x <= (int64_t)nx - 2, in1 = x + 1 >= 1 && x + 1 <= (int64_t)nx - 2;
    const int64_t yr0 = y0 + RYT * wy;
    double acc_a[RYT][2], acc_b[RYT][2];
#pragma unroll
    for (int j = 0; j < RYT; ++j) acc_a[j][0] = acc_a[j][1] = acc_b[j][0] = acc_b[j][1] = 0.0;
    // row loader: columns cb+1 .. cb+4 of stage row r (x - 1 .. x + 2)
    auto row4 = [&](const double* T, int r, double (&q)[4]) {
        const double2 lo = *reinterpret_cast<const double2*>(T + r * BX + cb);
        const double2 mid = *reinterpret_cast<const double2*>(T + r * BX + cb + 2);
        const double2 hi = *reinterpret_cast<const double2*>(T + r * BX + cb + 4);
        q[0] = lo.y;
        q[1] = mid.x;
        q[2] = mid.y;
        q[3] = hi.x;
    };
    // warps whose rows all lie past the tile (13-14-row balanced tiles) only
    // keep the ring protocol (warp 0, the producer's, always has rows)
    const bool live = yr0 < yhi;
    for (int k = 0; k < np; ++k) {
        ring.wait_full(k);
        if (!live) {
            ring.release(k);
            continue;
        }
        const double* T = ring.stage(k);
        double pm[RYT][2], p0[RYT][2];
        double up[4], md[4];
        row4(T, rbase - 1, up);
        row4(T, rbase, md);
#pragma unroll
        for (int j = 0; j < RYT; ++j) {
            double dn[4];
            row4(T, rbase + j + 1, dn);
            double vs[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) vs[q] = up[q] + dn[q];
            // column A = q 1, column B = q 2
            const double s1a = vs[1] + (md[0] + md[2]), s2a = vs[0] + vs[2];
            const double s1b = vs[2] + (md[1] + md[3]), s2b = vs[1] + vs[3];
            p0[j][0] = fma(g2, s2a, fma(g1, s1a, g0 * md[1]));
            p0[j][1] = fma(g2, s2b, fma(g1, s1b, g0 * md[2]));
            pm[j][0] = fma(g3, s2a, fma(g2, s1a, g1 * md[1]));
            pm[j][1] = fma(g3, s2b, fma(g2, s1b, g1 * md[2]));
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                up[q] = md[q];
                md[q] = dn[q];
            }
        }
        ring.release(k);
        if (tid == 0 && k + S < np) {
            ring.wait_empty(k);
            issue(k + S);
        }
        double o[RYT][2];
#pragma unroll
        for (int j = 0; j < RYT; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                o[j][h] = acc_a[j][h] + pm[j][h];  // P_+1 of plane p == P_-1 (class symmetry)
                acc_a[j][h] = acc_b[j][h] + p0[j][h];
                acc_b[j][h] = pm[j][h];
            }
        if (k >= 2) {
            const uint64_t p = za - 2 + (uint64_t)k;
#pragma unroll
            for (int j = 0; j < RYT; ++j) {
                const int64_t y = yr0 + j;
                if (y >= 1 && y <= (int64_t)ny - 2 && y < yhi) {
                    double* dst = v + (p * ny + (uint64_t)y) * nx + x;
                    if (in0 && in1)
                        asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(dst), "d"(o[j][0]), "d"(o[j][1])
                                     : "memory");
                    else {
                        if (in0) dst[0] = o[j][0];
                        if (in1) dst[1] = o[j][1];
                    }
                }
            }
        }
    }
}

// ===========================================================================
// Tensor core, 2d5pt: 16 8x8 tiles per stage; warp w -> row block w>>1,
// column blocks 4*(w&1) .. +3.
// ===========================================================================
template <int S>
__global__ void __launch_bounds__(128) st2d_tma_tc(const __grid_constant__ CUtensorMap tm,
                                                   double* __restrict__ v, uint64_t nx, uint64_t y_begin,
                                                   uint64_t y_end, int seg_rows, int strips, StencilDesc d) {
    constexpr int BX = kBX, STAGE = stage_doubles(BX);
    extern __shared__ __align__(128) double smem[];
    Ring<S, STAGE> ring(smem);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int r = lane >> 2, c = lane & 3;
    const int rb = warp >> 1, cb0 = 4 * (warp & 1);
    const int64_t x0 = (int64_t)(blockIdx.x % strips) * kTX;
    const uint64_t ya = y_begin + (uint64_t)(blockIdx.x / strips) * seg_rows;
    if (ya >= y_end) return;
    const uint64_t yb = min(ya + (uint64_t)seg_rows, y_end);
    const int nblk = (int)((yb - ya + kTY - 1) / kTY);
    const int64_t xs = x0 - kCofs;
    const int cofs = kCofs;
    ring.init(4);
    auto issue = [&](int k) {
        mbar_expect_tx(ring.full + (k % S), kBY * BX * 8);
        tma2d(ring.stage(k), &tm, ring.full + (k % S), (int)xs, (int)(ya + (uint64_t)k * kTY) - 1);
    };
    auto cc = [&](int i) { return min(max(i, 0), BX - 1); };  // clamp a stage column
    if (tid == 0)
        for (int k = 0; k < S && k < nblk; ++k) issue(k);
    double ty[3], tx[3];
#pragma unroll
    for (int kb = 0; kb < 3; ++kb) {
        ty[kb] = bandv(4 * kb + c, r, d.w[1], d.w[0], d.w[2]);
        tx[kb] = bandv(4 * kb + c, r, d.w[3], 0.0, d.w[4]);
    }
    for (int k = 0; k < nblk; ++k) {
        ring.wait_full(k);
        const double* T = ring.stage(k);
        double D0[4], D1[4];
        double carry = 0.0;  // k-step 2 operand of tile cb == k-step 0 operand of tile cb+1
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int cb = cb0 + t;
            double d0 = 0.0, d1 = 0.0;
#pragma unroll
            for (int kb = 0; kb < 3; ++kb) {
                const int j = min(4 * kb + c, 9);
                dmma_m8n8k4(d0, d1, ty[kb], T[(8 * rb + j) * BX + cc(8 * cb + r + cofs)], d0, d1);
            }
#pragma unroll
            for (int kb = 0; kb < 3; ++kb) {
                double a;
                if (kb == 0 && t > 0) a = carry;
                else a = T[(8 * rb + r + 1) * BX + cc(8 * cb + 4 * kb + c - 1 + cofs)];
                if (kb == 2) carry = a;
                dmma_m8n8k4(d0, d1, a, tx[kb], d0, d1);
            }
            D0[t] = d0;
            D1[t] = d1;
        }
        ring.release(k);
        if (tid == 0 && k + S < nblk) {
            ring.wait_empty(k);
            issue(k + S);
        }
        const uint64_t y = ya + (uint64_t)k * kTY + 8 * rb + r;
        if (y < yb) {
            double* vr = v + y * nx;
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const int64_t xx = x0 + 8 * (cb0 + t) + 2 * c;
                const bool i0 = xx >= 1 && xx <= (int64_t)nx - 2, i1 = xx + 1 <= (int64_t)nx - 2;
                if (i0 && i1)
                    asm volatile("st.global.v2.f64 [%0], {%1,%2};" ::"l"(vr + xx), "d"(D0[t]), "d"(D1[t]) : "memory");
                else {
                    if (i0) vr[xx] = D0[t];
                    if (xx + 1 >= 1 && i1) vr[xx + 1] = D1[t];
                }
            }
        }
    }
}

// ===========================================================================
// Tensor core, 2d5pt, x-band on DMMA (the default 2D TC kernel): the 3D
// st3d_tma_tch scheme in 2D -- D = U . band(w_x-, 0, w_x+) + C with
// C = w_c u + w_y- u[y-1] + w_y+ u[y+1] formed by DFMA at the accumulator
// positions: 3 DMMA per 8x8 tile instead of the 6 of st2d_tma_tc, fragment
// rows permuted (frag_row) for conflict-free 128-bit accumulator loads.
// ===========================================================================
__device__ __forceinline__ int frag_row2(int m) { return (m & 4) | ((m & 1) << 1) | ((m >> 1) & 1); }

template <int S>
__global__ void __launch_bounds__(128) st2d_tma_tch(const __grid_constant__ CUtensorMap tm,
                                                    double* __restrict__ v, uint64_t nx, uint64_t y_begin,
                                                    uint64_t y_end, int seg_rows, int strips, StencilDesc d) {
    constexpr int BX = kBX, STAGE = stage_doubles(BX);
    extern __shared__ __align__(128) double smem[];
    Ring<S, STAGE> ring(smem);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int r = lane >> 2, c = lane & 3;
    const int rb = warp >> 1, cb0 = 4 * (warp & 1);
    const int64_t x0 = (int64_t)(blockIdx.x % strips) * kTX;
    const uint64_t ya = y_begin + (uint64_t)(blockIdx.x / strips) * seg_rows;
    if (ya >= y_end) return;
    const uint64_t yb = min(ya + (uint64_t)seg_rows, y_end);
    const int nblk = (int)((yb - ya + kTY - 1) / kTY);
    ring.init(4);
    auto issue = [&](int k) {
        mbar_expect_tx(ring.full + (k % S), kBY * BX * 8);
        tma2d(ring.stage(k), &tm, ring.full + (k % S), (int)(x0 - kCofs), (int)(ya + (uint64_t)k * kTY) - 1);
    };
    if (tid == 0)
        for (int k = 0; k < S && k < nblk; ++k) issue(k);
    double bx[3];
#pragma unroll
    for (int kb = 0; kb < 3; ++kb) bx[kb] = bandv(4 * kb + c, r, d.w[3], 0.0, d.w[4]);
    const double w0 = d.w[0], w1 = d.w[1], w2 = d.w[2];
    const int fr = frag_row2(r), pr = 8 * rb + fr + 1;
    for (int k = 0; k < nblk; ++k) {
        ring.wait_full(k);
        const double* Pc = ring.stage(k) + pr * BX;
        double a[9];
#pragma unroll
        for (int i = 0; i < 9; ++i) a[i] = Pc[min(8 * cb0 + 4 * i + c + 1, BX - 1)];
        double D0[4], D1[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int dc = 8 * (cb0 + t) + 2 * c + kCofs;
            const double2 ct = *reinterpret_cast<const double2*>(Pc + dc);
            const double2 up = *reinterpret_cast<const double2*>(Pc - BX + dc);
            const double2 dn = *reinterpret_cast<const double2*>(Pc + BX + dc);
            double d0 = fma(w2, dn.x, fma(w1, up.x, w0 * ct.x));
            double d1 = fma(w2, dn.y, fma(w1, up.y, w0 * ct.y));
#pragma unroll
            for (int kb = 0; kb < 3; ++kb) dmma_m8n8k4(d0, d1, a[2 * t + kb], bx[kb], d0, d1);
            D0[t] = d0;
            D1[t] = d1;
        }
        ring.release(k);
        if (tid == 0 && k + S < nblk) {
            ring.wait_empty(k);
            issue(k + S);
        }
        const uint64_t y = ya + (uint64_t)k * kTY + 8 * rb + fr;
        if (y < yb) {
            double* vr = v + y * nx;
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const int64_t xx = x0 + 8 * (cb0 + t) + 2 * c;
                const bool i0 = xx >= 1 && xx <= (int64_t)nx - 2, i1 = xx + 1 <= (int64_t)nx - 2;
                if (i0 && i1)
                    asm volatile("st.global.v2.f64 [%0], {%1,%2};" ::"l"(vr + xx), "d"(D0[t]), "d"(D1[t]) : "memory");
                else {
                    if (i0) vr[xx] = D0[t];
                    if (i1) vr[xx + 1] = D1[t];
                }
            }
        }
    }
}

// ===========================================================================
// Tensor core, 3D: planes z-1, z, z+1 resident (S >= 5).
// KIND 0: 3d7pt, 1: 3d27pt class weights, 2: 3d27pt general.
// ===========================================================================
template <int KIND, int S>
__global__ void __launch_bounds__(128) st3d_tma_tc(const __grid_constant__ CUtensorMap tm,
                                                   double* __restrict__ v, StencilDesc d, uint64_t z_begin,
                                                   uint64_t z_end, int zchunk, int tiles_x, int tiles_xy) {
    constexpr int BX = kBX, STAGE = stage_doubles(BX);
    extern __shared__ __align__(128) double smem[];
    Ring<S, STAGE> ring(smem);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int r = lane >> 2, c = lane & 3;
    const int rb = warp >> 1, cb0 = 4 * (warp & 1);
    const int tile = blockIdx.x % tiles_xy;
    const uint64_t za = z_begin + (uint64_t)(blockIdx.x / tiles_xy) * zchunk;
    if (za >= z_end) return;
    const uint64_t zb = min(za + (uint64_t)zchunk, z_end);
    const int np = (int)(zb - za) + 2;
    const int64_t x0 = (int64_t)(tile % tiles_x) * kTX, y0 = (int64_t)(tile / tiles_x) * kTY;
    const uint64_t nx = d.nx, ny = d.ny;
    const int64_t xs = x0 - kCofs;
    const int cofs = kCofs;
    ring.init(4);
    auto issue = [&](int k) {
        mbar_expect_tx(ring.full + (k % S), kBY * BX * 8);
        tma3d(ring.stage(k), &tm, ring.full + (k % S), (int)xs, (int)(y0 - 1), (int)(za - 1 + k));
    };
    // stage index of (row y0-1+j, column x0-1+i), column clamped into the box
    auto at = [&](int j, int i) { return j * BX + min(max(i - 1 + cofs, 0), BX - 1); };
    if (tid == 0)
        for (int k = 0; k < S && k < np; ++k) issue(k);

    double fa[3], fb[3], fc[3];
#pragma unroll
    for (int kb = 0; kb < 3; ++kb) {
        const int kk = 4 * kb + c;
        if (KIND == 0) {
            fa[kb] = bandv(kk, r, d.w[3], d.w[0], d.w[4]);
            fb[kb] = bandv(kk, r, d.w[5], 0.0, d.w[6]);
            fc[kb] = 0.0;
        } else {
            fa[kb] = bandv(kk, r, d.w[1], d.w[0], d.w[1]);
            fb[kb] = bandv(kk, r, d.w[2], d.w[1], d.w[2]);
            fc[kb] = bandv(kk, r, d.w[3], d.w[2], d.w[3]);
        }
    }
    double gen[KIND == 2 ? 27 : 1];
    if (KIND == 2) {
#pragma unroll
        for (int q = 0; q < 9; ++q)
#pragma unroll
            for (int kb = 0; kb < 3; ++kb)
                gen[q * 3 + kb] = bandv(4 * kb + c, r, d.w[q * 3 + 0], d.w[q * 3 + 1], d.w[q * 3 + 2]);
    }

    const int64_t yo = y0 + 8 * rb + r;
    const bool row_ok = yo >= 1 && yo <= (int64_t)ny - 2;
    for (int i = 0; i + 2 < np; ++i) {  // output plane za + i uses items i, i+1, i+2
        if (i == 0) {
            ring.wait_full(0);
            ring.wait_full(1);
        }
        ring.wait_full(i + 2);
        const double* Pm = ring.stage(i);
        const double* P0 = ring.stage(i + 1);
        const double* Pp = ring.stage(i + 2);
        // Horizontal-product A operands: lane (r, c) of k-step kb reads window
        // column 8*cb + 4*kb + c (band rows 10/11 are zero, so the unclamped
        // columns are harmless) -- k-step 2 of tile cb is k-step 0 of tile
        // cb+1, so those operands are carried over instead of reloaded.
        double D0[4], D1[4];
        double ca0 = 0.0, ca1 = 0.0, ca2 = 0.0;           // carried (KIND 0/1)
        double cg[9];                                      // carried (KIND 2)
#pragma unroll
        for (int q = 0; q < 9; ++q) cg[q] = 0.0;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int cb = cb0 + t;
            double d0 = 0.0, d1 = 0.0;
            if (KIND == 0) {
                const int s = at(8 * rb + r + 1, 8 * cb + 2 * c + 1);
                d0 = fma(d.w[2], Pp[s], d.w[1] * Pm[s]);
                d1 = fma(d.w[2], Pp[s + 1], d.w[1] * Pm[s + 1]);
#pragma unroll
                for (int kb = 0; kb < 3; ++kb) {
                    const int j = min(4 * kb + c, 9);
                    dmma_m8n8k4(d0, d1, fa[kb], P0[at(8 * rb + j, 8 * cb + r + 1)], d0, d1);
                }
#pragma unroll
                for (int kb = 0; kb < 3; ++kb) {
                    double a;
                    if (kb == 0 && t > 0) a = ca0;
                    else a = P0[at(8 * rb + r + 1, 8 * cb + 4 * kb + c)];
                    if (kb == 2) ca0 = a;
                    dmma_m8n8k4(d0, d1, a, fb[kb], d0, d1);
                }
            } else if (KIND == 1) {
#pragma unroll
                for (int kb = 0; kb < 3; ++kb) {
                    double a0, a1, a2;
                    if (kb == 0 && t > 0) {
                        a0 = ca0; a1 = ca1; a2 = ca2;
                    } else {
                        const int colj = 8 * cb + 4 * kb + c;
                        const int up = at(8 * rb + r, colj), mid = at(8 * rb + r + 1, colj),
                                  dn = at(8 * rb + r + 2, colj);
                        a0 = P0[mid];
                        a1 = (P0[up] + P0[dn]) + (Pm[mid] + Pp[mid]);
                        a2 = (Pm[up] + Pm[dn]) + (Pp[up] + Pp[dn]);
                    }
                    if (kb == 2) { ca0 = a0; ca1 = a1; ca2 = a2; }
                    dmma_m8n8k4(d0, d1, a0, fa[kb], d0, d1);
                    dmma_m8n8k4(d0, d1, a1, fb[kb], d0, d1);
                    dmma_m8n8k4(d0, d1, a2, fc[kb], d0, d1);
                }
            } else {
#pragma unroll
                for (int kb = 0; kb < 3; ++kb) {
                    double g[9];
                    if (kb == 0 && t > 0) {
#pragma unroll
                        for (int q = 0; q < 9; ++q) g[q] = cg[q];
                    } else {
                        const int colj = 8 * cb + 4 * kb + c;
#pragma unroll
                        for (int dz = 0; dz < 3; ++dz) {
                            const double* P = dz == 0 ? Pm : (dz == 1 ? P0 : Pp);
#pragma unroll
                            for (int dy = 0; dy < 3; ++dy) g[dz * 3 + dy] = P[at(8 * rb + r + dy, colj)];
                        }
                    }
                    if (kb == 2) {
#pragma unroll
                        for (int q = 0; q < 9; ++q) cg[q] = g[q];
                    }
#pragma unroll
                    for (int q = 0; q < 9; ++q) dmma_m8n8k4(d0, d1, g[q], gen[q * 3 + kb], d0, d1);
                }
            }
            D0[t] = d0;
            D1[t] = d1;
        }
        ring.release(i);
        if (tid == 0 && i + S < np) {
            ring.wait_empty(i);
            issue(i + S);
        }
        if (row_ok) {
            const uint64_t z = za + (uint64_t)i;
            double* vr = v + (z * ny + (uint64_t)yo) * nx;
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const int64_t xx = x0 + 8 * (cb0 + t) + 2 * c;
                const bool i0 = xx >= 1 && xx <= (int64_t)nx - 2, i1 = xx + 1 <= (int64_t)nx - 2;
                if (i0 && i1)
                    asm volatile("st.global.v2.f64 [%0], {%1,%2};" ::"l"(vr + xx), "d"(D0[t]), "d"(D1[t]) : "memory");
                else {
                    if (i0) vr[xx] = D0[t];
                    if (xx + 1 >= 1 && i1) vr[xx + 1] = D1[t];
                }
            }
        }
    }
}

// ===========================================================================
// Tensor core, 3D, one plane at a time (partial sums, like the CUDA-core 3D
// kernel): plane p contributes P_-1(p) to output p+1, P_0(p) to p and P_+1(p)
// to p-1, accumulated in D-fragment registers.
//   KIND 0 (3d7pt): P_0 = in-plane banded products (6 DMMA), P_-1/P_+1 =
//     w_z-/w_z+ times the centre values at the accumulator positions.
//   KIND 1 (3d27pt class weights): with a = U[y] and b = U[y-1] + U[y+1],
//     P_0 = a*band(g1,g0,g1) + b*band(g2,g1,g2) and
//     P_+-1 = a*band(g2,g1,g2) + b*band(g3,g2,g3)                 12 DMMA
//   KIND 2 (general 27pt): P_dz = sum_dy U[y+dy]*band(w[dz][dy])    27 DMMA
// Only one stage is live, so shared-memory operand traffic is 3x lower than
// the 3-plane formulation for 27pt, at the price of more DMMA.
// ===========================================================================
template <int KIND, int S>
__global__ void __launch_bounds__(128) st3d_tma_tc1(const __grid_constant__ CUtensorMap tm,
                                                    double* __restrict__ v, StencilDesc d, uint64_t z_begin,
                                                    uint64_t z_end, int zchunk, int tiles_x, int tiles_xy) {
    constexpr int BX = kBX, STAGE = stage_doubles(BX);
    extern __shared__ __align__(128) double smem[];
    Ring<S, STAGE> ring(smem);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int r = lane >> 2, c = lane & 3;
    const int rb = warp >> 1, cb0 = 4 * (warp & 1);
    const int tile = blockIdx.x % tiles_xy;
    const uint64_t za = z_begin + (uint64_t)(blockIdx.x / tiles_xy) * zchunk;
    if (za >= z_end) return;
    const uint64_t zb = min(za + (uint64_t)zchunk, z_end);
    const int np = (int)(zb - za) + 2;
    const int64_t x0 = (int64_t)(tile % tiles_x) * kTX, y0 = (int64_t)(tile / tiles_x) * kTY;
    const uint64_t nx = d.nx, ny = d.ny;
    ring.init(4);
    auto issue = [&](int k) {
        mbar_expect_tx(ring.full + (k % S), kBY * BX * 8);
        tma3d(ring.stage(k), &tm, ring.full + (k % S), (int)(x0 - kCofs), (int)(y0 - 1), (int)(za - 1 + k));
    };
    if (tid == 0)
        for (int k = 0; k < S && k < np; ++k) issue(k);
    auto at = [&](int j, int i) { return j * BX + min(max(i - 1 + kCofs, 0), BX - 1); };

    // band fragments (B operand of the horizontal products, A of the vertical one)
    double f0[3], f1[3], f2[3];
#pragma unroll
    for (int kb = 0; kb < 3; ++kb) {
        const int kk = 4 * kb + c;
        if (KIND == 0) {
            f0[kb] = bandv(kk, r, d.w[3], d.w[0], d.w[4]);  // Ty (vertical, with centre)
            f1[kb] = bandv(kk, r, d.w[5], 0.0, d.w[6]);     // Tx
            f2[kb] = 0.0;
        } else {
            f0[kb] = bandv(kk, r, d.w[1], d.w[0], d.w[1]);  // g1 g0 g1
            f1[kb] = bandv(kk, r, d.w[2], d.w[1], d.w[2]);  // g2 g1 g2
            f2[kb] = bandv(kk, r, d.w[3], d.w[2], d.w[3]);  // g3 g2 g3
        }
    }
    // KIND 3: the class products concatenated along K (K = 10 + 10 -> 5
    // k-steps): P_0 = [a | b] * [B(g1,g0,g1); B(g2,g1,g2)] and
    // P_+-1 = [a | b] * [B(g2,g1,g2); B(g3,g2,g3)], 10 DMMA per tile, not 12
    double h0[KIND == 3 ? 5 : 1], h1[KIND == 3 ? 5 : 1];
    if (KIND == 3) {
#pragma unroll
        for (int s5 = 0; s5 < 5; ++s5) {
            const int kk = 4 * s5 + c;
            h0[s5] = kk < 10 ? bandv(kk, r, d.w[1], d.w[0], d.w[1]) : bandv(kk - 10, r, d.w[2], d.w[1], d.w[2]);
            h1[s5] = kk < 10 ? bandv(kk, r, d.w[2], d.w[1], d.w[2]) : bandv(kk - 10, r, d.w[3], d.w[2], d.w[3]);
        }
    }
    double gen[KIND == 2 ? 27 : 1];
    if (KIND == 2) {
#pragma unroll
        for (int q = 0; q < 9; ++q)
#pragma unroll
            for (int kb = 0; kb < 3; ++kb)
                gen[q * 3 + kb] = bandv(4 * kb + c, r, d.w[q * 3 + 0], d.w[q * 3 + 1], d.w[q * 3 + 2]);
    }

    double acc_a[4][2], acc_b[4][2];
#pragma unroll
    for (int t = 0; t < 4; ++t) acc_a[t][0] = acc_a[t][1] = acc_b[t][0] = acc_b[t][1] = 0.0;
    const int64_t yo = y0 + 8 * rb + r;
    const bool row_ok = yo >= 1 && yo <= (int64_t)ny - 2;
    for (int k = 0; k < np; ++k) {
        ring.wait_full(k);
        const double* P = ring.stage(k);
        double pm[4][2], p0[4][2], pp[4][2];
        double ca = 0.0, cbp = 0.0;  // operands carried from k-step 2 to the next tile's k-step 0
        double cg[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int cb = cb0 + t;
            if (KIND == 0) {
                double d0 = 0.0, d1 = 0.0;
#pragma unroll
                for (int kb = 0; kb < 3; ++kb) {
                    const int j = min(4 * kb + c, 9);
                    dmma_m8n8k4(d0, d1, f0[kb], P[at(8 * rb + j, 8 * cb + r + 1)], d0, d1);
                }
#pragma unroll
                for (int kb = 0; kb < 3; ++kb) {
                    double a;
                    if (kb == 0 && t > 0) a = ca;
                    else a = P[at(8 * rb + r + 1, 8 * cb + 4 * kb + c)];
                    if (kb == 2) ca = a;
                    dmma_m8n8k4(d0, d1, a, f1[kb], d0, d1);
                }
                const int s = at(8 * rb + r + 1, 8 * cb + 2 * c + 1);
                const double z0 = P[s], z1 = P[s + 1];
                p0[t][0] = d0; p0[t][1] = d1;
                pm[t][0] = d.w[1] * z0; pm[t][1] = d.w[1] * z1;
                pp[t][0] = d.w[2] * z0; pp[t][1] = d.w[2] * z1;
            } else if (KIND == 3) {
                double e0 = 0.0, e1 = 0.0, g0 = 0.0, g1 = 0.0;
#pragma unroll
                for (int s5 = 0; s5 < 5; ++s5) {
                    const int kk = 4 * s5 + c;
                    double av;
                    if (kk < 10) {
                        av = P[at(8 * rb + r + 1, 8 * cb + kk)];
                    } else {
                        const int k2 = kk - 10;
                        av = P[at(8 * rb + r, 8 * cb + k2)] + P[at(8 * rb + r + 2, 8 * cb + k2)];
                    }
                    dmma_m8n8k4(e0, e1, av, h0[s5], e0, e1);  // P_0
                    dmma_m8n8k4(g0, g1, av, h1[s5], g0, g1);  // P_+-1
                }
                p0[t][0] = e0; p0[t][1] = e1;
                pm[t][0] = pp[t][0] = g0; pm[t][1] = pp[t][1] = g1;
            } else if (KIND == 1) {
                double e0 = 0.0, e1 = 0.0, g0 = 0.0, g1 = 0.0;
#pragma unroll
                for (int kb = 0; kb < 3; ++kb) {
                    double a, b;
                    if (kb == 0 && t > 0) {
                        a = ca; b = cbp;
                    } else {
                        const int colj = 8 * cb + 4 * kb + c;
                        a = P[at(8 * rb + r + 1, colj)];
                        b = P[at(8 * rb + r, colj)] + P[at(8 * rb + r + 2, colj)];
                    }
                    if (kb == 2) { ca = a; cbp = b; }
                    dmma_m8n8k4(e0, e1, a, f0[kb], e0, e1);  // P_0
                    dmma_m8n8k4(e0, e1, b, f1[kb], e0, e1);
                    dmma_m8n8k4(g0, g1, a, f1[kb], g0, g1);  // P_+-1
                    dmma_m8n8k4(g0, g1, b, f2[kb], g0, g1);
                }
                p0[t][0] = e0; p0[t][1] = e1;
                pm[t][0] = pp[t][0] = g0; pm[t][1] = pp[t][1] = g1;
            } else {
                double m0 = 0.0, m1 = 0.0, e0 = 0.0, e1 = 0.0, q0 = 0.0, q1 = 0.0;
#pragma unroll
                for (int kb = 0; kb < 3; ++kb) {
                    double g[3];
                    if (kb == 0 && t > 0) {
                        g[0] = cg[0]; g[1] = cg[1]; g[2] = cg[2];
                    } else {
                        const int colj = 8 * cb + 4 * kb + c;
#pragma unroll
                        for (int dy = 0; dy < 3; ++dy) g[dy] = P[at(8 * rb + r + dy, colj)];
                    }
                    if (kb == 2) { cg[0] = g[0]; cg[1] = g[1]; cg[2] = g[2]; }
#pragma unroll
                    for (int dy = 0; dy < 3; ++dy) {
                        dmma_m8n8k4(m0, m1, g[dy], gen[(0 * 3 + dy) * 3 + kb], m0, m1);  // dz = -1
                        dmma_m8n8k4(e0, e1, g[dy], gen[(1 * 3 + dy) * 3 + kb], e0, e1);  // dz =  0
                        dmma_m8n8k4(q0, q1, g[dy], gen[(2 * 3 + dy) * 3 + kb], q0, q1);  // dz = +1
                    }
                }
                pm[t][0] = m0; pm[t][1] = m1;
                p0[t][0] = e0; p0[t][1] = e1;
                pp[t][0] = q0; pp[t][1] = q1;
            }
        }
        ring.release(k);
        if (tid == 0 && k + S < np) {
            ring.wait_empty(k);
            issue(k + S);
        }
        double o[4][2];
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                o[t][h] = acc_a[t][h] + pp[t][h];
                acc_a[t][h] = acc_b[t][h] + p0[t][h];
                acc_b[t][h] = pm[t][h];
            }
        if (k >= 2 && row_ok) {
            const uint64_t z = za - 2 + (uint64_t)k;
            double* vr = v + (z * ny + (uint64_t)yo) * nx;
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const int64_t xx = x0 + 8 * (cb0 + t) + 2 * c;
                const bool i0 = xx >= 1 && xx <= (int64_t)nx - 2, i1 = xx + 1 <= (int64_t)nx - 2;
                if (i0 && i1)
                    asm volatile("st.global.v2.f64 [%0], {%1,%2};" ::"l"(vr + xx), "d"(o[t][0]), "d"(o[t][1]) : "memory");
                else {
                    if (i0) vr[xx] = o[t][0];
                    if (i1) vr[xx + 1] = o[t][1];
                }
            }
        }
    }
}

// ===========================================================================
// Tensor core, 3D, x-band on DMMA with the rest on DFMA (the default 3D TC
// kernel).  DMMA and DFMA share one FP64 datapath on B200 (tools/micro/
// fp64_pipes.cu: 36.3 TF/s DFMA alone, 37.1 DMMA alone, <= 34.5 combined),
// and a banded 8x8 product spends 12 k-slots on 3 taps, so every tap moved to
// the DMMA costs 4 slots of the shared datapath; sustained runs also hit
// sw_power_cap sooner the more DMMA they issue.  This kernel keeps exactly
// one banded contraction per output tile on the tensor core -- the x
// direction, 3 DMMA per 8x8 tile -- and feeds everything else in through the
// accumulator C:
//   KIND 0 (3d7pt):  D = U_z . band(w_x-, 0, w_x+) + C,
//                    C = w_c u + w_y- u[y-1] + w_y+ u[y+1] + w_z- u[z-1] + w_z+ u[z+1]
//   KIND 1 (3d27pt, class weights g0..g3): every x-band of the box is
//     band(g(a+1), g(a), g(a+1)) = g(a+1) E + g(a) I with E = band(1, 0, 1),
//     a = |dy| + |dz|, so  out = alpha . E + beta  with the y-z class sums
//     S_a:  alpha = g1 S0 + g2 S1 + g3 S2 (A-fragment positions, one DMMA
//     operand per k-slot) and beta = g0 S0 + g1 S1 + g2 S2 (accumulator
//     positions).  Both are accumulated across planes like the CUDA-core
//     partial sums: plane q adds (g1 a + g2 b) to alpha(q) and (g2 a + g3 b)
//     to alpha(q +- 1), a = u[y], b = u[y-1] + u[y+1].
// 12 DMMA-FMA + ~5 (7pt) / ~15 (27pt) DFMA per point, against 24 / 40 DMMA-FMA
// in the full banded formulations (st3d_tma_tc / st3d_tma_tc1).
//
// KS = 2 shortens the band product to K = 8 (window columns x0-1 .. x0+6 of
// each 8-column tile): 2 DMMA per tile instead of 3.  The two taps that fall
// outside -- the x+1 taps of output columns 6 and 7 -- are the next tile's
// first two window columns, i.e. A-fragment elements already held by lanes
// c = 0 and 1 of the same row; two shuffles bring them to lane c = 3, whose
// accumulator holds columns 6 and 7, for one DFMA each.
//
// Fragment rows are permuted, MMA row m <-> tile row pi(m) (bits 0 and 1
// swapped), so the accumulator-position 128-bit loads (lane r, c reads
// columns 2c, 2c+1 of row pi(r)) are conflict-free with the 68-double stage
// pitch: a quarter-warp's rows pi(0), pi(1) = 0, 2 land 8 banks apart.
// ===========================================================================
__device__ __forceinline__ int frag_row(int m) { return (m & 4) | ((m & 1) << 1) | ((m >> 1) & 1); }

template <int KIND, int S, int KS, int TPW>
__global__ void __launch_bounds__(512 / TPW) st3d_tma_tch(const __grid_constant__ CUtensorMap tm,
                                                    double* __restrict__ v, StencilDesc d, uint64_t z_begin,
                                                    uint64_t z_end, int zchunk, int tiles_x, int tiles_xy) {
    constexpr int BX = kBX, STAGE = stage_doubles(BX);
    extern __shared__ __align__(128) double smem[];
    Ring<S, STAGE> ring(smem);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int r = lane >> 2, c = lane & 3;
    constexpr int NE = 2 * TPW + 1;         // A-fragment elements per lane (tiles share one)
    const int rb = warp / (8 / TPW), cb0 = TPW * (warp % (8 / TPW));
    const uint64_t nx = d.nx, ny = d.ny;
    const int tile = blockIdx.x % tiles_xy;
    const uint64_t za = z_begin + (uint64_t)(blockIdx.x / tiles_xy) * zchunk;
    if (za >= z_end) return;
    const uint64_t zb = min(za + (uint64_t)zchunk, z_end);
    const int np = (int)(zb - za) + 2;
    const int64_t x0 = (int64_t)(tile % tiles_x) * kTX;
    const uint64_t nty = (uint64_t)(tiles_xy / tiles_x), ty = (uint64_t)(tile / tiles_x);
    const int64_t y0 = (int64_t)(ty * d.ny / nty), yhi = (int64_t)((ty + 1) * d.ny / nty);  // rows [y0, yhi)
    ring.init(16 / TPW);
    auto issue = [&](int k) {
        mbar_expect_tx(ring.full + (k % S), kBY * BX * 8);
        tma3d(ring.stage(k), &tm, ring.full + (k % S), (int)(x0 - kCofs), (int)(y0 - 1), (int)(za - 1 + k));
    };
    if (tid == 0)
        for (int k = 0; k < S && k < np; ++k) issue(k);

    const int pr = 8 * rb + frag_row(r) + 1;  // stage row of this lane's fragment row
    // A-fragment element i (tile t = cb0 + i/2 .. k-step): window column 8 cb0 + 4 i + c,
    // stage column + 1 (window column 0 = x0 - 1 = stage column 1); columns past
    // the box only meet zero band rows (k = 10, 11), so they are clamped.
    auto acol = [&](int i) { return min(8 * cb0 + 4 * i + c + 1, BX - 1); };
    // accumulator pair of tile t: columns x0 + 8 (cb0 + t) + 2c (+1) -> stage column + 2
    auto dcol = [&](int t) { return 8 * (cb0 + t) + 2 * c + kCofs; };

    double bx[3];
#pragma unroll
    for (int kb = 0; kb < 3; ++kb)
        bx[kb] = KIND == 0 ? bandv(4 * kb + c, r, d.w[5], 0.0, d.w[6]) : bandv(4 * kb + c, r, 1.0, 0.0, 1.0);
    // KS = 2: weight of the two x+1 taps past the K = 8 window (lane c = 3 only)
    const double wfix = c == 3 ? (KIND == 0 ? d.w[6] : 1.0) : 0.0;
    const int src8 = lane & ~3, src9 = src8 | 1;

    double acc_a[TPW][2], acc_b[TPW][2];  // accumulator-position partial sums (C operand)
    double al_a[NE], al_b[NE];            // KIND 1: alpha partial sums at the A-fragment positions
#pragma unroll
    for (int t = 0; t < TPW; ++t) acc_a[t][0] = acc_a[t][1] = acc_b[t][0] = acc_b[t][1] = 0.0;
#pragma unroll
    for (int i = 0; i < NE; ++i) al_a[i] = al_b[i] = 0.0;
    const double w0 = d.w[0], w1 = d.w[1], w2 = d.w[2], w3 = d.w[3], w4 = d.w[4];
    const int64_t yo = y0 + 8 * rb + frag_row(r);
    const bool row_ok = yo >= 1 && yo <= (int64_t)ny - 2 && yo < yhi;

    for (int k = 0; k < np; ++k) {
        ring.wait_full(k);
        const double* P = ring.stage(k);
        const double* Pc = P + pr * BX;
        double o[TPW][2];
        if (KIND == 0) {
            // plane k: finishes output k-1 (its z+1 term), forms output k = U.Bx + C,
            // starts output k+1 (its z-1 term)
            double a[NE];
#pragma unroll
            for (int i = 0; i < NE; ++i) a[i] = Pc[acol(i)];
#pragma unroll
            for (int t = 0; t < TPW; ++t) {
                const double2 ct = *reinterpret_cast<const double2*>(Pc + dcol(t));
                const double2 up = *reinterpret_cast<const double2*>(Pc - BX + dcol(t));
                const double2 dn = *reinterpret_cast<const double2*>(Pc + BX + dcol(t));
                o[t][0] = fma(w2, ct.x, acc_a[t][0]);
                o[t][1] = fma(w2, ct.y, acc_a[t][1]);
                double d0 = fma(w4, dn.x, fma(w3, up.x, fma(w0, ct.x, acc_b[t][0])));
                double d1 = fma(w4, dn.y, fma(w3, up.y, fma(w0, ct.y, acc_b[t][1])));
                if (KS == 2) {
                    d0 = fma(wfix, __shfl_sync(0xffffffffu, a[2 * t + 2], src8), d0);
                    d1 = fma(wfix, __shfl_sync(0xffffffffu, a[2 * t + 2], src9), d1);
                }
#pragma unroll
                for (int kb = 0; kb < KS; ++kb) dmma_m8n8k4(d0, d1, a[2 * t + kb], bx[kb], d0, d1);
                acc_a[t][0] = d0;
                acc_a[t][1] = d1;
                acc_b[t][0] = w1 * ct.x;
                acc_b[t][1] = w1 * ct.y;
            }
        } else {
            const double g0 = d.w[0], g1 = d.w[1], g2 = d.w[2], g3 = d.w[3];
            double aout[NE];
#pragma unroll
            for (int i = 0; i < NE; ++i) {
                const int cc = acol(i);
                const double a = Pc[cc], b = Pc[cc - BX] + Pc[cc + BX];
                const double c1 = fma(g3, b, g2 * a);
                aout[i] = al_a[i] + c1;
                al_a[i] = al_b[i] + fma(g2, b, g1 * a);
                al_b[i] = c1;
            }
#pragma unroll
            for (int t = 0; t < TPW; ++t) {
                const double2 ct = *reinterpret_cast<const double2*>(Pc + dcol(t));
                const double2 up = *reinterpret_cast<const double2*>(Pc - BX + dcol(t));
                const double2 dn = *reinterpret_cast<const double2*>(Pc + BX + dcol(t));
                const double b0 = up.x + dn.x, b1 = up.y + dn.y;
                const double e0 = fma(g2, b0, g1 * ct.x), e1 = fma(g2, b1, g1 * ct.y);
                double d0 = acc_a[t][0] + e0, d1 = acc_a[t][1] + e1;
                acc_a[t][0] = acc_b[t][0] + fma(g1, b0, g0 * ct.x);
                acc_a[t][1] = acc_b[t][1] + fma(g1, b1, g0 * ct.y);
                acc_b[t][0] = e0;
                acc_b[t][1] = e1;
                if (k >= 2) {
                    if (KS == 2) {
                        d0 = fma(wfix, __shfl_sync(0xffffffffu, aout[2 * t + 2], src8), d0);
                        d1 = fma(wfix, __shfl_sync(0xffffffffu, aout[2 * t + 2], src9), d1);
                    }
#pragma unroll
                    for (int kb = 0; kb < KS; ++kb) dmma_m8n8k4(d0, d1, aout[2 * t + kb], bx[kb], d0, d1);
                }
                o[t][0] = d0;
                o[t][1] = d1;
            }
        }
        ring.release(k);
        if (tid == 0 && k + S < np) {
            ring.wait_empty(k);
            issue(k + S);
        }
        if (k >= 2 && row_ok) {
            const uint64_t z = za - 2 + (uint64_t)k;
            double* vr = v + (z * ny + (uint64_t)yo) * nx;
#pragma unroll
            for (int t = 0; t < TPW; ++t) {
                const int64_t xx = x0 + 8 * (cb0 + t) + 2 * c;
                const bool i0 = xx >= 1 && xx <= (int64_t)nx - 2, i1 = xx + 1 <= (int64_t)nx - 2;
                if (i0 && i1)
                    asm volatile("st.global.v2.f64 [%0], {%1,%2};" ::"l"(vr + xx), "d"(o[t][0]), "d"(o[t][1]) : "memory");
                else {
                    if (i0) vr[xx] = o[t][0];
                    if (i1) vr[xx + 1] = o[t][1];
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// host: tensor maps
// ---------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

bool make_map(CUtensorMap* m, const double* base, int rank, const uint64_t* dims, uint32_t box_x) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t gdim[3] = {dims[0], dims[1], rank == 3 ? dims[2] : 1};
    cuuint64_t gstride[2] = {dims[0] * 8, dims[0] * dims[1] * 8};
    cuuint32_t box[3] = {box_x, (cuuint32_t)kBY, 1};
    cuuint32_t estride[3] = {1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, (cuuint32_t)rank, const_cast<double*>(base), gdim, gstride,
              box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <class K>
cudaError_t prep(K kernel, size_t smem) {
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

bool class_weights(const double* w, double g[4]) {
    bool seen[4] = {false, false, false, false};
    for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
                const int m = (dz != 0) + (dy != 0) + (dx != 0);
                const double ww = w[(dz + 1) * 9 + (dy + 1) * 3 + (dx + 1)];
                if (!seen[m]) { g[m] = ww; seen[m] = true; }
                else if (g[m] != ww) return false;
            }
    return true;
}

// Split the marched axis so the grid fills about `per_sm` CTAs per SM.  For
// the CUDA-core kernels the measured optimum is one chunk per tile (a full
// march, ~1.7 CTAs/SM at the BASELINE grids); the tensor-core 3D kernels
// need more warps in flight to cover the DMMA chains.
int split_count(uint64_t tiles, uint64_t extent, int min_chunk, int per_sm) {
    const uint64_t slots = (uint64_t)kNumSMs * (uint64_t)per_sm;
    uint64_t n = tiles >= slots ? 1 : slots / tiles;
    const uint64_t cap = (extent + min_chunk - 1) / min_chunk;
    if (n > cap) n = cap;
    if (n < 1) n = 1;
    return (int)n;
}

}  // namespace

bool tma_encode_available() { return encode_fn() != nullptr; }

bool encode_map_2d(void* map, const double* base, uint64_t nx, uint64_t ny, uint32_t box_x, uint32_t box_y,
                   int l2_promotion) {
    static const CUtensorMapL2promotion promo[4] = {CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_64B,
                                                    CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B};
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t gdim[2] = {nx, ny};
    cuuint64_t gstride[1] = {nx * 8};
    cuuint32_t box[2] = {box_x, box_y};
    cuuint32_t estride[2] = {1, 1};
    return fn(static_cast<CUtensorMap*>(map), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), gdim,
              gstride, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
              promo[l2_promotion & 3], CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool encode_map_3d(void* map, const double* base, uint64_t nx, uint64_t ny, uint64_t nz, uint32_t box_x,
                   uint32_t box_y, int l2_promotion) {
    static const CUtensorMapL2promotion promo[4] = {CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_64B,
                                                    CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B};
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t gdim[3] = {nx, ny, nz};
    cuuint64_t gstride[2] = {nx * 8, nx * ny * 8};
    cuuint32_t box[3] = {box_x, box_y, 1};
    cuuint32_t estride[3] = {1, 1, 1};
    return fn(static_cast<CUtensorMap*>(map), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), gdim,
              gstride, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
              promo[l2_promotion & 3], CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool stencil_tma_eligible(const StencilDesc& d, const double* u, const double* v) {
    if (!tuning().stencil_tma) return false;
    if (d.preset != kP2d5 && d.preset != kP3d7 && d.preset != kP3d27) return false;
    if (d.nx % 2 != 0) return false;  // row pitch must be a multiple of 16 bytes
    if ((reinterpret_cast<uintptr_t>(u) & 15) || (reinterpret_cast<uintptr_t>(v) & 15)) return false;
    if (d.nx > (1ull << 31) || d.ny > (1ull << 31) || d.nz > (1ull << 31)) return false;
    return encode_fn() != nullptr;
}

cudaError_t launch_stencil_tma(int unit, const StencilDesc& d, uint64_t o0, uint64_t o1, const double* u,
                               double* v, cudaStream_t s) {
    const uint64_t dims[3] = {d.nx, d.ny, d.nz};
    CUtensorMap m;
    if (!make_map(&m, u, d.dim, dims, kBX)) return cudaErrorInvalidValue;
    cudaError_t e;
    if (d.dim == 2) {
        const int strips = (int)((d.nx + kTX - 1) / kTX);
        const int nseg = split_count(strips, o1 - o0, 64,
                                     unit == 1 ? tuning().stencil_tc_ctas_per_sm : tuning().stencil_ctas_per_sm);
        int seg_rows = (int)(((o1 - o0 + nseg - 1) / nseg + kTY - 1) / kTY * kTY);
        const int segs = (int)((o1 - o0 + seg_rows - 1) / seg_rows);
        const unsigned grid = (unsigned)(strips * segs);
        if (unit == 1) {
            constexpr int S = 4;
            const size_t sm = ring_bytes<S, kBX>();
            if (tuning().stencil_tc2d_hybrid) {
                if ((e = prep(st2d_tma_tch<S>, sm)) != cudaSuccess) return e;
                st2d_tma_tch<S><<<grid, 128, sm, s>>>(m, v, d.nx, o0, o1, seg_rows, strips, d);
            } else {
                if ((e = prep(st2d_tma_tc<S>, sm)) != cudaSuccess) return e;
                st2d_tma_tc<S><<<grid, 128, sm, s>>>(m, v, d.nx, o0, o1, seg_rows, strips, d);
            }
        } else {
            constexpr int S = 4;
            const size_t sm = ring_bytes<S, kBX>();
            const int ry = tuning().stencil2d_rows_per_thread;
#define RLB_CC2(R)                                                                                 \
    do {                                                                                           \
        if ((e = prep(st2d_tma_cc<S, R>, sm)) != cudaSuccess) return e;                           \
        st2d_tma_cc<S, R><<<grid, 64 * kTY / R, sm, s>>>(m, v, d.nx, o0, o1, seg_rows, strips, d); \
    } while (0)
            if (ry == 2) RLB_CC2(2); else if (ry == 4) RLB_CC2(4); else RLB_CC2(8);
#undef RLB_CC2
        }
        note_launch();
        return cudaGetLastError();
    }
    const int tiles_x = (int)((d.nx + kTX - 1) / kTX);
    int tiles_xy = tiles_x * (int)((d.ny + kTY - 1) / kTY);
    StencilDesc dd = d;
    int kind = 0;
    if (d.preset == kP3d27) {
        double g[4];
        if (class_weights(d.w, g)) {
            kind = 2;
            for (int i = 0; i < 4; ++i) dd.w[i] = g[i];
        } else {
            kind = 1;
        }
    }
    const bool tc_hybrid = unit == 1 && kind != 1 && tuning().stencil_tc3d_hybrid;
    const bool tc_onepl = unit == 1 && ((tuning().stencil_tc3d_mode >> (kind == 0 ? 0 : 1)) & 1);
    const int nch = split_count(tiles_xy, o1 - o0, 8,
                                unit == 1 ? (tc_hybrid ? (tuning().stencil_tch_ctas_per_sm
                                                              ? tuning().stencil_tch_ctas_per_sm
                                                              : (kind == 0 ? 1 : 16))
                                             : tc_onepl ? tuning().stencil_tc1_ctas_per_sm
                                                        : tuning().stencil_tc3d_ctas_per_sm)
                                          : tuning().stencil_ctas_per_sm);
    // Row balance (one z-front, nch == 1): 256 tiles of 16 rows on 148 SMs put
    // two tiles on most SMs and one on the rest; instead cut the rows into nty
    // tiles of <= 16 rows (row y0 = ty * ny / nty) so the busiest SM holds the
    // fewest rows -- 512 rows: 37 tiles of 13-14 rows, 296 CTAs = 2 per SM.
    // Kernels that take it: st3d_tma_cc, st3d_tma_cc27x2, st3d_tma_tch.
    const bool balanced_kernel = unit == 0 || tc_hybrid;
    if (balanced_kernel && nch == 1 && tuning().stencil3d_balance) {
        const uint64_t nty0 = (d.ny + kTY - 1) / kTY;
        uint64_t best = nty0, bcost = ~0ull;
        for (uint64_t nty = nty0; nty <= 2 * nty0; ++nty) {
            const uint64_t per_sm = ((uint64_t)tiles_x * nty + kNumSMs - 1) / kNumSMs;
            const uint64_t cost = per_sm * ((d.ny + nty - 1) / nty);
            if (cost < bcost) { bcost = cost; best = nty; }
        }
        tiles_xy = tiles_x * (int)best;
    }
    const int zchunk = (int)((o1 - o0 + nch - 1) / nch);
    const int zch = (int)((o1 - o0 + zchunk - 1) / zchunk);
    const unsigned grid = (unsigned)(tiles_xy * zch);
    if (tc_hybrid) {
#define RLB_TCHS(K, KS, TPW, S)                                                                            \
    do {                                                                                                   \
        const size_t sm = ring_bytes<S, kBX>();                                                            \
        if ((e = prep(st3d_tma_tch<K, S, KS, TPW>, sm)) != cudaSuccess) return e;                         \
        st3d_tma_tch<K, S, KS, TPW><<<grid, 512 / TPW, sm, s>>>(m, v, dd, o0, o1, zchunk, tiles_x, tiles_xy); \
    } while (0)
#define RLB_TCH(K, KS, TPW) \
    do { if (KS == 3 && tuning().stencil_tch_stages == 6) RLB_TCHS(K, 3, TPW, 6); else RLB_TCHS(K, KS, TPW, 4); } while (0)
#define RLB_TCH2(K, TPW) \
    do { if (tuning().stencil_tch_k8) RLB_TCH(K, 2, TPW); else RLB_TCH(K, 3, TPW); } while (0)
#define RLB_TCH3(K) \
    do { const int tp = tuning().stencil_tch_tpw ? tuning().stencil_tch_tpw : (K == 0 ? 2 : 4); if (tp == 4) RLB_TCH2(K, 4); else if (tp == 1) RLB_TCH2(K, 1); else RLB_TCH2(K, 2); } while (0)
        if (kind == 0) RLB_TCH3(0); else RLB_TCH3(1);
#undef RLB_TCH3
#undef RLB_TCH2
#undef RLB_TCH
#undef RLB_TCHS
    } else if (tc_onepl) {
        constexpr int S = 4;
        const size_t sm = ring_bytes<S, kBX>();
        const int tk = kind == 0 ? 0 : (kind == 2 ? (tuning().stencil_tc_concat ? 3 : 1) : 2);
#define RLB_TC1(K)                                                                             \
    do {                                                                                       \
        if ((e = prep(st3d_tma_tc1<K, S>, sm)) != cudaSuccess) return e;                      \
        st3d_tma_tc1<K, S><<<grid, 128, sm, s>>>(m, v, dd, o0, o1, zchunk, tiles_x, tiles_xy); \
    } while (0)
        if (tk == 0) RLB_TC1(0); else if (tk == 1) RLB_TC1(1); else if (tk == 3) RLB_TC1(3); else RLB_TC1(2);
#undef RLB_TC1
    } else if (unit == 1) {
        constexpr int S = 5;
        const size_t sm = ring_bytes<S, kBX>();
        const int tk = kind == 0 ? 0 : (kind == 2 ? 1 : 2);  // TC kinds: 0 7pt, 1 class, 2 general
#define RLB_TC3(K)                                                                            \
    do {                                                                                      \
        if ((e = prep(st3d_tma_tc<K, S>, sm)) != cudaSuccess) return e;                      \
        st3d_tma_tc<K, S><<<grid, 128, sm, s>>>(m, v, dd, o0, o1, zchunk, tiles_x, tiles_xy); \
    } while (0)
        if (tk == 0) RLB_TC3(0); else if (tk == 1) RLB_TC3(1); else RLB_TC3(2);
#undef RLB_TC3
    } else {
        // rows per thread: 0 = the measured default per preset (3d7pt 4: 6.18 vs
        // 5.80-6.01 TB/s at 2; 27pt 2: 5.86 vs 4.79 at 4, tools/sweep.py stencil3d_cc)
        const int ry = tuning().stencil_rows_per_thread ? tuning().stencil_rows_per_thread : (kind == 0 ? 4 : 2);
        const int st = tuning().stencil3d_cc_stages;
#define RLB_CC3(K, R, SS)                                                                                  \
    do {                                                                                                   \
        const size_t sm = ring_bytes<SS, kBX>();                                                           \
        if ((e = prep(st3d_tma_cc<K, SS, R>, sm)) != cudaSuccess) return e;                               \
        st3d_tma_cc<K, SS, R><<<grid, 64 * kTY / R, sm, s>>>(m, v, dd, o0, o1, zchunk, tiles_x, tiles_xy); \
    } while (0)
#define RLB_CC3S(K, R) \
    do { if (st == 6) RLB_CC3(K, R, 6); else if (st == 8) RLB_CC3(K, R, 8); else RLB_CC3(K, R, 4); } while (0)
#define RLB_CC3K(K) \
    do { if (ry == 2) RLB_CC3S(K, 2); else if (ry == 4) RLB_CC3S(K, 4); else RLB_CC3S(K, 8); } while (0)
        if (kind == 2 && tuning().stencil_cc27x2) {
            constexpr int S = 4;
            const size_t sm = ring_bytes<S, kBX>();
#define RLB_CC27(R)                                                                                           \
    do {                                                                                                      \
        if ((e = prep(st3d_tma_cc27x2<S, R>, sm)) != cudaSuccess) return e;                                  \
        st3d_tma_cc27x2<S, R><<<grid, 32 * kTY / R, sm, s>>>(m, v, dd, o0, o1, zchunk, tiles_x, tiles_xy); \
    } while (0)
            if (ry == 4) RLB_CC27(4); else if (ry == 8) RLB_CC27(8); else RLB_CC27(2);
#undef RLB_CC27
        } else if (kind == 0) RLB_CC3K(0); else if (kind == 1) RLB_CC3K(1); else RLB_CC3K(2);
#undef RLB_CC3K
#undef RLB_CC3S
#undef RLB_CC3
    }
    note_launch();
    return cudaGetLastError();
}

}  // namespace rlb
