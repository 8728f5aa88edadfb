// stencil_tb3.cu -- 3d7pt and 3d27pt temporal blocking of depth T (SURVEY.md
// §8f "next" #1 for 3D; stencil_model(shape, P, t),
// kernels.cpp:137-155).  3d7pt runs the register-blocked kernel
// (stencil_tb3r.cu) where it can; this z-column form covers the rest and 3d27pt.
//
// A CTA owns a TX x TY output tile and marches z through a chunk; each thread
// owns one (x, y) column of the loaded (TX + 2T) x (TY + 2T) region.  For
// every input plane the T levels of a skewed pipeline advance by one plane:
// level l keeps a 3-plane z-window of its column in registers, publishes the
// window's middle value to a per-level shared plane, and after one barrier
// reads its four in-plane neighbours from it.  The valid region shrinks by
// one column/row per level, so the inner TX x TY threads store level T.
// HBM sees one read of u and one write of v per T timesteps; the in-plane
// halo of a tile is re-read from L2 by the neighbouring tiles.
//
// Dirichlet points (any coordinate on the grid's first or last index) keep
// their value at every level; loads outside the grid read 0 and only feed
// boundary points or points outside a stored output's dependency cone.
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace rlb {
namespace {

template <int T>
struct Tb3Geom {
    static constexpr int TX = 32;
    static constexpr int TY = T == 2 ? 24 : (T == 3 ? 20 : 16);
    static constexpr int LX = TX + 2 * T, LY = TY + 2 * T;  // loaded region
    static constexpr int NT = LX * LY;                        // threads per CTA
    static_assert(NT <= 1024, "one thread per loaded column");
};

template <int T, int PF>
__global__ void __launch_bounds__(Tb3Geom<T>::NT) st3d7_tb(const double* __restrict__ u, double* __restrict__ v,
                                                           int nx, int ny, int nz, int z_begin, int z_end,
                                                           int zchunk, int tiles_x, int tiles_y,
                                                           const __grid_constant__ StencilDesc d) {
    using G = Tb3Geom<T>;
    __shared__ double plane[T][G::LY][G::LX];  // level l-1's middle plane, published for level l
    const int tid = threadIdx.x;
    const int lx = tid % G::LX, ly = tid / G::LX;
    const int tile = blockIdx.x % (tiles_x * tiles_y);
    const int za = z_begin + (blockIdx.x / (tiles_x * tiles_y)) * zchunk;
    if (za >= z_end) return;
    const int zb = min(za + zchunk, z_end);
    const int x = (tile % tiles_x) * G::TX - T + lx;
    const int y = (tile / tiles_x) * G::TY - T + ly;
    const bool inx = x >= 0 && x < nx, iny = y >= 0 && y < ny;
    const bool bxy = x <= 0 || x >= nx - 1 || y <= 0 || y >= ny - 1;
    const bool inner = lx >= T && lx < T + G::TX && ly >= T && ly < T + G::TY && inx && iny && !bxy;
    const int xl = lx > 0 ? lx - 1 : lx, xr = lx < G::LX - 1 ? lx + 1 : lx;  // edge threads read themselves
    const int yu = ly > 0 ? ly - 1 : ly, yd = ly < G::LY - 1 ? ly + 1 : ly;  // (invalid there anyway)
    const double w0 = d.w[0], wzm = d.w[1], wzp = d.w[2], wym = d.w[3], wyp = d.w[4], wxm = d.w[5], wxp = d.w[6];

    double win[T][3];  // level l z-window: planes r-1, r, r+1
#pragma unroll
    for (int l = 0; l < T; ++l) win[l][0] = win[l][1] = win[l][2] = 0.0;
    const int i0 = za - T, i1 = zb - 1 + T;  // input planes
    const int64_t pstride = (int64_t)nx * ny;
    const bool own = inx && iny;
    // pointers advanced one plane per step (no per-plane 64-bit multiplies)
    const double* pf = u + (own ? (int64_t)y * nx + x : 0) + (int64_t)i0 * pstride;
    double* dst = v + (own ? (int64_t)y * nx + x : 0) + (int64_t)(i0 - T) * pstride;  // plane ii - T
    double q[PF];
#pragma unroll
    for (int j = 0; j < PF; ++j) {
        const int i = i0 + j;
        q[j] = (own && i >= 0 && i < nz) ? __ldg(pf) : 0.0;
        pf += pstride;
    }

    for (int i = i0; i <= i1; i += PF) {
#pragma unroll
        for (int j = 0; j < PF; ++j) {
            const int ii = i + j;
            const double in = q[j];
            q[j] = (own && ii + PF >= 0 && ii + PF < nz) ? __ldg(pf) : 0.0;
            pf += pstride;
            win[0][0] = win[0][1];
            win[0][1] = win[0][2];
            win[0][2] = in;
#pragma unroll
            for (int l = 1; l <= T; ++l) {
                const double c = win[l - 1][1];
                plane[l - 1][ly][lx] = c;
                __syncthreads();
                const int r = ii - l;  // the plane this level produces
                double o = w0 * c;
                o = fma(wzm, win[l - 1][0], o);
                o = fma(wzp, win[l - 1][2], o);
                o = fma(wym, plane[l - 1][yu][lx], o);
                o = fma(wyp, plane[l - 1][yd][lx], o);
                o = fma(wxm, plane[l - 1][ly][xl], o);
                o = fma(wxp, plane[l - 1][ly][xr], o);
                if (bxy || r <= 0 || r >= nz - 1) o = c;  // Dirichlet: keep the value
                if (l < T) {
                    win[l][0] = win[l][1];
                    win[l][1] = win[l][2];
                    win[l][2] = o;
                } else {
                    if (inner && r >= za && r < zb) *dst = o;
                    dst += pstride;
                }
            }
        }
    }
}

// 3d27pt, any weights: per input plane every level publishes its newest
// plane once, reads the 3 x 3 in-plane neighbourhood of its column (9 shared
// loads) and folds it into three partial sums, one per output plane the
// arrival feeds (dz = +1 finishes plane p-1, dz = 0 and dz = -1 start planes
// p and p+1): 9 loads and 27 FMAs per point per level, weights straight from
// the kernel-parameter bank (canonical order, (dz, dy, dx) lexicographic).
template <int T, int PF, bool CLS>
__global__ void __launch_bounds__(Tb3Geom<T>::NT) st3d27_tb(const double* __restrict__ u, double* __restrict__ v,
                                                            int nx, int ny, int nz, int z_begin, int z_end,
                                                            int zchunk, int tiles_x, int tiles_y,
                                                            const __grid_constant__ StencilDesc d) {
    using G = Tb3Geom<T>;
    __shared__ double plane[T][G::LY][G::LX];  // level l-1's newest plane, published for level l
    const int tid = threadIdx.x;
    const int lx = tid % G::LX, ly = tid / G::LX;
    const int tile = blockIdx.x % (tiles_x * tiles_y);
    const int za = z_begin + (blockIdx.x / (tiles_x * tiles_y)) * zchunk;
    if (za >= z_end) return;
    const int zb = min(za + zchunk, z_end);
    const int x = (tile % tiles_x) * G::TX - T + lx;
    const int y = (tile / tiles_x) * G::TY - T + ly;
    const bool inx = x >= 0 && x < nx, iny = y >= 0 && y < ny;
    const bool bxy = x <= 0 || x >= nx - 1 || y <= 0 || y >= ny - 1;
    const bool inner = lx >= T && lx < T + G::TX && ly >= T && ly < T + G::TY && inx && iny && !bxy;
    const int xl = lx > 0 ? lx - 1 : lx, xr = lx < G::LX - 1 ? lx + 1 : lx;  // edge threads read themselves
    const int yu = ly > 0 ? ly - 1 : ly, yd = ly < G::LY - 1 ? ly + 1 : ly;  // (invalid there anyway)

    // level l state: A = the plane waiting for its dz = +1 term, B = the plane
    // after it (dz = -1 term only), pv = the centre value of A's plane
    double A[T], B[T], pv[T];
#pragma unroll
    for (int l = 0; l < T; ++l) A[l] = B[l] = pv[l] = 0.0;
    const int i0 = za - T, i1 = zb - 1 + T;  // input planes (level l emits plane ii - l)
    const int64_t pstride = (int64_t)nx * ny;
    const bool own = inx && iny;
    const double* pf = u + (own ? (int64_t)y * nx + x : 0) + (int64_t)i0 * pstride;
    double* dst = v + (own ? (int64_t)y * nx + x : 0) + (int64_t)(i0 - T) * pstride;  // plane ii - T
    double q[PF];
#pragma unroll
    for (int j = 0; j < PF; ++j) {
        const int i = i0 + j;
        q[j] = (own && i >= 0 && i < nz) ? __ldg(pf) : 0.0;
        pf += pstride;
    }
    for (int i = i0; i <= i1; i += PF) {
#pragma unroll
        for (int j = 0; j < PF; ++j) {
            const int ii = i + j;
            double a = q[j];  // level 0's arrival: input plane ii
            q[j] = (own && ii + PF >= 0 && ii + PF < nz) ? __ldg(pf) : 0.0;
            pf += pstride;
#pragma unroll
            for (int l = 1; l <= T; ++l) {
                // level l receives plane p = ii - l + 1 of level l-1 and emits plane p - 1
                plane[l - 1][ly][lx] = a;
                __syncthreads();
                double nb[3][3];
#pragma unroll
                for (int dy = 0; dy < 3; ++dy) {
                    const int yy = dy == 0 ? yu : (dy == 1 ? ly : yd);
                    nb[dy][0] = plane[l - 1][yy][xl];
                    nb[dy][1] = plane[l - 1][yy][lx];
                    nb[dy][2] = plane[l - 1][yy][xr];
                }
                double pp = 0.0, p0 = 0.0, pm = 0.0;  // dz = +1, 0, -1 contributions of the arrival
                if (CLS) {
                    // class weights g(|dx| + |dy| + |dz|): edge and corner sums once,
                    // and the dz = +1 and dz = -1 contributions coincide
                    const double E = (nb[0][1] + nb[2][1]) + (nb[1][0] + nb[1][2]);
                    const double K = (nb[0][0] + nb[0][2]) + (nb[2][0] + nb[2][2]);
                    const double g0 = d.w[13], g1 = d.w[12], g2 = d.w[9], g3 = d.w[0];
                    pp = fma(g3, K, fma(g2, E, g1 * nb[1][1]));
                    pm = pp;
                    p0 = fma(g2, K, fma(g1, E, g0 * nb[1][1]));
                } else {
#pragma unroll
                    for (int dy = 0; dy < 3; ++dy)
#pragma unroll
                        for (int dx = 0; dx < 3; ++dx) {
                            pp = fma(d.w[18 + 3 * dy + dx], nb[dy][dx], pp);
                            p0 = fma(d.w[9 + 3 * dy + dx], nb[dy][dx], p0);
                            pm = fma(d.w[3 * dy + dx], nb[dy][dx], pm);
                        }
                }
                const int r = ii - l;  // the plane this level finishes
                double o = A[l - 1] + pp;
                if (bxy || r <= 0 || r >= nz - 1) o = pv[l - 1];  // Dirichlet: keep the value
                A[l - 1] = B[l - 1] + p0;
                B[l - 1] = pm;
                pv[l - 1] = a;
                a = o;
                if (l == T) {
                    if (inner && r >= za && r < zb) *dst = o;
                    dst += pstride;
                }
            }
        }
    }
}

// Weights that depend only on |dx| + |dy| + |dz| (the BASELINE 27pt form).
bool class_weights_27(const StencilDesc& d) {
    const double g[4] = {d.w[13], d.w[12], d.w[9], d.w[0]};
    for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx)
                if (d.w[(dz + 1) * 9 + (dy + 1) * 3 + (dx + 1)] != g[std::abs(dx) + std::abs(dy) + std::abs(dz)])
                    return false;
    return true;
}

template <int T>
cudaError_t launch_tb3(const StencilDesc& d, uint64_t o0, uint64_t o1, const double* u, double* v,
                       cudaStream_t s) {
    using G = Tb3Geom<T>;
    const int tiles_x = (int)((d.nx + G::TX - 1) / G::TX), tiles_y = (int)((d.ny + G::TY - 1) / G::TY);
    const int tiles = tiles_x * tiles_y;
    const int planes = (int)(o1 - o0);
    // z chunks: ~tuning().stencil_tb_waves waves of one CTA per SM, chunks >= 8 T planes
    int nch = (int)(((uint64_t)kNumSMs * (uint64_t)tuning().stencil_tb_waves + tiles - 1) / tiles);
    nch = std::max(1, std::min(nch, std::max(1, planes / (8 * T))));
    const int zchunk = (planes + nch - 1) / nch;
    const int zch = (planes + zchunk - 1) / zchunk;
    if (d.preset == kP3d27 && class_weights_27(d))
        st3d27_tb<T, 4, true><<<(unsigned)(tiles * zch), G::NT, 0, s>>>(u, v, (int)d.nx, (int)d.ny, (int)d.nz,
                                                                          (int)o0, (int)o1, zchunk, tiles_x, tiles_y, d);
    else if (d.preset == kP3d27)
        st3d27_tb<T, 4, false><<<(unsigned)(tiles * zch), G::NT, 0, s>>>(u, v, (int)d.nx, (int)d.ny, (int)d.nz,
                                                                           (int)o0, (int)o1, zchunk, tiles_x, tiles_y, d);
    else
        st3d7_tb<T, 6><<<(unsigned)(tiles * zch), G::NT, 0, s>>>(u, v, (int)d.nx, (int)d.ny, (int)d.nz, (int)o0,
                                                                   (int)o1, zchunk, tiles_x, tiles_y, d);
    note_launch();
    return cudaGetLastError();
}

}  // namespace

bool stencil_tb3_supported(const StencilDesc& d, int t) {
    return (d.preset == kP3d7 || d.preset == kP3d27) && t >= 2 && t <= 4 && d.nx < (1u << 30) &&
           d.ny < (1u << 30) && d.nz < (1u << 30);
}

cudaError_t launch_stencil_tb3(const StencilDesc& d, int t, uint64_t o0, uint64_t o1, const double* u, double* v,
                               cudaStream_t s) {
    if (!stencil_tb3_supported(d, t)) return cudaErrorInvalidValue;
    switch (t) {
        case 2: return launch_tb3<2>(d, o0, o1, u, v, s);
        case 3: return launch_tb3<3>(d, o0, o1, u, v, s);
        default: return launch_tb3<4>(d, o0, o1, u, v, s);
    }
}

}  // namespace rlb
