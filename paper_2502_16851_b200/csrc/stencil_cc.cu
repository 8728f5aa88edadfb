// stencil_cc.cu -- K5/K7/K9: CUDA-core Jacobi stencils.
//
// Algorithmic bytes: 16 B per updated point per step (one load of u, one
// store of v; stencil_model, reference kernels.cpp:137-155).  Every kernel
// here reads each u value from HBM once per sweep (halo re-reads are L2 hits
// of neighbouring tiles) and writes each v value once.
//
//  2d5pt (K5): register streaming along y.  A warp owns a 128-column strip
//      (4 doubles per lane, 256-bit loads) of H rows; u rows y-1, y, y+1 live
//      in registers with a D-deep prefetch queue; x neighbours come from the
//      adjacent lanes by shuffle, the strip's two edge columns by scalar loads.
//  3d7pt / 3d27pt (K7/K9): 2.5D blocking.  A 256-thread CTA owns a 128 x TY
//      xy tile and marches z through a chunk of planes.  Each plane tile
//      (with its 1-cell halo) is staged in a double-buffered shared-memory
//      buffer (one __syncthreads per plane); the next planes are prefetched
//      into registers with 256-bit loads.  7pt keeps u(z-1), u(z), u(z+1) of
//      its own points in registers.  27pt accumulates per-plane partial sums
//      P_dz(p) = sum_{dy,dx} w[dz][dy][dx] u(p, y+dy, x+dx) into the outputs of
//      planes p+1, p, p-1 as plane p passes, so only one plane is staged; when
//      the weights depend only on |dx|+|dy|+|dz| (BASELINE.json's 27pt) each
//      plane contributes through 3 class sums (centre, 4 edges, 4 corners)
//      instead of 27 products.
//  Anything else (other presets, x rows not 32-byte aligned) takes the
//  generic one-thread-per-point kernel.
#include "common.cuh"
#include "kernels.h"

namespace rlb {
namespace {

// ---------------------------------------------------------------------------
// Generic kernel: any preset, any layout.
// ---------------------------------------------------------------------------
struct Offsets {
    int n;
    int64_t d[49];
};

__global__ void stencil_generic(const double* __restrict__ u, double* __restrict__ v,
                                StencilDesc desc, Offsets off, uint64_t o0, uint64_t o1) {
    const uint64_t nx = desc.nx, ny = desc.ny;
    const int r = desc.radius;
    const uint64_t inner_x = nx - 2 * r;
    const uint64_t per_o = desc.dim == 2 ? inner_x : inner_x * (ny - 2 * r);
    const uint64_t total = (o1 - o0) * per_o;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += stride) {
        const uint64_t o = o0 + t / per_o;
        const uint64_t rem = t % per_o;
        const uint64_t x = r + rem % inner_x;
        uint64_t p;
        if (desc.dim == 2) {
            p = o * nx + x;
        } else {
            const uint64_t y = r + rem / inner_x;
            p = (o * ny + y) * nx + x;
        }
        double acc = 0.0;
        for (int s = 0; s < off.n; ++s) acc = fma(desc.w[s], __ldg(u + p + off.d[s]), acc);
        v[p] = acc;
    }
}

// ---------------------------------------------------------------------------
// 2d5pt, register streaming.  Weights in canonical order:
// w0 centre, w1 (y-1), w2 (y+1), w3 (x-1), w4 (x+1).
// ---------------------------------------------------------------------------
struct Row4 {
    d4 v;
    double h;  // lane 0: u[y][c0-1]; lane 31: u[y][c0+4]
};

__device__ __forceinline__ Row4 load_row4(const double* __restrict__ u, uint64_t nx, uint64_t y,
                                          int64_t c0, int lane, uint64_t pol) {
    Row4 r;
    const double* row = u + y * nx;
    r.v = ld4_stream(row + c0, pol);
    r.h = 0.0;
    if (lane == 0 && c0 >= 1) r.h = ld_cached(row + c0 - 1);
    if (lane == 31 && c0 + 4 < (int64_t)nx) r.h = ld_cached(row + c0 + 4);
    return r;
}

template <int D>
__global__ void __launch_bounds__(128) st2d5_cc(const double* __restrict__ u,
                                                double* __restrict__ v, uint64_t nx,
                                                uint64_t y_begin, uint64_t y_end, int H,
                                                uint64_t strips, double w0, double w1,
                                                double w2, double w3, double w4) {
    const int lane = threadIdx.x & 31;
    const uint64_t wid = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t strip = wid % strips, seg = wid / strips;
    const uint64_t ya = y_begin + seg * (uint64_t)H;
    if (ya >= y_end) return;  // warp-uniform
    const uint64_t yb = min(ya + (uint64_t)H, y_end);
    const int64_t c0 = (int64_t)strip * 128 + 4 * lane;
    const bool active = c0 < (int64_t)nx;  // nx % 4 == 0 here
    const int64_t cl = active ? c0 : 0;    // inactive lanes read column 0 harmlessly
    const uint64_t pol = policy_evict_first();

    Row4 up = load_row4(u, nx, ya - 1, cl, lane, pol);
    Row4 cur = load_row4(u, nx, ya, cl, lane, pol);
    Row4 q[D];
#pragma unroll
    for (int k = 0; k < D; ++k)
        if (ya + 1 + k <= yb) q[k] = load_row4(u, nx, ya + 1 + k, cl, lane, pol);

    const bool full = active && c0 >= 1 && c0 + 4 <= (int64_t)nx - 1;
    for (uint64_t y = ya; y < yb; y += D) {
#pragma unroll
        for (int k = 0; k < D; ++k) {
            if (y + k < yb) {
                const Row4 dn = q[k];
                const uint64_t yn = y + k + 1 + D;
                if (yn <= yb) q[k] = load_row4(u, nx, yn, cl, lane, pol);
                // x neighbours: lane-1's last / lane+1's first element, edges from halo.
                double lft = __shfl_up_sync(0xffffffffu, cur.v.w, 1);
                double rgt = __shfl_down_sync(0xffffffffu, cur.v.x, 1);
                if (lane == 0) lft = cur.h;
                if (lane == 31) rgt = cur.h;
                d4 o;
                o.x = w0 * cur.v.x; o.x = fma(w1, up.v.x, o.x); o.x = fma(w2, dn.v.x, o.x);
                o.x = fma(w3, lft, o.x); o.x = fma(w4, cur.v.y, o.x);
                o.y = w0 * cur.v.y; o.y = fma(w1, up.v.y, o.y); o.y = fma(w2, dn.v.y, o.y);
                o.y = fma(w3, cur.v.x, o.y); o.y = fma(w4, cur.v.z, o.y);
                o.z = w0 * cur.v.z; o.z = fma(w1, up.v.z, o.z); o.z = fma(w2, dn.v.z, o.z);
                o.z = fma(w3, cur.v.y, o.z); o.z = fma(w4, cur.v.w, o.z);
                o.w = w0 * cur.v.w; o.w = fma(w1, up.v.w, o.w); o.w = fma(w2, dn.v.w, o.w);
                o.w = fma(w3, cur.v.z, o.w); o.w = fma(w4, rgt, o.w);
                double* out = v + (y + k) * nx + c0;
                if (full) {
                    st4_stream(out, o, pol);
                } else if (active) {
                    const double ov[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        if (c0 + e >= 1 && c0 + e <= (int64_t)nx - 2) out[e] = ov[e];
                }
                up = cur;
                cur = dn;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// 3D, 2.5D blocking with a shared-memory plane tile.
// ---------------------------------------------------------------------------
constexpr int TX = 128;

struct Plane4 {
    d4 own;    // u(p, y, x0+4L .. +3)
    d4 ext;    // ty==0: row y0-1;  ty==TY-1: row y0+TY
    double h;  // lane 0: (y, x0-1); lane 31: (y, x0+TX)
    double hc; // corners: ty==0 / ty==TY-1, lanes 0/31
};

template <int TY>
__device__ __forceinline__ Plane4 load_plane4(const double* __restrict__ u, uint64_t nx,
                                              uint64_t ny, uint64_t p, int64_t x0, int64_t y0,
                                              int lane, int ty, uint64_t pol) {
    Plane4 r;
    const double* pl = u + p * nx * ny;
    const int64_t xl = x0 + 4 * lane;
    const bool xin = xl < (int64_t)nx;
    const int64_t y = y0 + ty;
    const bool yin = y < (int64_t)ny;
    const d4 z{0.0, 0.0, 0.0, 0.0};
    r.own = (xin && yin) ? ld4_stream(pl + y * nx + xl, pol) : z;
    r.ext = z;
    if (ty == 0 && y0 >= 1 && xin) r.ext = ld4_cached(pl + (y0 - 1) * nx + xl);
    if (ty == TY - 1 && y0 + TY < (int64_t)ny && xin) r.ext = ld4_cached(pl + (y0 + TY) * nx + xl);
    r.h = 0.0;
    r.hc = 0.0;
    const int64_t hx = lane == 0 ? x0 - 1 : x0 + TX;
    const bool hxin = (lane == 0 || lane == 31) && hx >= 0 && hx < (int64_t)nx;
    if (hxin && yin) r.h = ld_cached(pl + y * nx + hx);
    if (hxin && ty == 0 && y0 >= 1) r.hc = ld_cached(pl + (y0 - 1) * nx + hx);
    if (hxin && ty == TY - 1 && y0 + TY < (int64_t)ny) r.hc = ld_cached(pl + (y0 + TY) * nx + hx);
    return r;
}

// tile layout: [TY+2][TX+2], tile[j][i] = u(y0-1+j, x0-1+i)
template <int TY>
__device__ __forceinline__ void stage_plane(double* tile, const Plane4& pl, int lane, int ty) {
    constexpr int W = TX + 2;
    double* row = tile + (ty + 1) * W + 1 + 4 * lane;
    row[0] = pl.own.x; row[1] = pl.own.y; row[2] = pl.own.z; row[3] = pl.own.w;
    if (ty == 0) {
        double* e = tile + 1 + 4 * lane;
        e[0] = pl.ext.x; e[1] = pl.ext.y; e[2] = pl.ext.z; e[3] = pl.ext.w;
    }
    if (ty == TY - 1) {
        double* e = tile + (TY + 1) * W + 1 + 4 * lane;
        e[0] = pl.ext.x; e[1] = pl.ext.y; e[2] = pl.ext.z; e[3] = pl.ext.w;
    }
    if (lane == 0) tile[(ty + 1) * W] = pl.h;
    if (lane == 31) tile[(ty + 1) * W + TX + 1] = pl.h;
    if (ty == 0 && lane == 0) tile[0] = pl.hc;
    if (ty == 0 && lane == 31) tile[TX + 1] = pl.hc;
    if (ty == TY - 1 && lane == 0) tile[(TY + 1) * W] = pl.hc;
    if (ty == TY - 1 && lane == 31) tile[(TY + 1) * W + TX + 1] = pl.hc;
}

// Read the 3 x 6 neighbourhood of this thread's 4 points from the tile:
// nb[j][i] = u(y-1+j, xl-1+i).
template <int TY>
__device__ __forceinline__ void read_nb(const double* tile, int lane, int ty, double (&nb)[3][6]) {
    constexpr int W = TX + 2;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        const double* r = tile + (ty + j) * W + 4 * lane;
#pragma unroll
        for (int i = 0; i < 6; ++i) nb[j][i] = r[i];
    }
}

__device__ __forceinline__ void store_out4(double* __restrict__ v, uint64_t nx, uint64_t ny,
                                           uint64_t p, int64_t xl, int64_t y, const double (&o)[4],
                                           uint64_t pol) {
    if (y < 1 || y > (int64_t)ny - 2 || xl >= (int64_t)nx) return;
    double* dst = v + (p * ny + (uint64_t)y) * nx + xl;
    if (xl >= 1 && xl + 4 <= (int64_t)nx - 1) {
        st4_stream(dst, d4{o[0], o[1], o[2], o[3]}, pol);
    } else {
#pragma unroll
        for (int e = 0; e < 4; ++e)
            if (xl + e >= 1 && xl + e <= (int64_t)nx - 2) dst[e] = o[e];
    }
}

// KIND 0: 3d7pt (w: centre, z-1, z+1, y-1, y+1, x-1, x+1)
// KIND 1: 3d27pt general weights (w[(dz+1)*9 + (dy+1)*3 + (dx+1)])
// KIND 2: 3d27pt class weights g[m], m = |dx|+|dy|+|dz| (passed in w[0..3])
template <int KIND, int TY, int D>
__global__ void __launch_bounds__(32 * TY) st3d_cc(const double* __restrict__ u,
                                                   double* __restrict__ v, StencilDesc desc,
                                                   uint64_t z_begin, uint64_t z_end, int zchunk,
                                                   uint64_t tiles_x) {
    __shared__ double tiles[2][(TY + 2) * (TX + 2)];
    const int lane = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const uint64_t nx = desc.nx, ny = desc.ny;
    const uint64_t tile = blockIdx.x;
    const int64_t x0 = (int64_t)(tile % tiles_x) * TX;
    const int64_t y0 = (int64_t)(tile / tiles_x) * TY;
    const uint64_t za = z_begin + (uint64_t)blockIdx.y * (uint64_t)zchunk;
    if (za >= z_end) return;
    const uint64_t zb = min(za + (uint64_t)zchunk, z_end);
    const int64_t xl = x0 + 4 * lane, y = y0 + ty;
    const uint64_t pol = policy_evict_first();
    const double* w = desc.w;

    // Planes needed: za-1 .. zb.  q[k] holds plane (next + k).
    Plane4 q[D];
    uint64_t next = za - 1;
#pragma unroll
    for (int k = 0; k < D; ++k)
        if (next + k <= zb) q[k] = load_plane4<TY>(u, nx, ny, next + k, x0, y0, lane, ty, pol);

    d4 prev{0, 0, 0, 0}, cur{0, 0, 0, 0};  // 7pt: own u at planes p-1, p
    double acc_a[4] = {0, 0, 0, 0}, acc_b[4] = {0, 0, 0, 0};  // 27pt partial outputs
    int buf = 0;
    for (uint64_t p0 = za - 1; p0 <= zb; p0 += D) {
#pragma unroll
        for (int k = 0; k < D; ++k) {
            const uint64_t p = p0 + k;
            if (p <= zb) {
                const Plane4 pl = q[k];
                if (p + D <= zb) q[k] = load_plane4<TY>(u, nx, ny, p + D, x0, y0, lane, ty, pol);
                double* t = tiles[buf];
                stage_plane<TY>(t, pl, lane, ty);
                __syncthreads();
                double nb[3][6];
                read_nb<TY>(t, lane, ty, nb);
                if (KIND == 1 || KIND == 2) {
                    double Pm[4], P0[4], Pp[4];  // P_{-1}, P_0, P_{+1} of plane p
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        if (KIND == 2) {
                            const double s0 = nb[1][e + 1];
                            const double s1 = (nb[0][e + 1] + nb[2][e + 1]) + (nb[1][e] + nb[1][e + 2]);
                            const double s2 = (nb[0][e] + nb[0][e + 2]) + (nb[2][e] + nb[2][e + 2]);
                            P0[e] = fma(w[2], s2, fma(w[1], s1, w[0] * s0));
                            Pm[e] = fma(w[3], s2, fma(w[2], s1, w[1] * s0));
                            Pp[e] = Pm[e];
                        } else {
                            double a = 0.0, b = 0.0, c = 0.0;
#pragma unroll
                            for (int dy = 0; dy < 3; ++dy)
#pragma unroll
                                for (int dx = 0; dx < 3; ++dx) {
                                    const double uu = nb[dy][e + dx];
                                    a = fma(w[0 * 9 + dy * 3 + dx], uu, a);
                                    b = fma(w[1 * 9 + dy * 3 + dx], uu, b);
                                    c = fma(w[2 * 9 + dy * 3 + dx], uu, c);
                                }
                            Pm[e] = a;  // dz = -1 weights: contributes to output p+1
                            P0[e] = b;
                            Pp[e] = c;  // dz = +1 weights: contributes to output p-1
                        }
                    }
                    // out(p-1) = acc_a + P_{+1}(p); acc_a <- acc_b + P_0(p); acc_b <- P_{-1}(p)
                    double o[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        o[e] = acc_a[e] + Pp[e];
                        acc_a[e] = acc_b[e] + P0[e];
                        acc_b[e] = Pm[e];
                    }
                    if (p >= za + 1) store_out4(v, nx, ny, p - 1, xl, y, o, pol);
                } else {
                    // 7pt: out(p-1) = w0*u(p-1) + w1*u(p-2) + w2*u(p) + in-plane(p-1).
                    // We hold the in-plane sum of plane p-1 in acc_a (computed last
                    // iteration), prev = u(p-2), cur = u(p-1).
                    double o[4];
                    const double pv[4] = {prev.x, prev.y, prev.z, prev.w};
                    const double nx4[4] = {pl.own.x, pl.own.y, pl.own.z, pl.own.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        double a = fma(w[1], pv[e], acc_a[e]);
                        o[e] = fma(w[2], nx4[e], a);
                        // in-plane part of plane p for the next output (p)
                        double ip = w[0] * nb[1][e + 1];
                        ip = fma(w[3], nb[0][e + 1], ip);
                        ip = fma(w[4], nb[2][e + 1], ip);
                        ip = fma(w[5], nb[1][e], ip);
                        ip = fma(w[6], nb[1][e + 2], ip);
                        acc_a[e] = ip;
                    }
                    if (p >= za + 1) store_out4(v, nx, ny, p - 1, xl, y, o, pol);
                    prev = cur;
                    cur = pl.own;
                }
                buf ^= 1;
            }
        }
    }
}

bool is_class_symmetric_27(const double* w, double g[4]) {
    for (int m = 0; m < 4; ++m) g[m] = 0.0;
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

}  // namespace

// Offsets of the generic kernel, canonical order (matches oracle/oracle.c).
static Offsets make_offsets(const StencilDesc& d) {
    Offsets o{};
    const int64_t sy = (int64_t)d.nx, sz = (int64_t)(d.nx * d.ny);
    auto add = [&](int dz, int dy, int dx) { o.d[o.n++] = dz * sz + dy * sy + dx; };
    switch (d.preset) {
        case kP2d5: add(0, 0, 0); add(0, -1, 0); add(0, 1, 0); add(0, 0, -1); add(0, 0, 1); break;
        case kP3d7:
            add(0, 0, 0); add(-1, 0, 0); add(1, 0, 0); add(0, -1, 0); add(0, 1, 0);
            add(0, 0, -1); add(0, 0, 1);
            break;
        case kP2d9: case kP2d49: {
            const int r = d.preset == kP2d9 ? 1 : 3;
            for (int dy = -r; dy <= r; ++dy)
                for (int dx = -r; dx <= r; ++dx) add(0, dy, dx);
            break;
        }
        case kP2d13:
            add(0, 0, 0);
            for (int k = 1; k <= 3; ++k) { add(0, -k, 0); add(0, k, 0); add(0, 0, -k); add(0, 0, k); }
            break;
        case kP3d27:
            for (int dz = -1; dz <= 1; ++dz)
                for (int dy = -1; dy <= 1; ++dy)
                    for (int dx = -1; dx <= 1; ++dx) add(dz, dy, dx);
            break;
    }
    return o;
}

cudaError_t launch_stencil_generic(const StencilDesc& d, uint64_t o0, uint64_t o1,
                                   const double* u, double* v, cudaStream_t s) {
    const Offsets off = make_offsets(d);
    const int threads = 256;
    uint64_t blocks = (uint64_t)kNumSMs * 16;
    stencil_generic<<<(unsigned)blocks, threads, 0, s>>>(u, v, d, off, o0, o1); note_launch();
    return cudaGetLastError();
}

cudaError_t launch_stencil_cc(const StencilDesc& d, uint64_t o0, uint64_t o1, const double* u,
                              double* v, cudaStream_t s) {
    if (stencil_tma_eligible(d, u, v)) return launch_stencil_tma(0, d, o0, o1, u, v, s);
    if (tuning().stencil_tma && stencil_r_eligible(d, u, v)) return launch_stencil_r(0, d, o0, o1, u, v, s);
    const Tuning& t = tuning();
    const bool vec_ok = (d.nx % 4 == 0) && aligned32(u) && aligned32(v);
    if (d.preset == kP2d5 && vec_ok) {
        const int H = t.stencil2d_rows > 0 ? t.stencil2d_rows : 256;
        const uint64_t strips = (d.nx + 127) / 128;
        const uint64_t segs = (o1 - o0 + H - 1) / H;
        const uint64_t warps = strips * segs;
        const uint64_t blocks = (warps + 3) / 4;
        st2d5_cc<4><<<(unsigned)blocks, 128, 0, s>>>(u, v, d.nx, o0, o1, H, strips, d.w[0],
                                                    d.w[1], d.w[2], d.w[3], d.w[4]); note_launch();
        return cudaGetLastError();
    }
    if ((d.preset == kP3d7 || d.preset == kP3d27) && vec_ok) {
        constexpr int TY = 8;
        const int Z = t.stencil3d_zchunk > 0 ? t.stencil3d_zchunk : 64;
        const uint64_t tiles_x = (d.nx + TX - 1) / TX;
        const uint64_t tiles_y = (d.ny + TY - 1) / TY;
        const uint64_t zch = (o1 - o0 + Z - 1) / Z;
        dim3 grid((unsigned)(tiles_x * tiles_y), (unsigned)zch);
        if (d.preset == kP3d7) {
            st3d_cc<0, TY, 2><<<grid, 32 * TY, 0, s>>>(u, v, d, o0, o1, Z, tiles_x); note_launch();
        } else {
            double g[4];
            if (is_class_symmetric_27(d.w, g)) {
                StencilDesc dc = d;
                for (int m = 0; m < 4; ++m) dc.w[m] = g[m];
                st3d_cc<2, TY, 2><<<grid, 32 * TY, 0, s>>>(u, v, dc, o0, o1, Z, tiles_x); note_launch();
            } else {
                st3d_cc<1, TY, 2><<<grid, 32 * TY, 0, s>>>(u, v, d, o0, o1, Z, tiles_x); note_launch();
            }
        }
        return cudaGetLastError();
    }
    return launch_stencil_generic(d, o0, o1, u, v, s);
}

}  // namespace rlb
