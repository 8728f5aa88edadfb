// stencil_tc.cu -- K6/K8/K10: tensor-core Jacobi stencils as banded-matrix
// products on DMMA m8n8k4 (the ConvStencil idea the paper evaluates,
// PAPER.md:537-538; K-padding 10 -> 12, 3 MMA k-steps per product).
//
// Output tiles are 8x8 (one MMA accumulator).  With U the tile's input
// window (rows y0-1..y0+8, columns x0-1..x0+8) and band(a,b,c) the 12x8
// matrix with B[n][n]=a, B[n+1][n]=b, B[n+2][n]=c:
//
//   2d5pt  D = Ty * U[:,1:9]  +  U[1:9,:] * band(w_x-, 0, w_x+)      6 DMMA
//          Ty = band(w_y-, w_c, w_y+)^T (8x12, A operand, constant)
//   3d7pt  same in-plane products; the two z neighbours enter as the
//          accumulator input C = w_z- u(z-1) + w_z+ u(z+1) (DFMA)   6 DMMA
//   3d27pt weights depending only on m=|dx|+|dy|+|dz| (BASELINE.json):
//          by linearity out = P0(U_z) + P1(U_{z-1} + U_{z+1}) and each 2D
//          symmetric 9-point operator splits into a centre-row band and a
//          (row-1 + row+1) band, so three products suffice:
//            U_z[y]                                  * band(g1,g0,g1)
//            (U_z[y-1]+U_z[y+1]+U_{z-1}[y]+U_{z+1}[y]) * band(g2,g1,g2)
//            (U_{z-1}[y-1]+U_{z-1}[y+1]+U_{z+1}[y-1]+U_{z+1}[y+1])
//                                                    * band(g3,g2,g3)  9 DMMA
//          general 27-point weights: sum over (dz,dy) of U_{z+dz}[y+dy] *
//          band(w[dz][dy][-1..1])                                     27 DMMA
//
// Data movement is warp-private: each warp owns a 64-column strip and
// streams its input rows (2D: a 24-row ring) or plane tiles (3D: a 4-plane
// ring of 10x66 windows) into shared memory with cp.async (16-byte LDGSTS,
// 8-byte for the halo columns), one group ahead of the MMAs.  The ring is
// zeroed first so padded K slots always read finite values (0 * finite = 0
// inside the MMA; a NaN there would poison the whole accumulator row).
// Row stride 76 doubles (== 12 mod 16 in 8-byte banks) makes the operand
// gathers of both MMA orientations conflict-free.
#include "common.cuh"
#include "kernels.h"

namespace rlb {
namespace {

constexpr int kStride = 76;     // doubles per staged row
constexpr int kRing2d = 24;     // rows in the 2D ring
constexpr int kPlaneRows = 10;  // 3D window rows (8 + halo)
constexpr int kRing3d = 4;      // planes in the 3D ring

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp16(double* s, const double* g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp8(double* s, const double* g) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Element (k, n) of band(a, b, c): k = input offset in the 12-wide window.
__device__ __forceinline__ double band(int k, int n, double a, double b, double c) {
    return k == n ? a : (k == n + 1 ? b : (k == n + 2 ? c : 0.0));
}

// Copy `count` (even) doubles of a row into smem at dst (16-byte path) or
// element-wise (8-byte path), plus the two halo columns.
template <bool V16>
__device__ __forceinline__ void stage_row(double* dst, const double* src_row, int64_t x0,
                                          int64_t nx, int lane) {
    const int64_t x = x0 + 2 * lane;
    if (V16) {
        if (x < nx) cp16(dst + 2 + 2 * lane, src_row + x);
    } else {
        if (x < nx) cp8(dst + 2 + 2 * lane, src_row + x);
        if (x + 1 < nx) cp8(dst + 3 + 2 * lane, src_row + x + 1);
    }
    if (lane == 0 && x0 >= 1) cp8(dst + 1, src_row + x0 - 1);
    if (lane == 31 && x0 + 64 < nx) cp8(dst + 66, src_row + x0 + 64);
}

// Store one 8x8 accumulator: lane holds (row r, cols 2c, 2c+1).
template <bool V16>
__device__ __forceinline__ void store_tile(double* __restrict__ v_row, int64_t x, int64_t nx,
                                           double d0, double d1) {
    const bool in0 = x >= 1 && x <= nx - 2;
    const bool in1 = x + 1 >= 1 && x + 1 <= nx - 2;
    if (V16 && in0 && in1) {
        asm volatile("st.global.v2.f64 [%0], {%1,%2};" ::"l"(v_row + x), "d"(d0), "d"(d1) : "memory");
    } else {
        if (in0) v_row[x] = d0;
        if (in1) v_row[x + 1] = d1;
    }
}

// ---------------------------------------------------------------------------
// 2d5pt (w: centre, y-1, y+1, x-1, x+1)
// ---------------------------------------------------------------------------
template <bool V16>
__global__ void __launch_bounds__(128) st2d5_tc(const double* __restrict__ u,
                                                double* __restrict__ v, uint64_t nx,
                                                uint64_t y_begin, uint64_t y_end, int H,
                                                uint64_t strips, StencilDesc d) {
    extern __shared__ double smem[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int r = lane >> 2, c = lane & 3;
    double* ring = smem + wib * (kRing2d * kStride);
    const uint64_t wid = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t strip = wid % strips, seg = wid / strips;
    const uint64_t ya = y_begin + seg * (uint64_t)H;
    if (ya >= y_end) return;
    const uint64_t yb = min(ya + (uint64_t)H, y_end);
    const int64_t xs0 = (int64_t)strip * 64;
    const int64_t NX = (int64_t)nx;

    for (int i = lane; i < kRing2d * kStride; i += 32) ring[i] = 0.0;
    __syncwarp();

    double ty[3], tx[3];
#pragma unroll
    for (int kb = 0; kb < 3; ++kb) {
        ty[kb] = band(4 * kb + c, r, d.w[1], d.w[0], d.w[2]);  // A[r][k]: rows y-1, y, y+1
        tx[kb] = band(4 * kb + c, r, d.w[3], 0.0, d.w[4]);     // B[k][n]: cols x-1, x+1
    }
    auto slot = [&](uint64_t y) { return ring + ((y - (ya - 1)) % kRing2d) * kStride; };
    auto load_rows = [&](uint64_t lo, uint64_t hi) {  // rows [lo, hi] clipped to yb
        for (uint64_t y = lo; y <= hi && y <= yb; ++y)
            stage_row<V16>(slot(y), u + y * nx, xs0, NX, lane);
        cp_commit();
    };
    load_rows(ya - 1, ya + 8);
    load_rows(ya + 9, ya + 16);

    for (uint64_t y0 = ya; y0 < yb; y0 += 8) {
        cp_wait<1>();
        __syncwarp();
        const double* rowc = slot(y0 + r);  // centre row of this lane's output row
        double* vrow = v + (y0 + r) * nx;
        const bool row_ok = y0 + r < yb;
#pragma unroll 1
        for (int t = 0; t < 8; ++t) {
            const int64_t x0 = xs0 + 8 * t;
            if (x0 >= NX) break;
            double d0 = 0.0, d1 = 0.0;
#pragma unroll
            for (int kb = 0; kb < 3; ++kb) {
                const int j = min(4 * kb + c, 9);
                dmma_m8n8k4(d0, d1, ty[kb], slot(y0 - 1 + j)[8 * t + r + 2], d0, d1);
            }
#pragma unroll
            for (int kb = 0; kb < 3; ++kb) {
                const int j = min(4 * kb + c, 9);
                dmma_m8n8k4(d0, d1, rowc[8 * t + j + 1], tx[kb], d0, d1);
            }
            if (row_ok) store_tile<V16>(vrow, x0 + 2 * c, NX, d0, d1);
        }
        __syncwarp();
        load_rows(y0 + 17, y0 + 24);
    }
    cp_wait<0>();
}

// ---------------------------------------------------------------------------
// 3D: KIND 0 = 3d7pt (w: c, z-, z+, y-, y+, x-, x+), 1 = 3d27pt class weights
// (w[0..3] = g0..g3), 2 = 3d27pt general (w[(dz+1)*9 + (dy+1)*3 + dx+1]).
// ---------------------------------------------------------------------------
template <int KIND, bool V16>
__global__ void __launch_bounds__(128) st3d_tc(const double* __restrict__ u,
                                               double* __restrict__ v, StencilDesc d,
                                               uint64_t z_begin, uint64_t z_end, int zchunk,
                                               uint64_t tiles_x, uint64_t tiles_xy) {
    extern __shared__ double smem[];
    constexpr int kPlane = kPlaneRows * kStride;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int r = lane >> 2, c = lane & 3;
    double* ring = smem + wib * (kRing3d * kPlane);
    const uint64_t wid = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t tile = wid % tiles_xy, zc = wid / tiles_xy;
    const uint64_t za = z_begin + zc * (uint64_t)zchunk;
    if (za >= z_end) return;
    const uint64_t zb = min(za + (uint64_t)zchunk, z_end);
    const int64_t NX = (int64_t)d.nx, NY = (int64_t)d.ny;
    const int64_t x0 = (int64_t)(tile % tiles_x) * 64;
    const int64_t y0 = (int64_t)(tile / tiles_x) * 8;

    for (int i = lane; i < kRing3d * kPlane; i += 32) ring[i] = 0.0;
    __syncwarp();

    auto plane = [&](uint64_t p) { return ring + ((p - (za - 1)) % kRing3d) * kPlane; };
    auto load_plane = [&](uint64_t p) {
        if (p <= zb) {
            double* base = plane(p);
            const double* src = u + p * d.nx * d.ny;
#pragma unroll 1
            for (int j = 0; j < kPlaneRows; ++j) {
                const int64_t y = y0 - 1 + j;
                if (y < 0 || y >= NY) continue;
                stage_row<V16>(base + j * kStride, src + y * NX, x0, NX, lane);
            }
        }
        cp_commit();
    };

    // Constant band fragments.
    double fa[3], fb[3], fc[3];
#pragma unroll
    for (int kb = 0; kb < 3; ++kb) {
        const int k = 4 * kb + c;
        if (KIND == 0) {
            fa[kb] = band(k, r, d.w[3], d.w[0], d.w[4]);  // Ty (A operand)
            fb[kb] = band(k, r, d.w[5], 0.0, d.w[6]);     // Tx (B operand)
            fc[kb] = 0.0;
        } else {
            fa[kb] = band(k, r, d.w[1], d.w[0], d.w[1]);
            fb[kb] = band(k, r, d.w[2], d.w[1], d.w[2]);
            fc[kb] = band(k, r, d.w[3], d.w[2], d.w[3]);
        }
    }
    double gen[KIND == 2 ? 27 : 1];
    if (KIND == 2) {
#pragma unroll
        for (int q = 0; q < 9; ++q)
#pragma unroll
            for (int kb = 0; kb < 3; ++kb)
                gen[q * 3 + kb] = band(4 * kb + c, r, d.w[q * 3 + 0], d.w[q * 3 + 1], d.w[q * 3 + 2]);
    }

    load_plane(za - 1);
    load_plane(za);
    load_plane(za + 1);
    load_plane(za + 2);

    const int64_t yo = y0 + r;  // this lane's output row
    const bool row_ok = yo >= 1 && yo <= NY - 2;
    for (uint64_t z = za; z < zb; ++z) {
        cp_wait<1>();
        __syncwarp();
        const double* Pm = plane(z - 1);
        const double* P0 = plane(z);
        const double* Pp = plane(z + 1);
        double* vrow = v + (z * d.ny + (uint64_t)(row_ok ? yo : 0)) * d.nx;
#pragma unroll 1
        for (int t = 0; t < 8; ++t) {
            const int64_t xt = x0 + 8 * t;
            if (xt >= NX) break;
            double d0 = 0.0, d1 = 0.0;
            if (KIND == 0) {
                const int s = (r + 1) * kStride + 8 * t + 2 * c + 2;
                d0 = fma(d.w[2], Pp[s], d.w[1] * Pm[s]);
                d1 = fma(d.w[2], Pp[s + 1], d.w[1] * Pm[s + 1]);
#pragma unroll
                for (int kb = 0; kb < 3; ++kb) {
                    const int j = min(4 * kb + c, 9);
                    dmma_m8n8k4(d0, d1, fa[kb], P0[j * kStride + 8 * t + r + 2], d0, d1);
                }
#pragma unroll
                for (int kb = 0; kb < 3; ++kb) {
                    const int j = min(4 * kb + c, 9);
                    dmma_m8n8k4(d0, d1, P0[(r + 1) * kStride + 8 * t + j + 1], fb[kb], d0, d1);
                }
            } else if (KIND == 1) {
#pragma unroll
                for (int kb = 0; kb < 3; ++kb) {
                    const int col = 8 * t + min(4 * kb + c, 9) + 1;
                    const int up = r * kStride + col, mid = up + kStride, dn = mid + kStride;
                    const double a0 = P0[mid];
                    const double a1 = (P0[up] + P0[dn]) + (Pm[mid] + Pp[mid]);
                    const double a2 = (Pm[up] + Pm[dn]) + (Pp[up] + Pp[dn]);
                    dmma_m8n8k4(d0, d1, a0, fa[kb], d0, d1);
                    dmma_m8n8k4(d0, d1, a1, fb[kb], d0, d1);
                    dmma_m8n8k4(d0, d1, a2, fc[kb], d0, d1);
                }
            } else {
#pragma unroll
                for (int dz = 0; dz < 3; ++dz) {
                    const double* P = dz == 0 ? Pm : (dz == 1 ? P0 : Pp);
#pragma unroll
                    for (int dy = 0; dy < 3; ++dy)
#pragma unroll
                        for (int kb = 0; kb < 3; ++kb) {
                            const int col = 8 * t + min(4 * kb + c, 9) + 1;
                            dmma_m8n8k4(d0, d1, P[(r + dy) * kStride + col],
                                        gen[(dz * 3 + dy) * 3 + kb], d0, d1);
                        }
                }
            }
            if (row_ok) store_tile<V16>(vrow, xt + 2 * c, NX, d0, d1);
        }
        __syncwarp();
        load_plane(z + 3);
    }
    cp_wait<0>();
}

bool class_weights_27(const double* w, double g[4]) {
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

template <class K>
cudaError_t with_smem(K kernel, size_t bytes) {
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

}  // namespace

cudaError_t launch_stencil_tc(const StencilDesc& d, uint64_t o0, uint64_t o1, const double* u,
                              double* v, cudaStream_t s) {
    if (stencil_tma_eligible(d, u, v)) return launch_stencil_tma(1, d, o0, o1, u, v, s);
    const Tuning& t = tuning();
    const bool v16 = (d.nx % 2 == 0) && ((reinterpret_cast<uintptr_t>(u) & 15) == 0) &&
                     ((reinterpret_cast<uintptr_t>(v) & 15) == 0);
    cudaError_t e;
    if (d.preset == kP2d5) {
        const int H = 256;
        const uint64_t strips = (d.nx + 63) / 64;
        const uint64_t segs = (o1 - o0 + H - 1) / H;
        const uint64_t blocks = (strips * segs + 3) / 4;
        const size_t sm = 4 * kRing2d * kStride * sizeof(double);
        if (v16) {
            if ((e = with_smem(st2d5_tc<true>, sm)) != cudaSuccess) return e;
            st2d5_tc<true><<<(unsigned)blocks, 128, sm, s>>>(u, v, d.nx, o0, o1, H, strips, d);
        } else {
            if ((e = with_smem(st2d5_tc<false>, sm)) != cudaSuccess) return e;
            st2d5_tc<false><<<(unsigned)blocks, 128, sm, s>>>(u, v, d.nx, o0, o1, H, strips, d);
        }
        note_launch();
        return cudaGetLastError();
    }
    if (d.preset == kP3d7 || d.preset == kP3d27) {
        const int Z = t.tc_stencil_zchunk > 0 ? t.tc_stencil_zchunk : 32;
        const uint64_t tiles_x = (d.nx + 63) / 64, tiles_y = (d.ny + 7) / 8;
        const uint64_t tiles_xy = tiles_x * tiles_y;
        const uint64_t warps = tiles_xy * ((o1 - o0 + Z - 1) / Z);
        const uint64_t blocks = (warps + 3) / 4;
        const size_t sm = 4 * kRing3d * kPlaneRows * kStride * sizeof(double);
        StencilDesc dd = d;
        int kind = 0;
        if (d.preset == kP3d27) {
            double g[4];
            if (class_weights_27(d.w, g)) {
                kind = 1;
                for (int m = 0; m < 4; ++m) dd.w[m] = g[m];
            } else {
                kind = 2;
            }
        }
#define RLB_LAUNCH_3D(K, V)                                                                   \
    do {                                                                                      \
        if ((e = with_smem(st3d_tc<K, V>, sm)) != cudaSuccess) return e;                      \
        st3d_tc<K, V><<<(unsigned)blocks, 128, sm, s>>>(u, v, dd, o0, o1, Z, tiles_x, tiles_xy); \
    } while (0)
        if (kind == 0) { if (v16) RLB_LAUNCH_3D(0, true); else RLB_LAUNCH_3D(0, false); }
        else if (kind == 1) { if (v16) RLB_LAUNCH_3D(1, true); else RLB_LAUNCH_3D(1, false); }
        else { if (v16) RLB_LAUNCH_3D(2, true); else RLB_LAUNCH_3D(2, false); }
#undef RLB_LAUNCH_3D
        note_launch();
        return cudaGetLastError();
    }
    // No tensor-core formulation for the other presets: refuse rather than
    // silently running the CUDA-core kernel under the tensor-core name.
    return cudaErrorNotSupported;
}

}  // namespace rlb
