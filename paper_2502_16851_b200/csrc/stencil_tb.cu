// stencil_tb.cu -- 2d5pt temporal blocking of depth T in registers (SURVEY.md
// §8f "next" #1; the reference's stencil_model(shape, P, t)
// and min_temporal_depth, kernels.cpp:137-155 / bounds.cpp:111-125).
//
// HBM sees one read of u and one write of v per T timesteps.  A warp owns a
// 64-column strip (two adjacent columns per lane) and marches a row segment
// top to bottom.  For every input row it advances a skewed pipeline of T
// levels: level l keeps a 3-row window (rows r-1, r, r+1 of timestep l) in
// registers, and each new level-(l-1) row yields level-l row r =
// S(window of level l-1) one row behind.  Vertical neighbours are the window
// registers; horizontal neighbours are one shuffle each way (the lane's two
// columns cover each other).  A level's lanes at the strip edge read an
// invalid neighbour, so the valid region shrinks by one column per level: a
// warp's 64 loaded columns (T halo columns each side) yield 64 - 2T outputs.
// No shared memory, no barriers; per input row a lane does one 16-byte load,
// T x (2 shuffles + 10 DFMA) and, after the pipeline fills, one 16-byte
// store.
//
// Dirichlet points (global row 0 / ny-1, column 0 / nx-1) keep their value at
// every level; loads outside the grid read 0 and only ever feed boundary
// points, which ignore them, or lanes/rows outside the dependency cone of a
// stored output.
#include <cuda.h>

#include "common.cuh"
#include "kernels.h"
#include "tma.cuh"

namespace rlb {
namespace {

template <int T>
struct TbGeom {
    static constexpr int kCols = 64;            // columns a warp loads
    static constexpr int kOut = kCols - 2 * T;  // columns it stores
    static_assert(T >= 2 && T <= 8, "temporal depth 2..8");
    static constexpr bool kVec = T % 2 == 0;    // even T: the lane's column pair is 16-byte aligned
};

// One warp's march over rows [ya, yb) of its strip.  EDGE: the warp's loaded
// rows or columns reach the grid's edge (Dirichlet rows/columns, points
// outside the grid); otherwise it runs with no bounds checks and the weights
// straight from the parameter bank.
template <int T, int PF, bool EDGE>
__device__ __forceinline__ void tb_march(const double* __restrict__ u, double* __restrict__ v, int nx, int ny,
                                         int ya, int yb, int strip, int lane, const StencilDesc& d) {
    using G = TbGeom<T>;
    // this lane's two columns; the strip's first loaded column is even when T is
    const int xa = strip * G::kOut - T + 2 * lane;
    const bool in0 = xa >= 0 && xa < nx, in1 = xa + 1 >= 0 && xa + 1 < nx;
    const bool bnd0 = xa <= 0 || xa >= nx - 1, bnd1 = xa + 1 <= 0 || xa + 1 >= nx - 1;
    // columns valid after T levels: [strip * kOut, strip * kOut + kOut)
    const int olo = strip * G::kOut, ohi = olo + G::kOut;
    const bool st0 = xa >= olo && xa < ohi && !bnd0 && in0;
    const bool st1 = xa + 1 >= olo && xa + 1 < ohi && !bnd1 && in1;
    // per-column weights at the edge: a Dirichlet column keeps its value
    // (w = 1, 0, 0, 0, 0); interior launches read d.w from the parameter bank
    const double a0 = EDGE && bnd0 ? 1.0 : d.w[0], a1 = EDGE && bnd0 ? 0.0 : d.w[1],
                 a2 = EDGE && bnd0 ? 0.0 : d.w[2], a3 = EDGE && bnd0 ? 0.0 : d.w[3],
                 a4 = EDGE && bnd0 ? 0.0 : d.w[4];
    const double b0 = EDGE && bnd1 ? 1.0 : d.w[0], b1 = EDGE && bnd1 ? 0.0 : d.w[1],
                 b2 = EDGE && bnd1 ? 0.0 : d.w[2], b3 = EDGE && bnd1 ? 0.0 : d.w[3],
                 b4 = EDGE && bnd1 ? 0.0 : d.w[4];

    // level windows: lv[l][0] = row r-1, [1] = row r, [2] = row r+1 (two columns each)
    double2 lv[T][3];
#pragma unroll
    for (int l = 0; l < T; ++l) lv[l][0] = lv[l][1] = lv[l][2] = make_double2(0.0, 0.0);

    const int i0 = ya - T;          // first input row
    const int i1 = yb - 1 + T;      // last input row (the loop runs to a multiple of PF)
    const double* src = u + (int64_t)i0 * nx + xa;
    auto load = [&](int i, const double* p) -> double2 {
        double2 r = make_double2(0.0, 0.0);
        if (!EDGE || (i >= 0 && i < ny)) {
            if (G::kVec && (!EDGE || (in0 && in1))) {
                r = __ldg(reinterpret_cast<const double2*>(p));
            } else {
                if (in0) r.x = __ldg(p);
                if (in1) r.y = __ldg(p + 1);
            }
        }
        return r;
    };
    // software prefetch queue: PF rows in flight
    double2 q[PF];
#pragma unroll
    for (int j = 0; j < PF; ++j) q[j] = load(i0 + j, src + (int64_t)j * nx);
    const double* pf = src + (int64_t)PF * nx;
    double* dst = v + (int64_t)(i0 - T) * nx + xa;  // output row r = ii - T (advanced once per input row)

    for (int i = i0; i <= i1; i += PF) {
#pragma unroll
        for (int j = 0; j < PF; ++j) {
            const int ii = i + j;
            const double2 in = q[j];
            q[j] = load(ii + PF, pf);
            pf += nx;
            lv[0][0] = lv[0][1];
            lv[0][1] = lv[0][2];
            lv[0][2] = in;
#pragma unroll
            for (int l = 1; l <= T; ++l) {
                const double2 up = lv[l - 1][0], c = lv[l - 1][1], dn = lv[l - 1][2];
                const double left = __shfl_up_sync(0xffffffffu, c.y, 1);    // column xa - 1
                const double right = __shfl_down_sync(0xffffffffu, c.x, 1); // column xa + 2
                double2 o;
                o.x = a0 * c.x;
                o.x = fma(a1, up.x, o.x);
                o.x = fma(a2, dn.x, o.x);
                o.x = fma(a3, left, o.x);
                o.x = fma(a4, c.y, o.x);
                o.y = b0 * c.y;
                o.y = fma(b1, up.y, o.y);
                o.y = fma(b2, dn.y, o.y);
                o.y = fma(b3, c.x, o.y);
                o.y = fma(b4, right, o.y);
                if (EDGE) {
                    const int r = ii - l;
                    if (r <= 0 || r >= ny - 1) o = c;  // Dirichlet row: keep the value
                }
                if (l < T) {
                    lv[l][0] = lv[l][1];
                    lv[l][1] = lv[l][2];
                    lv[l][2] = o;
                } else {
                    const int r = ii - T;
                    if (r >= ya && r < yb) {
                        if (G::kVec && st0 && st1)
                            asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(dst), "d"(o.x), "d"(o.y)
                                         : "memory");
                        else {
                            if (st0) dst[0] = o.x;
                            if (st1) dst[1] = o.y;
                        }
                    }
                    dst += nx;
                }
            }
        }
    }
}

template <int T, int PF>
__global__ void __launch_bounds__(256, 2) st2d_cc_tb(const double* __restrict__ u, double* __restrict__ v, int nx, int ny,
                                                  int y_begin, int y_end, int seg_rows, int strips,
                                                  const __grid_constant__ StencilDesc d) {
    using G = TbGeom<T>;
    const int lane = threadIdx.x & 31;
    const int gw = (int)(((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int strip = gw % strips;
    const int ya = y_begin + (gw / strips) * seg_rows;
    if (ya >= y_end) return;
    const int yb = min(ya + seg_rows, y_end);
    const bool edge = ya - T <= 0 || yb - 1 + T + 2 * PF >= ny - 1 ||  // prefetch reaches row i1 + 2 PF - 1
                      strip * G::kOut - T <= 0 || strip * G::kOut - T + G::kCols >= nx - 1;
    if (edge)
        tb_march<T, PF, true>(u, v, nx, ny, ya, yb, strip, lane, d);
    else
        tb_march<T, PF, false>(u, v, nx, ny, ya, yb, strip, lane, d);
}

// The same march fed by TMA instead of a register queue (t >= 4, where the
// level windows leave no registers for prefetch): each warp streams its
// strip's input rows, RR at a time, through a ring of NS shared-memory
// slots (one mbarrier each; lane 0 issues the 2D box, OOB rows/columns arrive
// as zeros), so ~NS x RR rows are in flight at no register cost.  Odd T
// loads the box from the even column before the strip (16-byte aligned TMA
// start) and reads the lane's pair unaligned.
template <int T>
struct TbtGeom {
    static constexpr int kOdd = T & 1;
    static constexpr int kBoxX = 64 + 2 * kOdd;                  // 64 or 66 columns
    static constexpr int kRow = kBoxX;                           // doubles per smem row
};

template <int T, int NS, int RR, bool EDGE>
__device__ __forceinline__ void tbt_march(const CUtensorMap* tm, double* __restrict__ v, int nx, int ny, int ya,
                                          int yb, int strip, int lane, double* ring, uint64_t* bar,
                                          const StencilDesc& d) {
    using G = TbGeom<T>;
    using H = TbtGeom<T>;
    constexpr int SLOT = ((RR * H::kRow * 8 + 127) / 128) * 128 / 8;  // doubles per slot (128-byte aligned)
    const int xa = strip * G::kOut - T + 2 * lane;
    const int xbox = strip * G::kOut - T - H::kOdd;  // even
    const bool in0 = xa >= 0 && xa < nx, in1 = xa + 1 >= 0 && xa + 1 < nx;
    const bool bnd0 = xa <= 0 || xa >= nx - 1, bnd1 = xa + 1 <= 0 || xa + 1 >= nx - 1;
    const int olo = strip * G::kOut, ohi = olo + G::kOut;
    const bool st0 = xa >= olo && xa < ohi && !bnd0 && in0;
    const bool st1 = xa + 1 >= olo && xa + 1 < ohi && !bnd1 && in1;
    const double a0 = EDGE && bnd0 ? 1.0 : d.w[0], a1 = EDGE && bnd0 ? 0.0 : d.w[1],
                 a2 = EDGE && bnd0 ? 0.0 : d.w[2], a3 = EDGE && bnd0 ? 0.0 : d.w[3],
                 a4 = EDGE && bnd0 ? 0.0 : d.w[4];
    const double b0 = EDGE && bnd1 ? 1.0 : d.w[0], b1 = EDGE && bnd1 ? 0.0 : d.w[1],
                 b2 = EDGE && bnd1 ? 0.0 : d.w[2], b3 = EDGE && bnd1 ? 0.0 : d.w[3],
                 b4 = EDGE && bnd1 ? 0.0 : d.w[4];

    double2 lv[T][3];
#pragma unroll
    for (int l = 0; l < T; ++l) lv[l][0] = lv[l][1] = lv[l][2] = make_double2(0.0, 0.0);

    const int i0 = ya - T, i1 = yb - 1 + T;
    const int groups = (i1 - i0 + RR) / RR;
    auto issue = [&](int g) {
        const int sl = g % NS;
        tmaop::mbar_expect_tx(bar + sl, RR * H::kBoxX * 8);
        tmaop::tma2d(ring + sl * SLOT, tm, bar + sl, xbox, i0 + g * RR);
    };
    if (lane == 0)
        for (int g = 0; g < NS && g < groups; ++g) issue(g);
    double* dst = v + (int64_t)(i0 - T) * nx + xa;
    const double* mine = ring + 2 * lane + H::kOdd;
    for (int g = 0; g < groups; ++g) {
        const int sl = g % NS;
        tmaop::mbar_wait(bar + sl, (uint32_t)((g / NS) & 1));
        const double* rows = mine + sl * SLOT;
#pragma unroll
        for (int j = 0; j < RR; ++j) {
            const int ii = i0 + g * RR + j;
            double2 in;
            if (H::kOdd) {
                in.x = rows[j * H::kRow];
                in.y = rows[j * H::kRow + 1];
            } else {
                in = *reinterpret_cast<const double2*>(rows + j * H::kRow);
            }
            lv[0][0] = lv[0][1];
            lv[0][1] = lv[0][2];
            lv[0][2] = in;
#pragma unroll
            for (int l = 1; l <= T; ++l) {
                const double2 up = lv[l - 1][0], c = lv[l - 1][1], dn = lv[l - 1][2];
                const double left = __shfl_up_sync(0xffffffffu, c.y, 1);
                const double right = __shfl_down_sync(0xffffffffu, c.x, 1);
                double2 o;
                o.x = a0 * c.x;
                o.x = fma(a1, up.x, o.x);
                o.x = fma(a2, dn.x, o.x);
                o.x = fma(a3, left, o.x);
                o.x = fma(a4, c.y, o.x);
                o.y = b0 * c.y;
                o.y = fma(b1, up.y, o.y);
                o.y = fma(b2, dn.y, o.y);
                o.y = fma(b3, c.x, o.y);
                o.y = fma(b4, right, o.y);
                if (EDGE) {
                    const int r = ii - l;
                    if (r <= 0 || r >= ny - 1) o = c;
                }
                if (l < T) {
                    lv[l][0] = lv[l][1];
                    lv[l][1] = lv[l][2];
                    lv[l][2] = o;
                } else {
                    const int r = ii - T;
                    if (r >= ya && r < yb) {
                        if (G::kVec && st0 && st1)
                            asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(dst), "d"(o.x), "d"(o.y)
                                         : "memory");
                        else {
                            if (st0) dst[0] = o.x;
                            if (st1) dst[1] = o.y;
                        }
                    }
                    dst += nx;
                }
            }
        }
        __syncwarp();  // every lane has read slot sl
        if (lane == 0 && g + NS < groups) issue(g + NS);
    }
}

template <int T, int NS, int RR>
__global__ void __launch_bounds__(256, 2) st2d_cc_tbt(const __grid_constant__ CUtensorMap tm, double* __restrict__ v,
                                                   int nx, int ny, int y_begin, int y_end, int seg_rows, int strips,
                                                   const __grid_constant__ StencilDesc d) {
    using G = TbGeom<T>;
    using H = TbtGeom<T>;
    constexpr int SLOT = ((RR * H::kRow * 8 + 127) / 128) * 128 / 8;
    extern __shared__ __align__(128) double smem[];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    double* ring = smem + wl * NS * SLOT;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 8 * NS * SLOT) + wl * NS;
    if (lane == 0) {
        for (int s = 0; s < NS; ++s) tmaop::mbar_init(bar + s, 1);
        tmaop::mbar_fence_init();
    }
    __syncwarp();
    const int gw = (int)(((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int strip = gw % strips;
    const int ya = y_begin + (gw / strips) * seg_rows;
    if (ya >= y_end) return;
    const int yb = min(ya + seg_rows, y_end);
    const bool edge = ya - T <= 0 || yb - 1 + T >= ny - 1 || strip * G::kOut - T <= 0 ||
                      strip * G::kOut - T + G::kCols >= nx - 1;
    if (edge)
        tbt_march<T, NS, RR, true>(&tm, v, nx, ny, ya, yb, strip, lane, ring, bar, d);
    else
        tbt_march<T, NS, RR, false>(&tm, v, nx, ny, ya, yb, strip, lane, ring, bar, d);
}

template <int T, int NS, int RR>
constexpr size_t tbt_smem() {
    constexpr int SLOT = ((RR * TbtGeom<T>::kRow * 8 + 127) / 128) * 128 / 8;
    return (size_t)8 * NS * SLOT * 8 + 8 * NS * 8;
}

// Rows in flight per warp (a multiple of 3, so the unrolled body returns
// every level window to the same registers).  The kernel is occupancy-bound
// by registers (2 CTAs/SM), so its HBM parallelism is this prefetch queue.
// Per timestep at 16384^2 (tools/sweep.py temporal_t, 3 / 6 / 9 rows):
// t = 2 0.53 / 0.42 / 0.38 ms, t = 3 0.30 / 0.26 / -, t = 4 0.29 / 0.27 / -,
// t = 5 0.21 / 0.24 / -; deeper t sit at the 128-register cap, where longer
// queues spill and lose.  (A two-row partial-sum window per level measured
// slower: t = 2 0.72 ms at 9 rows.)
template <int T>
constexpr int tb_pf() {
    return T == 2 ? 9 : (T <= 4 ? 6 : 3);
}

template <int T, int NS, int RR>
cudaError_t launch_tbt(const StencilDesc& d, uint64_t o0, uint64_t o1, const double* u, double* v, cudaStream_t s) {
    using G = TbGeom<T>;
    alignas(64) CUtensorMap m;
    if (!encode_map_2d(&m, u, d.nx, d.ny, TbtGeom<T>::kBoxX, RR, 1)) return cudaErrorInvalidValue;
    constexpr size_t smem = tbt_smem<T, NS, RR>();
    auto kern = st2d_cc_tbt<T, NS, RR>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    static int bps = 0;
    if (!bps) {
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, 256, smem) != cudaSuccess || bps < 1) bps = 1;
    }
    const int strips = (int)((d.nx + G::kOut - 1) / G::kOut);
    const uint64_t rows = o1 - o0;
    const uint64_t want_warps = (uint64_t)kNumSMs * (uint64_t)bps * 8 * (uint64_t)tuning().stencil_tb_waves;
    uint64_t nseg = want_warps / (uint64_t)strips;
    const uint64_t cap = rows / (uint64_t)(16 * T) > 0 ? rows / (uint64_t)(16 * T) : 1;
    if (nseg > cap) nseg = cap;
    if (nseg < 1) nseg = 1;
    const int seg_rows = (int)((rows + nseg - 1) / nseg);
    const uint64_t segs = (rows + seg_rows - 1) / seg_rows;
    const uint64_t warps = (uint64_t)strips * segs;
    const unsigned blocks = (unsigned)((warps + 7) / 8);
    kern<<<blocks, 256, smem, s>>>(m, v, (int)d.nx, (int)d.ny, (int)o0, (int)o1, seg_rows, strips, d);
    note_launch();
    return cudaGetLastError();
}

template <int T>
cudaError_t launch_tb(const StencilDesc& d, uint64_t o0, uint64_t o1, const double* u, double* v, cudaStream_t s) {
    const int tma_from = tuning().stencil_tb_tma;
    if (tma_from > 0 && T >= tma_from && (reinterpret_cast<uintptr_t>(u) & 15) == 0 && d.nx % 2 == 0 &&
        tma_encode_available())
        return launch_tbt<T, 4, 3>(d, o0, o1, u, v, s);  // 6x3, 4x6, 8x3 slots x rows measured no better
    using G = TbGeom<T>;
    const int strips = (int)((d.nx + G::kOut - 1) / G::kOut);
    // row segments: one wave of resident warps (occupancy from the register
    // count) times stencil_tb_waves; each segment recomputes T rows above and
    // below (halo), so keep it >= 16 T rows
    static int bps = 0;
    if (!bps) {
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, st2d_cc_tb<T, tb_pf<T>()>, 256, 0) != cudaSuccess ||
            bps < 1)
            bps = 1;
    }
    const uint64_t rows = o1 - o0;
    const uint64_t want_warps = (uint64_t)kNumSMs * (uint64_t)bps * 8 * (uint64_t)tuning().stencil_tb_waves;
    uint64_t nseg = want_warps / (uint64_t)strips;
    const uint64_t cap = rows / (uint64_t)(16 * T) > 0 ? rows / (uint64_t)(16 * T) : 1;
    if (nseg > cap) nseg = cap;
    if (nseg < 1) nseg = 1;
    const int seg_rows = (int)((rows + nseg - 1) / nseg);
    const uint64_t segs = (rows + seg_rows - 1) / seg_rows;
    const uint64_t warps = (uint64_t)strips * segs;
    const unsigned blocks = (unsigned)((warps + 7) / 8);
    st2d_cc_tb<T, tb_pf<T>()><<<blocks, 256, 0, s>>>(u, v, (int)d.nx, (int)d.ny, (int)o0, (int)o1, seg_rows, strips, d);
    note_launch();
    return cudaGetLastError();
}

}  // namespace

bool stencil_tb_supported(const StencilDesc& d, int t, const double* u, const double* v) {
    if (d.preset != kP2d5 || t < 2 || t > 8) return false;
    if (d.nx >= (1ull << 30) || d.ny >= (1ull << 30) || d.nx * d.ny >= (1ull << 62)) return false;  // int rows/cols
    if (t % 2 == 0 && ((reinterpret_cast<uintptr_t>(u) & 15) || (reinterpret_cast<uintptr_t>(v) & 15) || d.nx % 2))
        return false;  // the vector path needs 16-byte aligned rows
    return true;
}

cudaError_t launch_stencil_tb(const StencilDesc& d, int t, uint64_t o0, uint64_t o1, const double* u, double* v,
                              cudaStream_t s) {
    if (!stencil_tb_supported(d, t, u, v)) return cudaErrorInvalidValue;
    switch (t) {
        case 2: return launch_tb<2>(d, o0, o1, u, v, s);
        case 3: return launch_tb<3>(d, o0, o1, u, v, s);
        case 4: return launch_tb<4>(d, o0, o1, u, v, s);
        case 5: return launch_tb<5>(d, o0, o1, u, v, s);
        case 6: return launch_tb<6>(d, o0, o1, u, v, s);
        case 7: return launch_tb<7>(d, o0, o1, u, v, s);
        default: return launch_tb<8>(d, o0, o1, u, v, s);
    }
}

}  // namespace rlb
