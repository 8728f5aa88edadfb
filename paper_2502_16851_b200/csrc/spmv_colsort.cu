// spmv_colsort.cu -- K17: the SpMV plan's column-sorted row-block layout.
//
// Why: on the BASELINE band matrix the CSR kernels (spmv.cu) are bound by one
// L1 request per x gather (67.1 M random 8-byte gathers per call, ~1 per SM
// per cycle), not by HBM.  Here a block of R rows keeps its nonzeros sorted
// by COLUMN, so a warp instruction's 32 consecutive entries read x from a
// few L1 lines (~40 columns at R ~ 7000 and 16 nonzeros per row) instead of
// 32 random ones; the products are added into the block's y rows held in
// shared memory.
//
// Layout (built once on the host by rl_spmv_plan_create; bytes <= CSR's):
//   val  f64  per entry
//   meta u32  per entry = (col - block.col_lo) << rb | (row - block.row0)
//   blocks    {first entry, col_lo, row0, rows, entries}; entries padded to a
//             multiple of 32 with (val = 0, column col_lo, row = rows): the
//             padding adds into a scratch slot past the block's rows that is
//             never written back.
// FP64 rows: within each window of 128 sorted entries the host orders the
// entries so every aligned half-warp of 16 has distinct row % 16 where the
// window allows: the 64-bit shared-memory accesses of a half-warp then hit
// distinct bank pairs (tools/micro/spmv_colsort.cu: 0.2017 -> 0.1829 ms).
// The fixed-point grid's 32-bit atomics gain nothing from such an order and
// keep the plain column order, which reads x from the fewest lines
// (tools/micro/colsort_banks.py: 0.1593 ms vs 0.1601-0.1617 with groups).
//
// CUDA core: 1024-thread CTAs, two per SM (y rows <= 8192 -> 64 KB each),
// persistent over the blocks; each thread streams entries e, e+1024, e+2048
// (val/meta evict_first, x gathers evict_last so x stays in L2), multiplies
// and adds the product into its row in shared memory.
//
// Row sums (spmv_colsort_fixed = 1, the CUDA-core default): on a 64-bit
// fixed-point grid per block, q = RN(p 2^S) with S = 62 - hl - Et, where
// |p| < 2^Et for every product of the block and a row has <= 2^hl of them, so
// |row sum| <= 2^62 and nothing wraps; a q is added as two native 32-bit
// shared atomics (low word, then high word plus the carry the first one's old
// value gives).  Integer additions commute: the result does not depend on the
// order, calls are bit-identical.  Et comes from the block's previous call
// (plan creation: a guess assuming |x| < 1) and is checked against this
// call's largest product; a mismatch redoes the block on the grid the data
// calls for (Et rounded up to a multiple of 8, so x drifting by less than
// 2^8 costs no redo).  Rows whose sum holds fewer than 45 + hl bits of the
// grid (sum far below the block's largest product, or cancelling; ~0.1% of
// the BASELINE rows) are summed again in FP64 from the CSR by 4 lanes each in
// a fixed order, so every row is within 2^-46 of its own magnitude or within
// the FP64 recursive-summation bound.  Inf/NaN products switch the block to
// FP64 atomics (IEEE propagation).
// spmv_colsort_fixed = 0 (and the tensor-core unit at 1): shared-memory FP64
// atomicAdd (a CAS loop on sm_100a), FP64 arithmetic but the order of a row's
// additions is not fixed, so repeated calls may differ in the last bits.
// Measured (profiles/spmv_colsort_r2.md): CAS 0.178 ms, 64-bit grid 0.162 ms
// (0.155 + the FP64 row kernel; summing the flagged rows inside the main
// kernel stalls its stream: 0.191 ms); exact 96-bit rows (three atomics per entry)
// 0.185-0.21 ms, MIO-bound.
// Tensor core: the same blocks and accumulation; the 32 products of a warp
// step come out of TWO DMMA m8n8k4.  A product of per-entry operands is
// isolated in an output only when that output's other three k terms are zero,
// so each MMA's k slots own disjoint quadrants of the 8x8 output: k's A
// column is non-zero on 4 rows M_k, its B row on 4 columns N_k, the four
// M_k x N_k tile the output, and a bijection M_k -> N_k pairs 4 (val, x)
// per k -- 16 isolated products per MMA (the most four disjoint rectangles in
// 8x8 allow), 32 per two.  The second MMA uses the complementary A and B
// slots and the opposite diagonal, so every lane owns exactly one A operand,
// one B operand and one useful output across the pair.  The host stores each
// 32-entry group permuted to those roles (tc_roles): val in A-slot order, the
// column bits of meta in B-slot order, the row bits in output order -- the
// same 12 B per entry, no shuffles (the FP64 fallback below unpermutes with
// two).  Measured against the round's first form (4 masked DMMA per step,
// 8 useful outputs each, shuffled home): see profiles/spmv_colsort_r2.md.
#include <algorithm>
#include <cstring>
#include <thread>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace rlb {

namespace {
constexpr int kThreads = 1024;

// Tensor-core lane roles of the entry whose value sits in A slot `la` = 4m+k
// (A[m][k]): which MMA of the pair (first: rows 0-3 with k < 2, rows 4-7 with
// k >= 2), its B slot lb (B[k][n] is held by lane 4n+k) and the lane ld whose
// output D[m][n] holds its product (lane 4m + n/2, element n & 1 = m & 1).
// First MMA: k even -> columns 0-3, k odd -> 4-7, n = m mod 4 (+4); second:
// the other half, n = (m mod 4) ^ 2 (+4).
__host__ __device__ __forceinline__ void tc_roles(int la, int& lb, int& ld) {
    const int m = la >> 2, k = la & 3;
    const bool first = ((la >> 4) & 1) == ((la >> 1) & 1);
    const int n = first ? (m & 3) + ((k & 1) << 2) : ((m & 3) ^ 2) + ((k & 1) ? 0 : 4);
    lb = 4 * n + k;
    ld = 4 * m + (n >> 1);
}
constexpr int kUnroll = 3;  // entry loads in flight per thread (measured: U2 0.183, U3 0.173, U4 0.193 ms)

__device__ __forceinline__ void ld_stream2(const double* p, uint64_t pol, double& a, double& b) {
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(a), "=d"(b) : "l"(p), "l"(pol));
}
__device__ __forceinline__ void ld_meta2(const unsigned* p, uint64_t pol, unsigned& a, unsigned& b) {
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0, %1}, [%2], %3;" : "=r"(a), "=r"(b) : "l"(p), "l"(pol));
}
__device__ __forceinline__ void ld_meta4(const unsigned* p, uint64_t pol, unsigned& a, unsigned& b, unsigned& c,
                                         unsigned& d) {
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
        : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
        : "l"(p), "l"(pol));
}
__device__ __forceinline__ unsigned ld_meta(const unsigned* p, uint64_t pol) {
    unsigned v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}

// Grid exponent a block's products call for: Et with |p| <= 2^Et, rounded up
// to a multiple of kColsortQuantum so the grid -- and the result -- depends on
// the data alone; kColsortFp64 when a product is Inf/NaN; `keep` when every
// product is zero (any grid gives 0).  The products are tracked as integers:
// mh = the largest high word of |p| (IEEE order is integer order for
// non-negative doubles, Inf/NaN the largest: exponent field 0x7FF), ml = the OR
// of the low words (a product with a zero high word is still non-zero).
__device__ __forceinline__ int grid_of(unsigned mh, unsigned ml, int keep) {
    if (mh >= 0x7ff00000u) return kColsortFp64;
    if ((mh | ml) == 0u) return keep;
    const int e = (int)(mh >> 20);
    const int ea = e ? e - 1022 : -1022;  // |p| < 2^ea
    return (ea >= 0 ? (ea + kColsortQuantum - 1) / kColsortQuantum : -((-ea) / kColsortQuantum)) * kColsortQuantum;
}

// One product onto the block's 64-bit grid: q = RN(p 2^S) (|q| < 2^62), low
// word by a native shared atomic whose old value gives the carry, high word
// (with the carry) by a second one.  Integer sums do not depend on order.
__device__ __forceinline__ void add64(unsigned* __restrict__ lo, unsigned* __restrict__ hi, unsigned row, double p,
                                      double f) {
    const long long q = __double2ll_rn(p * f);
    const unsigned l = (unsigned)q;
    const unsigned old = atomicAdd(lo + row, l);
    atomicAdd(hi + row, (unsigned)(q >> 32) + ((old + l) < old ? 1u : 0u));
}

// TRACK: keep the largest |product| and an Inf/NaN witness (the grid check)
template <bool TC, bool FIXED, bool TRACK, int NT, int UF, bool PIPE, int V>
__device__ __forceinline__ void block_entries(double* __restrict__ ys, unsigned* __restrict__ lo,
                                              unsigned* __restrict__ hi, const double* __restrict__ vb,
                                              const unsigned* __restrict__ mb, const double* __restrict__ xb,
                                              unsigned nent, int rb, double f, uint64_t pol, uint64_t polx,
                                              unsigned& mh, unsigned& ml) {
    const unsigned rmask = (1u << rb) - 1;
    const int lane = threadIdx.x & 31;
    auto add = [&](unsigned row, double p) {
        if (TRACK) {  // integer ops only: the FP64 pipe is the tensor core's too
            mh = max(mh, (unsigned)__double2hiint(p) & 0x7fffffffu);
            ml |= (unsigned)__double2loint(p);
        }
        if (FIXED) add64(lo, hi, row, p, f);
        else atomicAdd(ys + row, p);
    };
    // tensor core, lane-permuted layout: this lane's A operand (v) and B
    // operand (xv) belong to the first MMA or the second, and so does its output
    const bool a_first = ((lane >> 4) & 1) == ((lane >> 1) & 1);
    const bool b_first = (lane & 1) == ((lane >> 4) & 1);
    const bool d_first = (lane & 1) == ((lane >> 3) & 1);
    const bool d_odd = (lane >> 2) & 1;
    int lb = 0, ld = 0;
    tc_roles(lane, lb, ld);
    auto step = [&](double v, unsigned mt, double xv) {
        if (!TC) {
            add(mt & rmask, v * xv);
        } else if (FIXED) {
            // two DMMA give the warp's 32 products, one per lane, no data exchange.
            // A zero operand meeting an Inf/NaN x makes a neighbour's product NaN:
            // the block's witness then sends it to the FP64 pass below.
            double d10, d11, d20, d21;
            dmma_m8n8k4(d10, d11, a_first ? v : 0.0, b_first ? xv : 0.0, 0.0, 0.0);
            dmma_m8n8k4(d20, d21, a_first ? 0.0 : v, b_first ? 0.0 : xv, 0.0, 0.0);
            add(mt & rmask, d_first ? (d_odd ? d11 : d10) : (d_odd ? d21 : d20));
        } else {
            // FP64 pass (and Inf/NaN data): bring this A slot's x and row home
            // with two shuffles, then 4 DMMA with both operands masked to one k
            // slot, so an Inf/NaN never meets another entry's zero (Inf * 0 = NaN).
            // The product of lane 4c+j is D_j[c][c], held by lane 4c + (c >> 1) in
            // slot c & 1; one shuffle per MMA brings it back.
            const double xa = __shfl_sync(0xffffffffu, xv, lb);
            const unsigned ra = __shfl_sync(0xffffffffu, mt & rmask, ld);
            const int c = lane >> 2;
            const int home = 4 * c + (c >> 1);
            double p = 0.0;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                double d0, d1;
                const bool mine = (lane & 3) == j;
                dmma_m8n8k4(d0, d1, mine ? v : 0.0, mine ? xa : 0.0, 0.0, 0.0);
                const double q = __shfl_sync(0xffffffffu, (c & 1) ? d1 : d0, home);
                if (mine) p = q;
            }
            add(ra, p);
        }
    };
    // A thread takes units of V consecutive entries (V = 2: one 128-bit val and
    // one 64-bit meta load per unit); nent is a multiple of 32 V, so every warp
    // step is full.  Unit i covers entries [V i, V i + V).
    auto load = [&](unsigned i, double (&v)[V], unsigned (&m)[V]) {
        if (V == 1) {
            v[0] = ld_stream(vb + i, pol);
            m[0] = ld_meta(mb + i, pol);
        } else if (V == 2) {
            ld_stream2(vb + 2 * i, pol, v[0], v[V - 1]);
            ld_meta2(mb + 2 * i, pol, m[0], m[V - 1]);
        } else {
            const d4 q = ld4_stream(vb + 4 * i, pol);  // 256-bit
            v[0] = q.x, v[1 % V] = q.y, v[2 % V] = q.z, v[3 % V] = q.w;
            ld_meta4(mb + 4 * i, pol, m[0], m[1 % V], m[2 % V], m[3 % V]);
        }
    };
    unsigned i = threadIdx.x;
    constexpr int U = (TC && !FIXED) ? (V == 1 ? 2 : 1) : UF;  // the FP64 tensor-core step needs more registers
    if (PIPE && FIXED) {
        // software-pipelined: the next U units' val/meta loads are in flight
        // while this step gathers x and adds, so the stream never waits on the
        // x gather and the add chain
        double v[U][V];
        unsigned mt[U][V];
        if (V * (i + (U - 1) * NT) < nent) {
#pragma unroll
            for (int u = 0; u < U; ++u) load(i + u * NT, v[u], mt[u]);
            for (;;) {
                const bool more = V * (i + (2 * U - 1) * NT) < nent;
                double vn[U][V], xv[U][V];
                unsigned mn[U][V];
                if (more) {
#pragma unroll
                    for (int u = 0; u < U; ++u) load(i + (U + u) * NT, vn[u], mn[u]);
                }
#pragma unroll
                for (int u = 0; u < U; ++u)
#pragma unroll
                    for (int k = 0; k < V; ++k) xv[u][k] = ld_policy(xb + (mt[u][k] >> rb), polx);
#pragma unroll
                for (int u = 0; u < U; ++u)
#pragma unroll
                    for (int k = 0; k < V; ++k) step(v[u][k], mt[u][k], xv[u][k]);
                i += U * NT;
                if (!more) break;
#pragma unroll
                for (int u = 0; u < U; ++u)
#pragma unroll
                    for (int k = 0; k < V; ++k) v[u][k] = vn[u][k], mt[u][k] = mn[u][k];
            }
        }
    } else {
        for (; V * (i + (U - 1) * NT) < nent; i += U * NT) {
            double v[U][V], xv[U][V];
            unsigned mt[U][V];
#pragma unroll
            for (int u = 0; u < U; ++u) load(i + u * NT, v[u], mt[u]);
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int k = 0; k < V; ++k) xv[u][k] = ld_policy(xb + (mt[u][k] >> rb), polx);
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int k = 0; k < V; ++k) step(v[u][k], mt[u][k], xv[u][k]);
        }
    }
    // tail: whole warps only (nent is a multiple of 32 V), so the TC steps stay full
    for (; V * (i - lane) < nent; i += NT) {
        double v[V], xv[V];
        unsigned mt[V];
        load(i, v, mt);
#pragma unroll
        for (int k = 0; k < V; ++k) xv[k] = ld_policy(xb + (mt[k] >> rb), polx);
#pragma unroll
        for (int k = 0; k < V; ++k) step(v[k], mt[k], xv[k]);
    }
}

// Re-sum listed rows in FP64 from the CSR, by threads [t, T) of the caller
// (T a multiple of 32): CUDA core, 4 lanes per row (lane c takes entries c,
// c + 4, ... in CSR order, then a fixed xor tree); tensor core, 8 rows per
// warp as the rows of an m8n8k4 A fragment (lane 4r+k holds A[r][k] = val and
// B[k][r] = x of row r's entry 4s+k at step s; D[r][r] accumulates row r, so
// the diagonal only meets its own row's operands and Inf/NaN propagate as in
// FP64).  Both orders are fixed: bit-reproducible.  Trip counts are uniform
// per warp (full-mask shuffles).
template <bool TC>
__device__ __forceinline__ void resum_rows(const int* __restrict__ list, unsigned n, const ColsortRun& run,
                                           const double* __restrict__ x, double* __restrict__ y, unsigned t,
                                           unsigned T) {
    const int lane = t & 31;
    if (!TC) {
        const int c = lane & 3;
        for (unsigned i0 = 0; i0 < n; i0 += T / 4) {
            const unsigned i = i0 + t / 4;
            double sum = 0.0;
            int r = -1;
            if (i < n) {
                r = __ldcg(list + i);
                const int a = __ldg(run.rp + r), e = __ldg(run.rp + r + 1);
                for (int j = a + c; j < e; j += 4)
                    sum = fma(__ldg(run.val + j), __ldg(x + (__ldg(run.col + j) - run.col_base)), sum);
            }
            sum += __shfl_xor_sync(0xffffffffu, sum, 1);
            sum += __shfl_xor_sync(0xffffffffu, sum, 2);
            if (c == 0 && r >= 0) y[r] = sum;
        }
    } else {
        const int r = lane >> 2, k = lane & 3;
        for (unsigned g = (t / 32) * 8; g < n; g += (T / 32) * 8) {
            const unsigned i = g + r;
            int a = 0, e = 0, row = -1;
            if (i < n) {
                row = __ldcg(list + i);
                a = __ldg(run.rp + row);
                e = __ldg(run.rp + row + 1);
            }
            int steps = (e - a + 3) >> 2;
#pragma unroll
            for (int o = 4; o < 32; o <<= 1) steps = max(steps, __shfl_xor_sync(0xffffffffu, steps, o));
            double d0 = 0.0, d1 = 0.0;
            for (int s = 0; s < steps; ++s) {
                const int j = a + 4 * s + k;
                double av = 0.0, bv = 0.0;
                if (j < e) {
                    av = __ldg(run.val + j);
                    bv = __ldg(x + (__ldg(run.col + j) - run.col_base));
                }
                dmma_m8n8k4(d0, d1, av, bv, d0, d1);
            }
            // D[r][r] sits on lane 4r + (r >> 1), element r & 1
            if (row >= 0 && k == (r >> 1)) y[row] = (r & 1) ? d1 : d0;
        }
    }
}

constexpr int kDefer = 4;  // blocks per CTA whose flagged rows wait for the CTA's end

template <bool TC, int NT, int UF, bool PIPE, int V>
__global__ void __launch_bounds__(NT, 2)
    spmv_colsort(const SpmvKBlock* __restrict__ blks, int b0, int b1, int rb, const double* __restrict__ val,
                 const unsigned* __restrict__ meta, const double* __restrict__ x, double* __restrict__ y,
                 ColsortRun run) {
    // shared: (rows + 1) doubles (FP64 mode) or the grid's low and high words
    // (2 (rows + 1) words, fixed-point mode) -- the same bytes
    extern __shared__ double ys[];
    __shared__ unsigned s_red[2][NT / 32];
    // fused flagged rows (run.fuse): a block's flagged rows are listed at
    // run.list[row0 ...] (room for every row of the block) and re-summed at the
    // CTA's end, so no barrier of a later block waits on them
    __shared__ unsigned s_fcnt, s_dcnt[kDefer], s_drow0[kDefer];
    const uint64_t pol = policy_evict_first(), polx = policy_evict_last();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int jb = 0;  // this CTA's blocks so far
    for (int b = b0 + blockIdx.x; b < b1; b += gridDim.x, ++jb) {
        const SpmvKBlock blk = blks[b];
        const unsigned stride = blk.rows + 1;
        unsigned* lo = reinterpret_cast<unsigned*>(ys);
        unsigned* hi = lo + stride;
        // the grid of the last call (plan creation: a guess from the block's
        // values with |x| < 1), checked against this call's products below
        int et = run.grid ? run.grid[b] : kColsortFp64;
        for (int pass = 0;; ++pass) {
            const int S = 62 - (int)blk.hl - et;
            const bool fixed = et != kColsortFp64 && S >= -1000 && S <= 1000;
            for (unsigned i = threadIdx.x; i < 2 * stride; i += NT) lo[i] = 0u;  // = stride doubles
            if (threadIdx.x == 0) s_fcnt = 0u;
            __syncthreads();
            unsigned mh = 0u, ml = 0u;
            if (fixed)
                block_entries<TC, true, true, NT, UF, PIPE, V>(ys, lo, hi, val + blk.e0, meta + blk.e0, x + blk.col_lo, blk.nent, rb,
                                              scalbn(1.0, S), pol, polx, mh, ml);
            else if (run.grid)
                block_entries<TC, false, true, NT, UF, PIPE, V>(ys, lo, hi, val + blk.e0, meta + blk.e0, x + blk.col_lo, blk.nent, rb,
                                               0.0, pol, polx, mh, ml);
            else
                block_entries<TC, false, false, NT, UF, PIPE, V>(ys, lo, hi, val + blk.e0, meta + blk.e0, x + blk.col_lo, blk.nent,
                                                rb, 0.0, pol, polx, mh, ml);
            if (run.grid) {  // block-wide largest |product| (with the Inf/NaN witness)
                mh = __reduce_max_sync(0xffffffffu, mh);
                ml = __reduce_or_sync(0xffffffffu, ml);
                if (lane == 0) s_red[0][warp] = mh, s_red[1][warp] = ml;
            }
            __syncthreads();
            if (run.grid) {
                mh = 0u;
                ml = 0u;
#pragma unroll 8
                for (int w = 0; w < NT / 32; ++w) mh = max(mh, s_red[0][w]), ml |= s_red[1][w];
            }
            // The grid the data calls for.  A fixed-point pass on another grid is
            // redone (too fine a grid may have wrapped, a coarser one rounds
            // differently), and so is an FP64 pass the data would allow on a
            // grid, so the result depends on the data alone.
            const int want = run.grid ? grid_of(mh, ml, fixed ? et : 0) : kColsortFp64;
            const bool again = pass < 2 && (fixed ? want != et : want != kColsortFp64);
            if (threadIdx.x == 0 && run.grid) run.grid[b] = want;
            if (!again) {
                if (fixed) {
                    // rows whose sum holds fewer than 45 + hl bits of the grid (it
                    // lies far below the block's largest product, or cancels) are
                    // summed again by the FP64 row kernel, so every row is within 2^-46 relative
                    const long long lim = 1ll << (45 + (int)blk.hl);
                    const double inv = scalbn(1.0, -S);
                    for (unsigned i = threadIdx.x; i < blk.rows; i += NT) {
                        const long long V = (long long)(((unsigned long long)hi[i] << 32) | lo[i]);
                        const bool flag = (mh | ml) != 0u && V > -lim && V < lim;
                        if (!flag) y[blk.row0 + i] = __ll2double_rn(V) * inv;
                        const unsigned am = __activemask();
                        const unsigned bal = __ballot_sync(am, flag);
                        if (bal) {
                            const int lead = __ffs(am) - 1;
                            unsigned base = 0;
                            if (lane == lead)
                                base = run.fuse ? atomicAdd(&s_fcnt, (unsigned)__popc(bal))
                                                : atomicAdd(run.count, (unsigned)__popc(bal));
                            base = __shfl_sync(am, base, lead);
                            if (flag)
                                run.list[(run.fuse ? blk.row0 : 0u) + base + __popc(bal & ((1u << lane) - 1))] =
                                    (int)(blk.row0 + i);
                        }
                    }
                } else {
                    for (unsigned i = threadIdx.x; i < blk.rows; i += NT) y[blk.row0 + i] = ys[i];
                }
                __syncthreads();
                if (run.fuse && fixed) {
                    if (jb < kDefer) {
                        if (threadIdx.x == 0) s_dcnt[jb] = s_fcnt, s_drow0[jb] = blk.row0;
                    } else {  // more blocks than the deferral slots: re-sum now
                        const unsigned nf = s_fcnt;
                        __syncthreads();  // every thread has nf before thread 0 resets s_fcnt for the next block
                        resum_rows<TC>(run.list + blk.row0, nf, run, x, y, threadIdx.x, NT);
                    }
                } else if (run.fuse && jb < kDefer && threadIdx.x == 0) {
                    s_dcnt[jb] = 0u;
                }
                break;
            }
            et = want;
            __syncthreads();
        }
    }
    if (run.fuse && run.grid) {
        __syncthreads();
        for (int j = 0; j < jb && j < kDefer; ++j)
            if (s_dcnt[j]) resum_rows<TC>(run.list + s_drow0[j], s_dcnt[j], run, x, y, threadIdx.x, NT);
    }
}

// The last CTA of a flagged-row kernel resets the list for the next call.
__device__ __forceinline__ void flagged_rows_done(const ColsortRun& run) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(run.done, 1u) == gridDim.x - 1) {
            *run.count = 0;
            *run.done = 0;
            __threadfence();
        }
    }
}

// The rows the fixed-point blocks handed over, summed in FP64 by 4 lanes each
// (lane c takes entries c, c+4, ... in CSR order, then a fixed xor tree:
// bit-reproducible); 8 rows per warp.  The list entry is read beside the
// count (the list has room for every row) to save one dependent load.  The
// last CTA to finish resets the count for the next call.
__global__ void __launch_bounds__(256) spmv_flagged_rows(ColsortRun run, const double* __restrict__ x,
                                                         double* __restrict__ y) {
    const int c = threadIdx.x & 3;
    const unsigned ng = gridDim.x * 64, g0 = blockIdx.x * 64 + (threadIdx.x >> 2);
    const int r0 = g0 < run.rows ? __ldcg(run.list + g0) : 0;
    const unsigned n = __ldcg(run.count);
    for (unsigned i0 = 0; i0 < n; i0 += ng) {  // uniform trip count per warp (full-mask shuffles)
        const unsigned i = i0 + g0;
        double sum = 0.0;
        int r = -1;
        if (i < n) {
            r = i0 == 0 ? r0 : __ldcg(run.list + i);
            const int a = __ldg(run.rp + r), e = __ldg(run.rp + r + 1);
            for (int j = a + c; j < e; j += 4)
                sum = fma(__ldg(run.val + j), __ldg(x + (__ldg(run.col + j) - run.col_base)), sum);
        }
        sum += __shfl_xor_sync(0xffffffffu, sum, 1);
        sum += __shfl_xor_sync(0xffffffffu, sum, 2);
        if (c == 0 && r >= 0) y[r] = sum;
    }
    flagged_rows_done(run);
}

// Tensor-core form of the flagged-row kernel: a warp takes 8 listed rows as
// the rows of an m8n8k4 A fragment, lane 4r+k holding A[r][k] = val and
// B[k][r] = x of row r's entry 4s+k at step s; D[r][r] accumulates row r in
// the MMA (a fixed order: bit-reproducible).  Off-diagonal outputs mix rows
// and are dropped; the diagonal only ever meets its own row's operands, so
// Inf/NaN propagate as in FP64.
__global__ void __launch_bounds__(256) spmv_flagged_rows_tc(ColsortRun run, const double* __restrict__ x,
                                                            double* __restrict__ y) {
    const int lane = threadIdx.x & 31, r = lane >> 2, k = lane & 3;
    const unsigned warps = gridDim.x * 8, w0 = blockIdx.x * 8 + (threadIdx.x >> 5);
    const unsigned n = __ldcg(run.count);
    for (unsigned g = w0 * 8; g < n; g += warps * 8) {  // warp-uniform
        const unsigned i = g + r;
        int a = 0, e = 0, row = -1;
        if (i < n) {
            row = __ldcg(run.list + i);
            a = __ldg(run.rp + row);
            e = __ldg(run.rp + row + 1);
        }
        int steps = (e - a + 3) >> 2;
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) steps = max(steps, __shfl_xor_sync(0xffffffffu, steps, o));
        double d0 = 0.0, d1 = 0.0;
        for (int s = 0; s < steps; ++s) {
            const int j = a + 4 * s + k;
            double av = 0.0, bv = 0.0;
            if (j < e) {
                av = __ldg(run.val + j);
                bv = __ldg(x + (__ldg(run.col + j) - run.col_base));
            }
            dmma_m8n8k4(d0, d1, av, bv, d0, d1);
        }
        // D[r][r] sits on lane 4r + (r >> 1), element r & 1
        if (row >= 0 && k == (r >> 1)) y[row] = (r & 1) ? d1 : d0;
    }
    flagged_rows_done(run);
}

// Order the entries of one window so that each aligned group of g takes one
// entry from as many distinct row % g classes as the window has, largest
// classes first: g = 16 for FP64 rows (a half-warp of 64-bit accesses, bank
// pairs), g = 32 for the fixed-point grid's 32-bit words (a warp, banks).
void bank_order(std::vector<std::pair<uint64_t, double>>& t, size_t w0, size_t w1, unsigned rmask, int g,
                std::vector<std::pair<uint64_t, double>>& out) {
    std::vector<std::pair<uint64_t, double>> cls[32];
    for (size_t i = w0; i < w1; ++i) cls[(t[i].first & rmask) % g].push_back(t[i]);
    size_t left = w1 - w0;
    out.clear();
    while (left) {
        int order[32];
        for (int c = 0; c < g; ++c) order[c] = c;
        std::stable_sort(order, order + g, [&](int a, int b) { return cls[a].size() > cls[b].size(); });
        int taken = 0;
        for (int oi = 0; oi < g && left; ++oi) {
            auto& c = cls[order[oi]];
            if (c.empty()) continue;
            out.push_back(c.back());
            c.pop_back();
            --left;
            ++taken;
        }
        while (taken < g && left) {  // fewer than g classes left: conflicts unavoidable
            int big = 0;
            for (int c = 1; c < g; ++c)
                if (cls[c].size() > cls[big].size()) big = c;
            out.push_back(cls[big].back());
            cls[big].pop_back();
            --left;
            ++taken;
        }
    }
    std::copy(out.begin(), out.end(), t.begin() + w0);
}
// vec > 1: a warp step's 32 vec entries go to vec shared-atomic instructions
// of 32 (entry parity = the lane's k-th entry).  Which entry takes which
// (parity, lane) slot changes neither the bytes nor the x lines the step
// reads, so the host deals each row % 32 bank class over the parities: a
// parity's 32 atomics then meet fewer repeated banks (random rows: ~3.5
// wavefronts per instruction before).  Entry of (parity p, lane j) goes to
// position g0 + vec j + p.
void spread_banks(std::vector<std::pair<uint64_t, double>>& t, size_t g0, int vec, unsigned rmask,
                  std::vector<std::pair<uint64_t, double>>& out) {
    std::vector<std::pair<uint64_t, double>> cls[32];
    const size_t n = 32 * (size_t)vec;
    for (size_t i = g0; i < g0 + n; ++i) cls[(t[i].first & rmask) & 31].push_back(t[i]);
    int order[32];
    for (int c = 0; c < 32; ++c) order[c] = c;
    std::stable_sort(order, order + 32, [&](int a, int b) { return cls[a].size() > cls[b].size(); });
    int fill[4] = {0, 0, 0, 0};
    out.assign(n, {0, 0.0});
    for (int oi = 0; oi < 32; ++oi) {
        int used[4] = {0, 0, 0, 0};  // this class's entries per parity so far
        for (auto& e : cls[order[oi]]) {
            // the parity this class has used least, then the one with the most room
            int best = -1;
            for (int q = 0; q < vec; ++q)
                if (fill[q] < 32 && (best < 0 || used[q] < used[best] || (used[q] == used[best] && fill[q] < fill[best])))
                    best = q;
            out[(size_t)vec * fill[best] + best] = e;
            ++fill[best];
            ++used[best];
        }
    }
    std::copy(out.begin(), out.end(), t.begin() + g0);
}
}  // namespace

bool spmv_colsort_build(uint64_t m, uint64_t n, const int32_t* rp, const int32_t* col, const double* val,
                        SpmvColsortLayout& L, const std::vector<ColsortSegment>& segments_in, int classes,
                        bool tc_lanes, int vec) {
    vec = (vec == 2 || vec == 4) ? vec : 1;
    (void)n;
    if (m == 0 || rp[m] == 0) return false;
    int64_t maxlen = 0;
    for (uint64_t i = 0; i < m; ++i) maxlen = std::max<int64_t>(maxlen, (int64_t)rp[i + 1] - rp[i]);
    if (maxlen > kColsortMaxRowLen) return false;  // one hot row would serialise its block's atomics
    // Default: one segment of two waves of two CTAs per SM (tools/micro/spmv_colsort.cu: 2 waves 0.173 ms,
    // 3 waves 0.191 ms at 2^22 rows).  Each segment's rows are cut into `blocks` equal blocks of at most
    // kColsortMaxRows (64 KB of y); all blocks are halved while a block's column span does not fit the
    // meta word.
    std::vector<ColsortSegment> segs = segments_in;
    if (segs.empty()) segs.push_back({m, 4 * (uint64_t)kNumSMsHost});
    for (int halve = 0;; ++halve) {
        std::vector<std::pair<uint64_t, uint64_t>> cut;  // (row0, rows)
        uint64_t seg0 = 0, Rmax = 1;
        for (const auto& sg : segs) {
            const uint64_t len = std::min(sg.row_end, m) - std::min(seg0, m);
            if (len) {
                uint64_t R = (len + sg.blocks - 1) / std::max<uint64_t>(1, sg.blocks);
                R = std::max<uint64_t>(32, std::min<uint64_t>(R, kColsortMaxRows)) >> halve;
                if (R < 1) return false;
                for (uint64_t r = seg0; r < seg0 + len; r += R) cut.push_back({r, std::min(R, seg0 + len - r)});
                Rmax = std::max(Rmax, R);
            }
            seg0 = std::max(seg0, std::min(sg.row_end, m));
        }
        if (seg0 < m || Rmax < 8) return false;
        int rb = 0;  // row field: 0..R (R = the padding's scratch slot)
        while ((1ull << rb) <= Rmax) ++rb;
        const uint64_t nb = cut.size();
        bool fits = true;
        for (uint64_t b = 0; b < nb && fits; ++b) {
            const uint64_t r0 = cut[b].first, r1 = r0 + cut[b].second;
            int32_t lo = INT32_MAX, hi = INT32_MIN;
            for (int64_t j = rp[r0]; j < rp[r1]; ++j) lo = std::min(lo, col[j]), hi = std::max(hi, col[j]);
            if (hi >= lo && (uint64_t)(hi - lo) >= (1ull << (32 - rb))) fits = false;
        }
        if (!fits) continue;
        L.rb = rb;
        L.rows = (int)Rmax;
        L.vec = vec;
        L.blocks.assign(nb, SpmvKBlock{});
        uint64_t e = 0;
        for (uint64_t b = 0; b < nb; ++b) {
            const uint64_t r0 = cut[b].first, r1 = r0 + cut[b].second;
            const uint64_t cnt = (uint64_t)(rp[r1] - rp[r0]);
            SpmvKBlock& k = L.blocks[b];
            k.e0 = e;
            k.row0 = (uint32_t)r0;
            k.rows = (uint32_t)(r1 - r0);
            const uint64_t gsz = 32 * (uint64_t)vec;  // a warp step's entries
            k.nent = (uint32_t)((cnt + gsz - 1) / gsz * gsz);
            int32_t lo = INT32_MAX;
            int ev = 0;
            bool nonfinite = false;
            for (int64_t j = rp[r0]; j < rp[r1]; ++j) {
                lo = std::min(lo, col[j]);
                uint64_t bits;
                std::memcpy(&bits, &val[j], 8);
                const int f = (int)((bits >> 52) & 0x7FF);
                if (f == 0x7FF) nonfinite = true;
                else ev = std::max(ev, f);
            }
            k.col_lo = cnt ? lo : 0;
            k.ev = (int16_t)ev;
            k.flags = nonfinite ? 1 : 0;
            int64_t mlen = 0;
            for (uint64_t r = r0; r < r1; ++r) mlen = std::max<int64_t>(mlen, (int64_t)rp[r + 1] - rp[r]);
            int hl = 0;
            while ((1ll << hl) < mlen) ++hl;  // a row sums <= 2^hl products: |V| <= 2^62
            k.hl = (uint8_t)hl;
            e += k.nent;
        }
        L.val.assign(e, 0.0);
        L.meta.assign(e, 0u);
        const unsigned rmask = (1u << rb) - 1;
        auto work = [&](uint64_t bfirst, uint64_t bstep) {
            std::vector<std::pair<uint64_t, double>> t, scratch;
            for (uint64_t b = bfirst; b < nb; b += bstep) {
                const SpmvKBlock& k = L.blocks[b];
                const uint64_t r0 = k.row0, r1 = r0 + k.rows;
                t.clear();
                for (uint64_t r = r0; r < r1; ++r)
                    for (int64_t j = rp[r]; j < rp[r + 1]; ++j)
                        t.push_back({((uint64_t)(col[j] - k.col_lo) << rb) | (r - r0), val[j]});
                std::sort(t.begin(), t.end(), [](const auto& a, const auto& c) { return a.first < c.first; });
                const size_t win = (size_t)std::max(32, tuning().spmv_colsort_window);
                const int g = std::min(32, std::max(1, classes));
                for (size_t w0 = 0; g > 1 && w0 < t.size(); w0 += win)
                    bank_order(t, w0, std::min(t.size(), w0 + win), rmask, g, scratch);
                while (t.size() < k.nent) t.push_back({k.rows, 0.0});  // padding: column col_lo, scratch row
                if (vec > 1 && tuning().spmv_colsort_spread == 1)
                    for (size_t g0 = 0; g0 < t.size(); g0 += 32 * vec) spread_banks(t, g0, vec, rmask, scratch);
                if (vec > 1 && tuning().spmv_colsort_spread == 2)  // halves: parity p = sorted entries [32p, 32p + 32)
                    for (size_t g0 = 0; g0 < t.size(); g0 += 32 * vec) {
                        scratch.assign(t.begin() + g0, t.begin() + g0 + 32 * vec);
                        for (int j = 0; j < 32; ++j)
                            for (int par = 0; par < vec; ++par) t[g0 + vec * j + par] = scratch[32 * par + j];
                    }
                if (!tc_lanes) {
                    for (size_t i = 0; i < t.size(); ++i) {
                        L.meta[k.e0 + i] = (uint32_t)t[i].first;
                        L.val[k.e0 + i] = t[i].second;
                    }
                } else {
                    // each 32-entry group in the tensor-core roles: value in its A
                    // slot, column bits in its B slot, row bits in its output lane
                    // (vec = 2: a lane's two entries sit side by side, so the warp
                    // step's even and odd entries are two such groups)
                    for (size_t g = 0; g < t.size(); g += 32 * vec)
                        for (int par = 0; par < vec; ++par)
                            for (int la = 0; la < 32; ++la) {
                                int lb, ld;
                                tc_roles(la, lb, ld);
                                const uint64_t key = t[g + vec * la + par].first;
                                L.val[k.e0 + g + vec * la + par] = t[g + vec * la + par].second;
                                L.meta[k.e0 + g + vec * lb + par] |= (uint32_t)(key & ~(uint64_t)rmask);
                                L.meta[k.e0 + g + vec * ld + par] |= (uint32_t)(key & rmask);
                            }
                }
            }
        };
        const unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
        std::vector<std::thread> pool;
        for (unsigned i = 1; i < nt; ++i) pool.emplace_back(work, i, nt);
        work(0, nt);
        for (auto& th : pool) th.join();
        return true;
    }
}

int colsort_initial_grid(const SpmvKBlock& k) {
    if (k.flags & 1) return kColsortFp64;
    const int ea = std::max((int)k.ev, 1) - 1022;  // |x| < 1 assumed: |p| < 2^(ev - 1023 + 1)
    return (ea >= 0 ? (ea + kColsortQuantum - 1) / kColsortQuantum : -((-ea) / kColsortQuantum)) * kColsortQuantum;
}

template <bool TC, int NT, int UF, bool PIPE, int V>
cudaError_t launch_main(const SpmvKBlock* blks, int b0, int b1, int rb, size_t smem, const double* val,
                        const unsigned* meta, const double* x, double* y, const ColsortRun& run, cudaStream_t s) {
    const cudaError_t e =
        cudaFuncSetAttribute(spmv_colsort<TC, NT, UF, PIPE, V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    spmv_colsort<TC, NT, UF, PIPE, V>
        <<<std::min(b1 - b0, 2 * kNumSMs), NT, smem, s>>>(blks, b0, b1, rb, val, meta, x, y, run);
    return cudaSuccess;
}

// CTA shape codes (tuning spmv_colsort_{cc,tc}_shape): threads x units per
// step, plain or software-pipelined loop; V = 2 layouts (entries paired per
// thread) take the V = 2 instantiations of the same shapes.
template <bool TC, int V>
cudaError_t launch_shape(int shape, const SpmvKBlock* blks, int b0, int b1, int rb, size_t smem, const double* val,
                         const unsigned* meta, const double* x, double* y, const ColsortRun& run, cudaStream_t s) {
    switch (shape) {
        case 7: return launch_main<TC, 640, 3, true, V>(blks, b0, b1, rb, smem, val, meta, x, y, run, s);
        case 8: return launch_main<TC, 512, 4, true, V>(blks, b0, b1, rb, smem, val, meta, x, y, run, s);
        case 10: return launch_main<TC, 1024, 1, false, V>(blks, b0, b1, rb, smem, val, meta, x, y, run, s);
        case 11: return launch_main<TC, 512, 2, true, V>(blks, b0, b1, rb, smem, val, meta, x, y, run, s);
        case 13: return launch_main<TC, 768, 1, true, V>(blks, b0, b1, rb, smem, val, meta, x, y, run, s);
        case 16: return launch_main<TC, 512, 1, true, V>(blks, b0, b1, rb, smem, val, meta, x, y, run, s);
        default: return launch_main<TC, kThreads, kUnroll, false, V>(blks, b0, b1, rb, smem, val, meta, x, y, run, s);
    }
}

cudaError_t launch_spmv_colsort(int unit, int vec, const SpmvKBlock* blks, int b0, int b1, int rb, int rows,
                                const double* val, const unsigned* meta, const double* x, double* y,
                                const ColsortRun& run, cudaStream_t s) {
    if (b1 <= b0) return cudaSuccess;
    const size_t smem = (size_t)(rows + 1) * 8;
    const int cs = tuning().spmv_colsort_cc_shape, ts = tuning().spmv_colsort_tc_shape;
    cudaError_t e = vec == 4
        ? (unit ? launch_shape<true, 4>(ts, blks, b0, b1, rb, smem, val, meta, x, y, run, s)
                : launch_shape<false, 4>(cs, blks, b0, b1, rb, smem, val, meta, x, y, run, s))
        : vec == 2
        ? (unit ? launch_shape<true, 2>(ts, blks, b0, b1, rb, smem, val, meta, x, y, run, s)
                : launch_shape<false, 2>(cs, blks, b0, b1, rb, smem, val, meta, x, y, run, s))
        : (unit ? launch_shape<true, 1>(ts, blks, b0, b1, rb, smem, val, meta, x, y, run, s)
                : launch_shape<false, 1>(cs, blks, b0, b1, rb, smem, val, meta, x, y, run, s));
    if (e != cudaSuccess) return e;
    note_launch();
    if ((e = cudaGetLastError()) != cudaSuccess || !run.grid) return e;
    if (run.fuse) return cudaSuccess;  // flagged rows re-summed inside the main kernel
    if (unit) spmv_flagged_rows_tc<<<2 * kNumSMs, 256, 0, s>>>(run, x, y);
    else spmv_flagged_rows<<<2 * kNumSMs, 256, 0, s>>>(run, x, y);
    note_launch();
    return cudaGetLastError();
}

}  // namespace rlb
