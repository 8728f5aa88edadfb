// kernels.h -- host-side launch interface of the sm_100a kernels (internal).
// The C-ABI (capi.cpp) validates arguments, then calls these.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include <vector>

namespace rlb {

// Kernel-variant knobs, settable through rl_tuning_set() for sweeps.
struct Tuning {
    int dist_graph = 1;            // rl_dist_* plans replay captured CUDA graphs after the first call
    int scale_blocks_per_sm = 32;  // STREAM grid = 148 * this (swept: tools/sweep.py)
    int scale_unroll = 8;          // 1, 2, 4, 8
    int gemv_rows = 4;             // rows per warp, CUDA-core GEMV (2, 4, 8)
    int gemv_unroll = 2;           // 128-column steps in flight per iteration (1, 2, 4)
    int spmv_rows = 2;             // rows per lane group per iteration (1, 2, 4)
    int spmv_blocks_per_sm = 1;    // CUDA-core SpMV grid = 148 * this
    int spmv_threads = 1024;       // CTA size of the CUDA-core kernel (multiple of 32, <= 1024)
    int spmv_tc_blocks_per_sm = 1; // tensor-core SpMV grid = 148 * this
    int spmv_tc_threads = 1024;
    int spmv_l1_carveout = -1;     // shared-memory carveout % for the CC kernel (-1 = driver default)
    int spmv_tc_rows = 1;          // 8-row blocks per warp iteration (1, 2)
    int spmv_long_rows = 1;        // divert long rows of the CSR kernels to a load-balanced second kernel
    int spmv_long_min = 64;        // ... rows longer than this many nonzeros
    int spmv_long_piece = 512;     // ... cut into pieces of this many nonzeros, balanced over the warps
    int spmv_long_group = 8;       // lanes per piece of the CUDA-core long-row kernel (8, 16, 32)
    int spmv_plan_chunks = 16;     // pipelined row/x chunks of rl_spmv_plan_execute_host
    int spmv_plan_streams = 1;     // compute streams of a column-sorted plan's execute_host (1: 1.02 ms, 4-8: 1.10 ms; tools/micro/plan_colsort_e2e.py)
    int spmv_plan_colsort_chunks = 8;  // pipeline chunks of a column-sorted plan (8: 1.02, 16: 1.21-1.26, 32: 1.36+ ms)
    int spmv_colsort_window = 128; // K17 plan build: entries per bank-ordering window (tools/micro/spmv_colsort.cu: 64 0.185, 128 0.183 ms)
    int stencil_tb27r = 1;         // 3d27pt t = 2 (class weights): the register-blocked kernel (stencil_tb27r.cu); 0: z-column
    int spmv_colsort_classes = 0;  // K17 bank-ordering group 1..32 (0: 1 = none on the fixed-point grid, 16 for FP64 rows)
    int spmv_colsort_fixed = 2;    // K17 rows on a 64-bit fixed-point grid (+ FP64 row kernel for flagged rows):
                                   // 1 CUDA-core unit only, 2 both units, 0 neither (FP64 shared atomics)
    int spmv_plan_colsort_blocks = 0; // K17 plan: row blocks over all rows (0: 4 x 148)
    int spmv_plan_dev_chunks = 0;     // developer probe: rl_spmv_plan_execute runs the execute_host chunks one by one
    int spmv_plan_probe_nocompute = 0; // developer probe: execute_host moves x and y but launches no kernel
    int spmv_plan_edge_blocks = 0;    // K17 plan: blocks of the first / last execute_host chunk each (0: uniform blocks)
    int spmv_colsort_fuse = 1;     // K17: flagged rows re-summed at each CTA's end inside the main kernel (0: a separate row kernel)
    int spmv_colsort_spread = 2;   // K17 plan build (vec > 1), which entries of a warp step share an instruction (parity):
                                   // 2 contiguous halves of the sorted step (fewest x lines per gather: CC 0.1604 vs 0.1652 ms),
                                   // 1 each bank class dealt over the parities, 0 alternate entries
    int spmv_colsort_vec = 4;      // K17 plan build: entries per thread unit (4: 256-bit val / 128-bit meta loads; 2: 128 / 64; 1)
    int spmv_colsort_tc_shape = 16; // K17 CTA shape (threads x units per step; p = software-pipelined loop):
                                    // 0 1024x3, 10 1024x1; p: 7 640x3, 8 512x4, 11 512x2, 13 768x1, 16 512x1
                                    // (tools/micro/spmv_shapes.py, 60 interleaved bursts of 25 calls, medians:
                                    // TC vec 4 shape 16 0.2014 ms, vec 2 13 0.2020; earlier vec 2 11 0.194 vs
                                    // 13 0.186, vec 1 0 0.222, vec 1 7 0.225; shapes 1 768x3, 4 1024x2,
                                    // 5 1024x1p, 6 768x2p, 12 640x2p, 14 512x3p, 15 384x4p measured no better)
    int spmv_colsort_cc_shape = 10; // ... CUDA-core kernel (vec 4 10 0.1542, vec 4 16 0.1586, vec 2 11 0.1620 ms)
    int spmv_plan_colsort = 1;     // plans (both units) use the column-sorted row-block layout (K17, spmv_colsort.cu) when eligible; 0: CSR
    int spmv_plan_xpieces = 0;     // max x upload pieces (first = chunk 0's prefix); 0: one per chunk
    int spmv_plan_ygroups = 0;     // y download copies (groups of consecutive chunks); 0: one per chunk
    int spmv_plan_taper = 0;       // 1: half-size first/last pipeline chunks (measured no gain)
    int spmv_plan_graph = 1;       // execute_host with pinned x/y as one captured CUDA graph
    int spmv_plan_zero_copy = 0;   // 1: store y straight into pinned host memory (measured slower)
    int spmv_sched = 1;            // 0 grid-stride, 1 contiguous row range per CTA
    int spmv_xhint = 0;            // x gathers: 0 L1 default, 1 L1::evict_last, 2 L1::no_allocate
    int stencil2d_rows = 256;      // rows marched per warp (2D CC)
    int stencil3d_zchunk = 64;     // planes marched per CTA (3D, non-TMA fallback)
    int tc_stencil_zchunk = 32;
    int stencil_tma = 1;           // 1: TMA-pipelined kernels when eligible
    int stencil_ctas_per_sm = 1;   // grid sizing target, TMA CUDA-core kernels
    int stencil_rows_per_thread = 0;   // 3D TMA CUDA-core kernels: 2, 4 or 8 (CTA = 64*16/this threads); 0 = per preset
    int stencil2d_rows_per_thread = 4; // 2D TMA CUDA-core kernel (swept: tools/sweep.py)
    int stencil_cc27x2 = 1;            // 3d27pt CC class weights: two columns per thread kernel
    int stencil_tc_concat = 1;         // 3d27pt TC one-plane: class products concatenated along K (10 DMMA/tile)
    int stencil3d_cc_stages = 4;       // 3D CUDA-core TMA ring depth (4, 6, 8)
    int stencil_tc_ctas_per_sm = 2;    // ... 2D tensor-core kernel (2: +3 % measured over 1)
    int stencil_tc3d_ctas_per_sm = 8;  // ... 3D tensor-core kernels (3-plane mode)
    int stencil_tc3d_mode = 2;         // 3D tensor core, one-plane partial-sum kernel for: bit0 3d7pt, bit1 3d27pt
    int stencil_tc1_ctas_per_sm = 8;   // ... partial-sum mode
    int stencil_tc3d_hybrid = 1;       // 3D tensor core: x-band on DMMA, centre/y/z on DFMA (st3d_tma_tch, 3 DMMA/tile); 3d7pt and class-weight 3d27pt
    int stencil_tch_ctas_per_sm = 0;   // ... grid sizing of that kernel (0: per preset, 3d7pt 1 = one z-front, 3d27pt 16)
    int stencil_tch_tpw = 0;           // ... 8x8 tiles per warp: 4 (128-thread CTAs), 2 (256), 1 (512); 0: per preset (3d7pt 2, 3d27pt 4)
    int stencil_tc2d_hybrid = 1;       // 2d5pt tensor core: x-band on DMMA, centre/y on DFMA (st2d_tma_tch, 3 DMMA/tile); 0: 6 DMMA/tile
    int stencil3d_balance = 1;         // 3D TMA kernels with one z-front: rows cut into tiles of <= 16 so the SMs hold equal rows
    int stencil_tch_stages = 4;        // ... TMA ring depth (4 or 6; 6 measured 7-9 % slower)
    int stencil_tch_k8 = 0;            // ... 1: K = 8 band window (2 DMMA/tile, two x+1 taps by shuffle + DFMA; measured no faster); 0: K = 12, 3 DMMA
    int stencil_r_cc_stages = 0;       // ... CUDA-core ring depth: 2-4, 0 = auto (2 for 2d49pt -> 4 CTAs/SM, else 4)
    int stencil_r_tc_stages = 0;       // TMA ring stages of the radius-R tensor-core kernels (0: 2 at radius 3, else 4)
    int stencil_r_ctas_per_sm = 32;
    int stencil_tb_waves = 4;          // register temporal blocking: grid = this many waves of resident warps
    int stencil_tb_tma = 4;            // 2d5pt depth >= this streams rows through a per-warp TMA ring (0: never; register queue)
    int stencil_tb3_shape = 0;         // stencil_tb3r rows per warp x warps: 0/1 4x8, 2 2x16, 3 4x16 (t=2)
    int stencil_tb3_chunks = 0;        // z chunks per tile for stencil_tb3r (0: auto)
    int stencil_tb3_l2promo = 2;       // TMA L2 promotion of the stencil_tb3r boxes (0 none .. 3 256 B)
    int stencil_r_l2promo = 1;         // ... TMA L2 promotion (0 none, 1 64 B, 2 128 B, 3 256 B)
    int stencil_r_sym = 1;             // 2d49pt CC: pair mirror-symmetric columns (fewer FP64 ops)    // 2d9pt/2d13pt/2d49pt TMA kernels: row segments so the grid is this deep
};
Tuning& tuning();
// whether a K17 layout for this unit accumulates on the fixed-point grid
inline bool colsort_fixed_for(bool tc) {
    const int f = tuning().spmv_colsort_fixed;
    return f == 2 || (f == 1 && !tc);
}

struct StencilDesc {
    int preset;          // see StencilPreset
    int dim;             // 2 or 3
    int radius;
    int npts;
    uint64_t nx, ny, nz; // nz = 1 for 2D
    double w[49];        // canonical offset order
};

enum StencilPreset : int {
    kP2d5 = 0, kP2d9 = 1, kP2d13 = 2, kP2d49 = 3, kP3d7 = 4, kP3d27 = 5
};

cudaError_t launch_scale(int unit, double* a, const double* b, double q, uint64_t n,
                         cudaStream_t s);
// Long-row diversion state of one SpMV launch (spmv.cu): rows longer than
// lmax leave the per-row kernel; each is cut into ceil(len / piece) pieces of
// at most `piece` nonzeros and appended to the list with its first global
// piece number (one 64-bit atomic: list index << 38 | pieces so far, so
// base[] ascends with the index).  spmv_long then hands every warp an equal
// run of pieces.  ctr[0..1] is that 64-bit counter, ctr[2] the exit count.
// ctr == nullptr: off.
struct LongRows {
    unsigned* ctr;
    int* rows;       // diverted rows (list order)
    unsigned* base;  // first global piece of each listed row (ascending)
    double* part;    // partial sums of split rows, by global piece (pcap)
    unsigned* done;  // per listed row: pieces finished
    int64_t lmax;
    int64_t piece;
    uint64_t pcap;
    bool vec;        // val 32-byte and col 16-byte aligned: vector loads allowed
};
constexpr int kLongIndexShift = 38;
// long_rows: -1 unknown (divert on the device), 0 known absent (no
// diversion), 1 known present.
cudaError_t launch_spmv(int unit, uint64_t r0, uint64_t r1, const int* rp, const int* col,
                        const double* val, const double* x, int64_t col_base, double* y,
                        int long_rows, cudaStream_t s);
cudaError_t launch_spmv_rows(int unit, uint64_t r0, uint64_t r1, const int* rp, const int* col,
                             const double* val, const double* x, int64_t col_base, double* y,
                             const LongRows& lr, cudaStream_t s);
// Per-(device, stream) diversion buffers for `rows` rows; allocates (outside
// stream capture) on first use or growth.
cudaError_t spmv_long_workspace(cudaStream_t s, uint64_t rows, LongRows& lr);
// One sweep over outer indices [o0, o1) (already clipped to the interior).
cudaError_t launch_stencil_cc(const StencilDesc& d, uint64_t o0, uint64_t o1, const double* u,
                              double* v, cudaStream_t s);
cudaError_t launch_stencil_tc(const StencilDesc& d, uint64_t o0, uint64_t o1, const double* u,
                              double* v, cudaStream_t s);

// TMA-pipelined stencils (2d5pt, 3d7pt, 3d27pt; even nx, 16-byte aligned).
bool stencil_tma_eligible(const StencilDesc& d, const double* u, const double* v);
cudaError_t launch_stencil_tma(int unit, const StencilDesc& d, uint64_t o0, uint64_t o1,
                               const double* u, double* v, cudaStream_t s);

// TMA 2D stencils of the other presets (2d9pt, 2d13pt, 2d49pt; stencil_r.cu).
bool stencil_r_eligible(const StencilDesc& d, const double* u, const double* v);
cudaError_t launch_stencil_r(int unit, const StencilDesc& d, uint64_t o0, uint64_t o1, const double* u,
                             double* v, cudaStream_t s);
// 2D FP64 tensor map (box_x x box_y, zero OOB fill) into a 64-byte-aligned
// CUtensorMap; false when the driver entry point is missing.
bool tma_encode_available();
bool encode_map_2d(void* map, const double* base, uint64_t nx, uint64_t ny, uint32_t box_x, uint32_t box_y,
                   int l2_promotion = 3);  // 0 none, 1 64 B, 2 128 B, 3 256 B
// 3D FP64 tensor map (box_x x box_y x 1), same conventions.
bool encode_map_3d(void* map, const double* base, uint64_t nx, uint64_t ny, uint64_t nz, uint32_t box_x,
                   uint32_t box_y, int l2_promotion = 3);

// 2d5pt with temporal depth t (2..8) in registers (stencil_tb.cu).
bool stencil_tb_supported(const StencilDesc& d, int t, const double* u, const double* v);
cudaError_t launch_stencil_tb(const StencilDesc& d, int t, uint64_t o0, uint64_t o1, const double* u, double* v,
                              cudaStream_t s);

// 3d7pt with temporal depth t (2..4): z-marching register pipeline (stencil_tb3.cu).
bool stencil_tb3_supported(const StencilDesc& d, int t);
cudaError_t launch_stencil_tb3(const StencilDesc& d, int t, uint64_t o0, uint64_t o1, const double* u, double* v,
                               cudaStream_t s);
// 3d7pt with temporal depth t (2..4), register-blocked and skewed: TMA plane
// tiles, one barrier per input plane (stencil_tb3r.cu).  Needs an even nx
// and 16-byte aligned u / v.
// 2d5pt temporal blocking on the tensor core (stencil_tbtc.cu): overlapped
// 64 x 64 tiles in shared memory, each level the x-band-on-DMMA form; one
// launch = one fused sweep of t timesteps over the interior (t = 2..4).
bool stencil_tbtc_supported(const StencilDesc& d, int t, const double* u, const double* v);
cudaError_t launch_stencil_tbtc(const StencilDesc& d, int t, const double* u, double* v, cudaStream_t s);
// 3d27pt (class weights), temporal depth 2, register-blocked (stencil_tb27r.cu).
bool stencil_tb27r_supported(const StencilDesc& d, int t, const double* u, const double* v);
cudaError_t launch_stencil_tb27r(const StencilDesc& d, int t, uint64_t o0, uint64_t o1, const double* u, double* v,
                                 cudaStream_t s);
bool stencil_tb3r_supported(const StencilDesc& d, int t, const double* u, const double* v);
cudaError_t launch_stencil_tb3r(const StencilDesc& d, int t, uint64_t o0, uint64_t o1, const double* u, double* v,
                                cudaStream_t s);

// Dense GEMV y = A*x, row-major A (m x n).
cudaError_t launch_gemv(int unit, uint64_t m, uint64_t n, const double* A, const double* x, double* y,
                        cudaStream_t s);

// Distributed SpMV plan create-time check (dist_kernels.cu): out[0] = widest
// |col - row|, out[1] = columns outside [0, n), out[2] = decreasing row_ptr
// entries (device buffer of 3 u64).
cudaError_t launch_band_check(uint64_t rows, const int* rp, const int* col, int64_t row0, int64_t n,
                              unsigned long long* out, cudaStream_t s);
// Longest-row probe of the CSR kernels' long-row diversion (spmv.cu), for
// callers that must decide before a stream capture: 1 when [r0, r1) has rows
// the per-row kernels divert, 0 when not, -1 when the probe failed.
int spmv_long_rows_probe(const int* rp, const int* col, const double* val, uint64_t r0, uint64_t r1,
                         cudaStream_t s);

constexpr int kNumSMsHost = 148;  // B200 SM count (host-side copy of common.cuh's kNumSMs)

// K17: column-sorted row-block layout (spmv_colsort.cu), the default layout
// of CUDA-core SpMV plans when eligible (rows <= kColsortMaxRowLen nonzeros;
// every block's column span fits the meta word).
constexpr int kColsortMaxRows = 8192;     // rows per block (y in shared memory: 64 KB, two CTAs per SM)
constexpr int kColsortMaxRowLen = 1024;   // longer rows stay on the CSR kernels (long-row path)
struct SpmvKBlock {
    uint64_t e0;     // first entry
    int32_t col_lo;  // smallest column of the block
    uint32_t row0;   // first row
    uint32_t rows;   // rows (<= kColsortMaxRows)
    uint32_t nent;   // entries, padded to a multiple of 32
    int16_t ev;      // largest IEEE exponent field of the block's finite values
    uint8_t hl;      // the longest row has <= 2^hl entries
    uint8_t flags;   // bit 0: a value is Inf/NaN
};
constexpr int kColsortQuantum = 8;         // grid exponents are multiples of this
constexpr int kColsortFp64 = -0x40000000;  // grid code: the block adds in FP64 (shared CAS atomics)
// Fixed-point mode state (null grid: FP64 atomics only): the per-block grid
// exponents of the last call, the rows handed to the FP64 row kernel, and the
// CSR that kernel sums them from (columns minus col_base index x).
struct ColsortRun {
    int* grid;
    int* list;        // capacity: `rows`
    unsigned* count;  // entries in `list` (reset by the row kernel)
    unsigned* done;   // CTAs of the row kernel finished (reset by its last CTA)
    unsigned rows;
    const int* rp;
    const int* col;
    const double* val;
    int64_t col_base;
    int fuse;  // 1: the main kernel re-sums its flagged rows (list indexed by block row0; no row kernel)
};
int colsort_initial_grid(const SpmvKBlock& k);
struct SpmvColsortLayout {
    int rb = 0;    // row bits of meta
    int rows = 0;  // rows of the largest block (shared-memory y per CTA)
    int vec = 1;   // entries per thread unit (2: paired 128-bit val / 64-bit meta loads)
    std::vector<SpmvKBlock> blocks;
    std::vector<double> val;
    std::vector<uint32_t> meta;  // (col - col_lo) << rb | (row - row0)
};
// Rows [previous row_end, row_end) are cut into `blocks` equal blocks (empty
// list: one segment of 4 x 148 blocks, two waves of two CTAs per SM).
struct ColsortSegment {
    uint64_t row_end;
    uint64_t blocks;
};
bool spmv_colsort_build(uint64_t m, uint64_t n, const int32_t* rp, const int32_t* col, const double* val,
                        SpmvColsortLayout& layout, const std::vector<ColsortSegment>& segments = {},
                        int classes = 16, bool tc_lanes = false, int vec = 1);
// bank-ordering classes of a K17 layout for this unit (1: plain column order on the
// fixed-point grid, 16: FP64 rows)
inline int colsort_classes(bool tc) {
    const int c = tuning().spmv_colsort_classes;
    return c ? c : (colsort_fixed_for(tc) ? 1 : 16);
}
cudaError_t launch_spmv_colsort(int unit, int vec, const SpmvKBlock* blks, int b0, int b1, int rb, int rows,
                                const double* val, const unsigned* meta, const double* x, double* y,
                                const ColsortRun& run, cudaStream_t s);

// Launch accounting (rl_kernel_launches): every <<<>>> site reports itself.
void note_launch(uint64_t n = 1);

cudaError_t launch_fill_uniform(double* out, uint64_t n, uint64_t seed, uint64_t stream_id,
                                uint64_t idx0, int kind, cudaStream_t s);
cudaError_t launch_gen_band_csr(uint64_t m_local, uint64_t row0, uint64_t n, uint32_t k,
                                uint64_t hb, uint64_t seed, int* rp, int* col, double* val,
                                cudaStream_t s);
cudaError_t launch_stencil_init(double* u, uint64_t nx, uint64_t ny, uint64_t nz, int dim,
                                uint64_t outer_begin, uint64_t outer_end, int radius,
                                uint64_t seed, cudaStream_t s);
cudaError_t launch_fp64_peak(int unit, uint64_t iters, double* sink, double* flops,
                             cudaStream_t s);

}  // namespace rlb
