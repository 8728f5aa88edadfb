/*
 * rooflens_b200.h -- C-ABI of the B200-native (sm_100a) FP64 memory-bound
 * kernels of arXiv 2502.16851: STREAM Scale, CSR SpMV and Jacobi stencils,
 * each with a CUDA-core (DFMA) and a tensor-core (DMMA) variant.
 *
 * The executing entry points sit behind the reference's kernel identities
 * (/root/reference/proj/include/rooflens/kernels.hpp:84-105): every call
 * returns, in its rl_kchar, exactly the W (flops) / Q (bytes) that the
 * reference model computes for the same arguments.
 *
 * Conventions
 *   - Plain pointers and sizes only.  Device pointers unless the function
 *     name ends in _host.  Calls are asynchronous on `stream` (a
 *     cudaStream_t; NULL = the legacy default stream) except _host calls and
 *     pure host functions.  No allocation happens in the device entry points.
 *   - Return codes: RL_OK (0); 1 + ErrorKind ordinal of the reference
 *     (error.hpp:10-32: MissingPeak=0 ... IoError=16); RL_ERR_CUDA_BASE +
 *     cudaError_t; RL_ERR_NCCL_BASE + ncclResult_t (rl_dist_* only).  rl_last_error() returns a thread-local copy of the
 *     message, formatted like the reference's exceptions ("<Kind>: <msg>",
 *     error.hpp:38-40).  No exception crosses the boundary.
 *   - Precision is FP64 only in this build (ValidationError otherwise).
 *   - Reentrant per stream.  There is no CPU fallback: on a machine without a
 *     usable sm_100a device the executing entry points fail with a CUDA code.
 */
#ifndef ROOFLENS_B200_H
#define ROOFLENS_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define RL_API __attribute__((visibility("default")))
#else
#define RL_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ExecutionUnit (hardware.hpp:19) -- selects the CC or TC kernel variant. */
typedef enum { RL_CUDA_CORE = 0, RL_TENSOR_CORE = 1 } rl_unit;
/* Precision (hardware.hpp:21) -- element_bytes 8/4/2 (hardware.cpp:27-34). */
typedef enum { RL_FP64 = 0, RL_FP32 = 1, RL_FP16 = 2 } rl_precision;
/* Boundedness (roofline.hpp:17). */
typedef enum { RL_MEMORY_BOUND = 0, RL_COMPUTE_BOUND = 1, RL_BALANCED = 2 } rl_boundedness;

typedef void* rl_stream; /* cudaStream_t */

/* Flattened KernelCharacterization (kernels.hpp:34-44). */
typedef struct {
    uint64_t work_flops;
    uint64_t traffic_bytes;
} rl_kchar;

/* HardwareSpec (hardware.hpp:43-58), SI units.  The reference's
 * map<(ExecutionUnit, Precision), peak> is the fixed table peaks[unit][precision]
 * (rl_unit x rl_precision ordinals); 0 = no entry (MissingPeak on use). */
typedef struct {
    char name[64];
    double memory_bandwidth; /* bytes/s */
    double l2_cache_bytes;
    double peaks[2][3];      /* flops/s */
} rl_hw_spec;

#define RL_OK 0
#define RL_ERR_KIND_BASE 1
#define RL_ERR_CUDA_BASE 100
#define RL_ERR_NCCL_BASE 200

/* ErrorKind ordinals (error.hpp:10-32). */
enum {
    RL_KIND_MISSING_PEAK = 0, RL_KIND_PARSE_ERROR, RL_KIND_VALIDATION_ERROR,
    RL_KIND_MISSING_FIELD, RL_KIND_UNKNOWN_HARDWARE, RL_KIND_INVALID_COUNT,
    RL_KIND_INVALID_INDEX_SIZE, RL_KIND_ZERO_INTENSITY, RL_KIND_INVALID_ALPHA,
    RL_KIND_ZERO_BALANCE, RL_KIND_INVALID_RANGE, RL_KIND_BAD_BANNER,
    RL_KIND_UNSUPPORTED_FORMAT, RL_KIND_MALFORMED_ENTRY, RL_KIND_INDEX_OUT_OF_RANGE,
    RL_KIND_TRUNCATED_FILE, RL_KIND_IO_ERROR
};

RL_API const char* rl_last_error(void);
RL_API const char* rl_version(void);

/* ---------------------------------------------------------------------------
 * Accounting (pure host functions) -- the reference models, restated.
 * ------------------------------------------------------------------------- */

/* replaces rooflens::scale_model            kernels.hpp:86,  kernels.cpp:74-86 */
RL_API int rl_scale_model(uint64_t n_elements, rl_precision precision, rl_kchar* out);
/* replaces rooflens::gemv_model             kernels.hpp:89,  kernels.cpp:88-101 */
RL_API int rl_gemv_model(uint64_t m, uint64_t n, rl_precision precision, rl_kchar* out);
/* replaces rooflens::spmv_generic_model     kernels.hpp:93-95, kernels.cpp:103-121 */
RL_API int rl_spmv_generic_model(uint64_t rows, uint64_t cols, uint64_t nnz,
                          uint64_t index_entry_count, uint64_t index_entry_bytes,
                          uint64_t packed_entry_count, uint64_t packed_entry_bytes,
                          rl_precision precision, rl_kchar* out);
/* replaces rooflens::spmv_csr_model         kernels.hpp:99-100, kernels.cpp:123-135 */
RL_API int rl_spmv_csr_model(uint64_t rows, uint64_t cols, uint64_t nnz, uint64_t index_bytes,
                      rl_precision precision, rl_kchar* out);
/* replaces rooflens::stencil_model          kernels.hpp:104-105, kernels.cpp:137-155 */
RL_API int rl_stencil_model(const char* preset, rl_precision precision, uint64_t temporal_depth,
                     rl_kchar* out);
/* replaces rooflens::stencil_preset         kernels.hpp:74, kernels.cpp:62-68
 * (dim 2|3, |S|, halo radius). */
RL_API int rl_stencil_preset(const char* name, int* dimensionality, uint64_t* point_count,
                      int* radius);
/* Default weights of a preset in canonical offset order (BASELINE.json). */
RL_API int rl_stencil_default_weights(const char* name, double* weights, uint64_t capacity);

/* ---------------------------------------------------------------------------
 * Executing kernels (device pointers, async on `stream`).
 * ------------------------------------------------------------------------- */

/* STREAM Scale a[i] = q*b[i].  CC: 256-bit LDG/STG DMUL.
 * TC: A = B*(qI) on DMMA m8n8k4.  Bit-exact vs q*b for
 * finite inputs; the TC variant returns +0 for b = -0 and propagates a
 * non-finite b into its 4-element fragment row (documented in DESIGN.md). */
RL_API int rl_scale(rl_unit unit, rl_precision precision, double* a, const double* b, double q,
             uint64_t n, rl_stream stream, rl_kchar* out);

/* Dense GEMV y = A*x, row-major A (m x n) (next row #4).
 * kchar = gemv_model(m, n, FP64) (kernels.cpp:88-101). */
RL_API int rl_gemv(rl_unit unit, rl_precision precision, uint64_t m, uint64_t n, const double* A,
                   const double* x, double* y, rl_stream stream, rl_kchar* out);

/* CSR SpMV y = A*x, int32 row_ptr (m+1) / col (nnz),
 * 0-based, column indices in [0, n).  kchar = spmv_csr_model(.., 4, FP64). */
RL_API int rl_spmv_csr(rl_unit unit, rl_precision precision, uint64_t m, uint64_t n, uint64_t nnz,
                const int32_t* row_ptr, const int32_t* col, const double* val,
                const double* x, double* y, rl_stream stream, rl_kchar* out);

/* Row-range form for row-partitioned / overlapped use: computes y[i] for
 * i in [row_begin, row_end) reading x[col[k] - col_base].  No accounting. */
RL_API int rl_spmv_csr_rows(rl_unit unit, rl_precision precision, uint64_t row_begin,
                     uint64_t row_end, const int32_t* row_ptr, const int32_t* col,
                     const double* val, const double* x, int64_t col_base, double* y,
                     rl_stream stream);

/* Jacobi stencil, `steps` double-buffered timesteps.
 * dims = {nx, ny, nz} (x fastest; nz ignored for 2D presets).  weights: |S|
 * doubles in canonical offset order, or NULL for the BASELINE defaults.  The
 * outer ring of width `radius` is a Dirichlet boundary and is never written
 * (initialise it identically in u and v).  Result in u if steps is even,
 * else in v.  kchar = stencil_model(preset, FP64, 1) x updated points x steps. */
RL_API int rl_stencil(rl_unit unit, rl_precision precision, const char* preset,
               const uint64_t* dims, const double* weights, uint64_t steps, double* u,
               double* v, rl_stream stream, rl_kchar* out);

/* Temporal blocking (stencil_model's temporal_depth t, kernels.cpp:137-155;
 * PAPER.md:223-236): `steps` timesteps executed as steps/t fused sweeps of t
 * timesteps each (plus steps%t single sweeps).  HBM sees one read of u and one
 * write of v per fused sweep.  t = 1 behaves like rl_stencil.  CUDA core:
 * t = 2..8 for 2d5pt (even t: even nx and 16-byte aligned rows), t = 2..4 for
 * 3d7pt and 3d27pt (any weights).  Tensor core: t = 2..4 for 2d5pt (even nx,
 * 16-byte aligned u and v; each level the x-band-on-DMMA form).  t > 8 is
 * InvalidRange; other presets / depths / units are ValidationError.
 * Buffers swap once per sweep: *result_in_v (optional) reports where the
 * final field is.  kchar = stencil_model(preset, FP64, t) x points x (steps/t)
 * + stencil_model(preset, FP64, 1) x points x (steps%t). */
RL_API int rl_stencil_temporal(rl_unit unit, rl_precision precision, const char* preset,
                               const uint64_t* dims, const double* weights, uint64_t steps,
                               uint64_t temporal_depth, double* u, double* v, rl_stream stream,
                               int* result_in_v, rl_kchar* out);

/* One sweep v = S(u) restricted to outer indices [o_begin, o_end) (rows in 2D,
 * planes in 3D) -- the slab / interior-vs-edge building block.  Boundary
 * indices inside the range are skipped.  No accounting. */
RL_API int rl_stencil_sweep(rl_unit unit, rl_precision precision, const char* preset,
                     const uint64_t* dims, const double* weights, uint64_t o_begin,
                     uint64_t o_end, const double* u, double* v, rl_stream stream);

/* ---------------------------------------------------------------------------
 * End-to-end entry points on HOST buffers: pinned staging, H2D copies,
 * kernel(s), D2H copy, all inside the call (synchronous).  Chunked and
 * pipelined on two streams so copies overlap each other and the kernels.
 * ------------------------------------------------------------------------- */

RL_API int rl_scale_host(rl_unit unit, rl_precision precision, double* a, const double* b, double q,
                  uint64_t n, rl_kchar* out);
RL_API int rl_spmv_csr_host(rl_unit unit, rl_precision precision, uint64_t m, uint64_t n,
                     uint64_t nnz, const int32_t* row_ptr, const int32_t* col,
                     const double* val, const double* x, double* y, rl_kchar* out);
RL_API int rl_stencil_host(rl_unit unit, rl_precision precision, const char* preset,
                    const uint64_t* dims, const double* weights, uint64_t steps, double* u,
                    double* v, rl_kchar* out);
/* SpMV plan: the CSR matrix is uploaded once (the iterative-solver pattern:
 * A is fixed, x changes every step) and each execute moves only x in and y
 * out.  At creation the plan re-lays A as column-sorted row blocks (K17,
 * y rows of a block in shared memory, x read in column order)
 * when every row has <= 1024 nonzeros and the block column spans fit, else
 * keeps the CSR (with the long-row path); the layout streams no more bytes
 * than the CSR.  The column-sorted layout sums each row on a 64-bit
 * fixed-point grid (both units; rows too small for 2^-46 relative precision
 * on it are re-summed in FP64 in a fixed order), so repeated executes are
 * bit-identical; CSR executes are bit-reproducible too.  Tuning
 * key spmv_plan_colsort = 0 keeps the CSR.  execute_host pipelines the x upload, the row-chunk kernels and the y download on three streams: row
 * chunk c starts as soon as the x prefix it references (max column, computed
 * at creation) has arrived.  The plan owns its device buffers; no allocation
 * happens in execute. */
typedef struct rl_spmv_plan_s* rl_spmv_plan;
RL_API int rl_spmv_plan_create(rl_unit unit, rl_precision precision, uint64_t m, uint64_t n,
                               uint64_t nnz, const int32_t* row_ptr, const int32_t* col,
                               const double* val, rl_spmv_plan* out);
RL_API int rl_spmv_plan_execute_host(rl_spmv_plan plan, const double* x, double* y, rl_kchar* out);
/* The same pipelined call, returning once it is enqueued: consecutive calls
 * overlap (call k + 1's x upload beside call k's compute and y download) on
 * three device buffer slots.  x must stay unchanged and y unread until
 * rl_spmv_plan_wait returns; a later rl_spmv_plan_execute_host waits first.
 * For streams of independent vectors (no rooflens counterpart: the reference
 * has no executing path). */
RL_API int rl_spmv_plan_execute_host_async(rl_spmv_plan plan, const double* x, double* y, rl_kchar* out);
RL_API int rl_spmv_plan_wait(rl_spmv_plan plan);
RL_API int rl_spmv_plan_execute(rl_spmv_plan plan, const double* x_dev, double* y_dev,
                                rl_stream stream, rl_kchar* out);
RL_API int rl_spmv_plan_destroy(rl_spmv_plan plan);
/* Layout of a plan: *layout = 0 CSR, 4 column-sorted row blocks (K17);
 * *layout_bytes = device bytes one execute streams for A. */
RL_API int rl_spmv_plan_info(rl_spmv_plan plan, int* layout, uint64_t* layout_bytes);

/* Release the device/pinned workspaces cached by the _host entry points. */
RL_API int rl_host_workspace_release(void);

/* ---------------------------------------------------------------------------
 * Deterministic input generators (device), bit-identical to oracle/oracle.c.
 * ------------------------------------------------------------------------- */

/* kind 0: U[0,1), kind 1: U[-1,1); element i keyed by (seed, stream_id, idx0+i). */
RL_API int rl_fill_uniform(double* out, uint64_t n, uint64_t seed, uint64_t stream_id, uint64_t idx0,
                    int kind, rl_stream stream);
/* Banded CSR rows [row0, row0+m_local) of an n-column matrix, k sorted distinct
 * columns per row uniform in [max(0,i-hb), min(n-1,i+hb)]; values U[-1,1).
 * row_ptr is local (starts at 0), columns are global. */
RL_API int rl_gen_band_csr(uint64_t m_local, uint64_t row0, uint64_t n, uint32_t k, uint64_t hb,
                    uint64_t seed, int32_t* row_ptr, int32_t* col, double* val,
                    rl_stream stream);
/* Stencil field: interior U[0,1) keyed by the global linear index, Dirichlet
 * ring (width radius) 0.  dims = global {nx, ny, nz} (nz ignored when dim==2);
 * the buffer holds outer indices [outer_begin, outer_end) of the global grid
 * (rows in 2D, planes in 3D) -- a whole grid or one rank's slab with ghosts. */
RL_API int rl_stencil_init(double* u, const uint64_t* dims, int dim, uint64_t outer_begin,
                           uint64_t outer_end, int radius, uint64_t seed, rl_stream stream);

/* ---------------------------------------------------------------------------
 * Matrix Market ingestion (host) and per-matrix roofline analysis.
 * ------------------------------------------------------------------------- */

/* replaces rooflens::parse_stats_file (matrix_market.cpp:126-201): rows, cols
 * and the expanded nnz (symmetric storage counted twice off the diagonal);
 * same ErrorKinds (BadBanner, UnsupportedFormat, MalformedEntry,
 * IndexOutOfRange, TruncatedFile, IoError, ValidationError). */
RL_API int rl_mtx_stats(const char* path, uint64_t* rows, uint64_t* cols, uint64_t* nnz);
/* Extension: materialise the CSR (0-based int32, columns sorted per row,
 * symmetric/skew storage expanded, pattern = 1.0) into caller buffers of at
 * least rows+1 / nnz entries (sizes from rl_mtx_stats). */
RL_API int rl_mtx_read_csr(const char* path, uint64_t row_capacity, uint64_t nnz_capacity,
                           int32_t* row_ptr, int32_t* col, double* val, uint64_t* rows,
                           uint64_t* cols, uint64_t* nnz);

/* replaces rooflens::stats_to_report (matrix_market.cpp:203-216). */
typedef struct {
    uint64_t work_flops;
    uint64_t traffic_bytes;
    int boundedness;          /* rl_boundedness vs the CUDA-core balance */
    double kernel_ceiling;    /* kernel_speedup_ceiling at the spec's alpha */
    int kernel_ceiling_warnings;
    double workload_ceiling;
    uint64_t csr_bytes;
    int fits_in_l2;
} rl_matrix_analysis;
RL_API int rl_matrix_analysis_of(uint64_t rows, uint64_t cols, uint64_t nnz, const rl_hw_spec* spec,
                                 rl_precision precision, rl_matrix_analysis* out);

/* ---------------------------------------------------------------------------
 * Hardware spec, roofline and speedup bounds (pure host functions).
 * ------------------------------------------------------------------------- */

/* replaces rooflens::load_spec (hardware.cpp:183-237): same JSON schema
 * (hardware.hpp:75-81), unknown keys -> ParseError, SI conversion. */
RL_API int rl_load_spec(const char* json_text, rl_hw_spec* out);
/* replaces rooflens::load_spec_file (hardware.cpp:239-247): IoError when the
 * file cannot be opened, else load_spec of its contents. */
RL_API int rl_load_spec_file(const char* path, rl_hw_spec* out);
/* replaces rooflens::serialize_spec (hardware.cpp:249-264): the same 2-space
 * JSON document, byte for byte.  Writes at most `capacity` bytes including
 * the terminating NUL; *length (optional) gets the full length without it
 * (InvalidRange when it does not fit). */
RL_API int rl_serialize_spec(const rl_hw_spec* spec, char* buffer, uint64_t capacity, uint64_t* length);
/* replaces rooflens::builtin_spec (hardware.cpp:121-150): "A100-80GB", "GH200". */
RL_API int rl_builtin_spec(const char* name, rl_hw_spec* out);
/* machine_balance (hardware.cpp:112-114) / tensor_alpha (hardware.cpp:116-119). */
RL_API int rl_machine_balance(const rl_hw_spec* spec, rl_unit unit, rl_precision precision,
                       double* out);
RL_API int rl_tensor_alpha(const rl_hw_spec* spec, rl_precision precision, double* out);
/* attainable = min(P, B*I) (roofline.cpp:21-28); classify (roofline.cpp:30-34). */
RL_API int rl_attainable(const rl_hw_spec* spec, rl_unit unit, rl_precision precision,
                  double intensity, double* out);
RL_API int rl_classify(double intensity, double balance);
/* ridge_point (roofline.cpp:36-38) and sample_curve (roofline.cpp:40-79):
 * n_points log-spaced intensities in [i_min, i_max] plus the ridge when it
 * falls inside; writes *count (<= n_points + 1) pairs into intensity[] and
 * attainable[] (capacity entries each; InvalidRange if too small). */
RL_API int rl_ridge_point(const rl_hw_spec* spec, rl_unit unit, rl_precision precision, double* out);
RL_API int rl_sample_curve(const rl_hw_spec* spec, rl_unit unit, rl_precision precision, double i_min,
                           double i_max, uint64_t n_points, double* intensity, double* attainable,
                           uint64_t capacity, uint64_t* count);
/* bounds.cpp:56-62, 72-135. */
RL_API int rl_unoverlapped_speedup(double t_cmp, double t_mem, double t_others, double alpha,
                            double* out);
/* mem_cmp_ratio = B / I (bounds.cpp:45-48); overlapped_total = max of the
 * time components (bounds.cpp:50-53). */
RL_API int rl_mem_cmp_ratio(double balance, double intensity, double* out);
RL_API int rl_overlapped_total(double t_cmp, double t_mem, double t_others, double* out);
RL_API int rl_kernel_speedup_ceiling(double alpha, double balance, double intensity, double* out,
                              int* n_warnings);
RL_API int rl_tensor_core_ceiling(double alpha, double* out);
RL_API int rl_workload_ceiling(double intensity, double balance, double* out);
RL_API int rl_min_temporal_depth(double balance, double single_step_intensity, uint64_t* out);
RL_API int rl_tc_scale_trick_throughput(double peak_tc, uint64_t m, uint64_t n, double* out);

/* SpeedupBound as a reportable object (bounds.hpp:27-45): value, BoundKind
 * ordinal (bounds.hpp:27-32: 0 exact un-overlapped, 1 kernel ceiling, 2
 * tensor-core ceiling, 3 workload ceiling) and the reference's assumption and
 * warning strings (bounds.cpp:64-108).  `text` receives the n_assumptions
 * assumption lines then the n_warnings warning lines, each '\n'-terminated,
 * NUL-terminated; *length (optional) gets the full length without the NUL; a
 * null `text` only sizes; a short buffer is InvalidRange. */
typedef struct {
    double value;
    int kind;
    int n_assumptions;
    int n_warnings;
} rl_speedup_bound;
/* to_string(BoundKind) (bounds.cpp:27-35); "?" for an unknown ordinal. */
RL_API const char* rl_bound_kind_name(int kind);
/* unoverlapped_bound (bounds.cpp:64-70). */
RL_API int rl_unoverlapped_bound(double t_cmp, double t_mem, double t_others, double alpha,
                                 rl_speedup_bound* out, char* text, uint64_t capacity, uint64_t* length);
/* kernel_speedup_ceiling (bounds.cpp:72-85), with its I >= B warning text. */
RL_API int rl_kernel_ceiling_bound(double alpha, double balance, double intensity, rl_speedup_bound* out,
                                   char* text, uint64_t capacity, uint64_t* length);
/* tensor_core_ceiling (bounds.cpp:87-96). */
RL_API int rl_tensor_core_bound(double alpha, rl_speedup_bound* out, char* text, uint64_t capacity,
                                uint64_t* length);
/* workload_ceiling (bounds.cpp:98-108). */
RL_API int rl_workload_bound(double intensity, double balance, rl_speedup_bound* out, char* text,
                             uint64_t capacity, uint64_t* length);

/* rooflens::build_analysis + render_text / render_json / render_csv
 * (report.hpp:19-48; the reference declares them without an implementation,
 * the behaviour follows SPEC.md cli_report): classification against the
 * CUDA-core balance at `precision` (or *balance_override when non-null), the
 * kernel / tensor-core / workload ceilings, the temporal-depth section when
 * single_step_intensity is non-null, notes and the verdict ("tensor cores
 * cannot exceed X× on this kernel/machine", X = min bound to 3 significant
 * digits).  Text uses 4 significant digits; json / csv full precision.
 * Buffer convention as rl_serialize_spec. */
#define RL_REPORT_TEXT 0
#define RL_REPORT_JSON 1
#define RL_REPORT_CSV 2
RL_API int rl_analysis_render(const rl_hw_spec* spec, rl_precision precision, const char* kernel_name,
                              uint64_t work_flops, uint64_t traffic_bytes, const double* balance_override,
                              const double* single_step_intensity, int format, char* buffer,
                              uint64_t capacity, uint64_t* length);

/* ---------------------------------------------------------------------------
 * Multi-GPU (north_star): one process per GPU, NCCL
 * point-to-point over NVLink/NVSwitch, the kernels above as per-part compute.
 * The reference has no multi-GPU form; these entry points are
 * the sharded counterparts of rl_scale / rl_spmv_csr / rl_stencil and return
 * the reference model's W/Q of the WHOLE (global) problem.
 *
 * A job is split into P = world * parts_local contiguous parts; process
 * `rank` owns parts [rank*parts_local, (rank+1)*parts_local).  Production
 * runs use parts_local = 1 (one part per GPU); parts_local > 1 runs several
 * parts on one GPU through the same NCCL schedule (self send/recv), which is
 * how the exchange is tested on a single device.  NCCL is loaded at
 * rl_dist_init (the copy already in the process, e.g. torch's, else
 * $RL_NCCL_LIBRARY, else libnccl.so.2); failures return RL_ERR_NCCL_BASE +
 * ncclResult_t.  Buffers are caller-owned device memory on the communicator's
 * device; plans keep pointers, streams, events and CUDA graphs.
 * ------------------------------------------------------------------------- */
typedef struct rl_dist_s* rl_dist;
#define RL_DIST_UNIQUE_ID_BYTES 128
/* ncclGetUniqueId on one process (rank 0); share the bytes out of band. */
RL_API int rl_dist_unique_id(uint8_t* id /* RL_DIST_UNIQUE_ID_BYTES */);
/* ncclCommInitRank on the current CUDA device. */
RL_API int rl_dist_init(int world, int rank, const uint8_t* id, rl_dist* out);
RL_API int rl_dist_destroy(rl_dist comm);
RL_API int rl_dist_info(rl_dist comm, int* world, int* rank, int* device, int* nccl_version);
/* Sum of one uint64 over all ranks (NCCL all-reduce; synchronous). */
RL_API int rl_dist_allreduce_u64(rl_dist comm, uint64_t* value);
/* Max of one double over all ranks (NCCL all-reduce; synchronous) -- the
 * max-over-ranks of a device-timed interval. */
RL_API int rl_dist_allreduce_max(rl_dist comm, double* value);

/* Partitions (pure host).  Part `part` of `parts`: contiguous block of n,
 * sizes differing by <= 1, larger blocks first. */
RL_API int rl_dist_block(uint64_t n, uint64_t parts, uint64_t part, uint64_t* begin, uint64_t* end);
/* SpMV rows [row_begin, row_end) and x window [col_begin, col_end) =
 * [max(0, row_begin - hb), min(n, row_end + hb)) of a part of an n x n
 * matrix with half-bandwidth hb.  ValidationError when a part holds fewer
 * than hb rows (the halo would span more than the neighbour). */
RL_API int rl_dist_spmv_part(uint64_t n, uint64_t hb, uint64_t parts, uint64_t part, uint64_t* row_begin,
                             uint64_t* row_end, uint64_t* col_begin, uint64_t* col_end);
/* Stencil slab of the outer axis (rows in 2D, planes in 3D; dims global):
 * owned [own_begin, own_end) and buffer [buf_begin, buf_end) = the owned
 * layers plus `radius` ghost layers per side where a neighbour exists.  The
 * part's u and v hold buf_end - buf_begin layers of the global layer size. */
RL_API int rl_dist_stencil_part(const char* preset, const uint64_t* dims, uint64_t parts, uint64_t part,
                                uint64_t* own_begin, uint64_t* own_end, uint64_t* buf_begin,
                                uint64_t* buf_end);

/* One halo transfer of the per-call / per-timestep exchange, in the order a
 * rank posts it inside one NCCL group: kind 0 = send, 1 = recv; `peer` =
 * the other rank; `part` = local part index; offset / count in doubles of
 * that part's x window (SpMV) or field buffer (stencil). */
typedef struct {
    int32_t kind;
    int32_t peer;
    int32_t part;
    int32_t reserved;
    uint64_t offset;
    uint64_t count;
} rl_dist_op;
RL_API int rl_dist_spmv_schedule(uint64_t n, uint64_t hb, int world, int parts_local, int rank,
                                 rl_dist_op* ops, uint64_t capacity, uint64_t* count);
RL_API int rl_dist_stencil_schedule(const char* preset, const uint64_t* dims, int world, int parts_local,
                                    int rank, rl_dist_op* ops, uint64_t capacity, uint64_t* count);

/* STREAM Scale on this rank's chunk rl_dist_block(n_global, world, rank):
 * a / b hold that chunk.  No communication.  kchar = scale_model(n_global). */
RL_API int rl_dist_scale(rl_dist comm, rl_unit unit, rl_precision precision, double* a, const double* b,
                         double q, uint64_t n_global, rl_stream stream, rl_kchar* out);

/* Row-partitioned CSR SpMV of an n x n matrix with half-bandwidth hb.  For
 * local part i: row_ptr[i] (rows+1, starting at 0), col[i] (GLOBAL columns),
 * val[i], x[i] = the part's x window (col_end - col_begin doubles; the
 * caller writes the owned x at offset row_begin - col_begin before each
 * execute), y[i] (rows).  create checks every column against [0, n) and the
 * band (ValidationError otherwise), sums nnz over the ranks, and reserves the
 * plan's streams, events and long-row workspace. */
typedef struct rl_dist_spmv_s* rl_dist_spmv;
RL_API int rl_dist_spmv_create(rl_dist comm, rl_unit unit, rl_precision precision, uint64_t n, uint64_t hb,
                               int parts_local, const int32_t* const* row_ptr, const int32_t* const* col,
                               const double* const* val, double* const* x, double* const* y,
                               rl_dist_spmv* out);
/* One y = A x: the halo exchange (NCCL group on a high-priority stream)
 * overlaps the interior rows; the edge rows follow.  Ordered after prior work
 * on `stream`; later work on `stream` sees y.  kchar = spmv_csr_model of the
 * global matrix.  Replayed as a CUDA graph after the first call. */
RL_API int rl_dist_spmv_execute(rl_dist_spmv plan, rl_stream stream, rl_kchar* out);
RL_API int rl_dist_spmv_destroy(rl_dist_spmv plan);

/* Slab-decomposed Jacobi stencil on the global grid `dims`.  u[i] / v[i]:
 * local part i's buffers (rl_dist_stencil_part layers; the Dirichlet ring
 * identical in both).  run performs `steps` timesteps starting from u: per
 * timestep the ghost layers go out on the NCCL stream while the slab interior
 * is swept, then the edge layers are swept.  Result in u for even steps, in v
 * for odd (*result_in_v).  Timestep pairs replay as one CUDA graph.  kchar =
 * stencil_model(preset, FP64, 1) x global interior points x steps. */
typedef struct rl_dist_stencil_s* rl_dist_stencil;
RL_API int rl_dist_stencil_create(rl_dist comm, rl_unit unit, rl_precision precision, const char* preset,
                                  const uint64_t* dims, const double* weights, int parts_local,
                                  double* const* u, double* const* v, rl_dist_stencil* out);
RL_API int rl_dist_stencil_run(rl_dist_stencil plan, uint64_t steps, rl_stream stream, int* result_in_v,
                               rl_kchar* out);
RL_API int rl_dist_stencil_destroy(rl_dist_stencil plan);

/* ---------------------------------------------------------------------------
 * K11: FP64 peak microbenchmarks (DFMA chains on the fp64 pipe, DMMA chains on
 * the tensor pipe), all SMs.  Launches one kernel on `stream`; *flops_out gets
 * the exact flop count it performs (divide by the event time).
 * ------------------------------------------------------------------------- */
RL_API int rl_fp64_peak_launch(rl_unit unit, uint64_t iters, rl_stream stream, double* sink,
                        double* flops_out);

/* Kernel-variant selection knobs (benchmark sweeps); returns previous value. */
RL_API int rl_tuning_set(const char* key, int64_t value, int64_t* previous);

/* Number of CUDA kernels this library has launched since load (evidence for
 * the benchmark's gpu_launches count). */
RL_API uint64_t rl_kernel_launches(void);

#ifdef __cplusplus
}
#endif

#endif /* ROOFLENS_B200_H */
