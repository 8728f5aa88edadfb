// rooflens_b200.hpp -- C++ entry points of the B200 kernels, mirroring the
// reference's kernel identities (/root/reference/proj/include/rooflens/
// kernels.hpp:84-105, hardware.hpp, roofline.hpp, bounds.hpp) with executing
// sm_100a variants behind them.  The C-ABI in rooflens_b200.h wraps these
// (exceptions -> status codes).  Everything here is new code: the reference's
// functions are restated from their documented formulas, not linked.
#pragma once

#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

namespace rooflens::b200 {

// error.hpp:10-32 -- identical ordinals.
enum class ErrorKind {
    MissingPeak, ParseError, ValidationError, MissingField, UnknownHardware,
    InvalidCount, InvalidIndexSize, ZeroIntensity, InvalidAlpha, ZeroBalance, InvalidRange,
    BadBanner, UnsupportedFormat, MalformedEntry, IndexOutOfRange, TruncatedFile, IoError,
};
const char* to_string(ErrorKind kind);

// error.hpp:36-46 -- message "<Kind>: <msg>".
class Error : public std::runtime_error {
public:
    Error(ErrorKind kind, const std::string& msg)
        : std::runtime_error(std::string(to_string(kind)) + ": " + msg), kind_(kind) {}
    ErrorKind kind() const { return kind_; }

private:
    ErrorKind kind_;
};

// A CUDA runtime failure inside an executing entry point.
class CudaError : public std::runtime_error {
public:
    CudaError(int code, const std::string& msg) : std::runtime_error(msg), code_(code) {}
    int code() const { return code_; }

private:
    int code_;
};

enum class ExecutionUnit { CudaCore, TensorCore };   // hardware.hpp:19
enum class Precision { FP64, FP32, FP16 };           // hardware.hpp:21
std::size_t element_bytes(Precision p);               // hardware.cpp:27-34
using Stream = void*;                                  // cudaStream_t

struct KernelCharacterization {  // kernels.hpp:34-44
    std::string kernel_name;
    std::uint64_t work_flops = 0;
    std::uint64_t traffic_bytes = 1;
    double intensity() const { return double(work_flops) / double(traffic_bytes); }
};

struct SparseMatrixStats {  // kernels.hpp:46-53
    std::uint64_t rows = 1, cols = 1, nnz = 1;
    void validate() const;
};

struct SparseMetadataTraffic {  // kernels.hpp:57-64
    std::uint64_t index_entry_count = 0, index_entry_bytes = 0;
    std::uint64_t packed_entry_count = 0, packed_entry_bytes = 0;
    void validate() const;
};

struct StencilShape {  // kernels.hpp:66-70 (+ halo radius, needed to execute)
    std::string name;
    int dimensionality = 2;
    std::uint64_t point_count = 1;
    int radius = 1;
};
const StencilShape& stencil_preset(std::string_view name);          // kernels.cpp:62-68
const std::vector<StencilShape>& stencil_presets();                 // kernels.cpp:54-60
std::vector<double> stencil_default_weights(std::string_view name); // BASELINE.json

inline constexpr std::uint64_t kDefaultIndexBytes = 4;  // kernels.hpp:77

// Accounting models (kernels.cpp:74-155).
KernelCharacterization scale_model(std::uint64_t n_elements, Precision precision);
KernelCharacterization gemv_model(std::uint64_t m, std::uint64_t n, Precision precision);
KernelCharacterization spmv_generic_model(const SparseMatrixStats& stats,
                                          const SparseMetadataTraffic& meta, Precision precision);
KernelCharacterization spmv_csr_model(const SparseMatrixStats& stats, std::uint64_t index_bytes,
                                      Precision precision);
KernelCharacterization stencil_model(const StencilShape& shape, Precision precision,
                                     std::uint64_t temporal_depth);

// Executing kernels (device pointers, asynchronous on `stream`).
KernelCharacterization scale(ExecutionUnit unit, Precision precision, double* a, const double* b,
                             double q, std::uint64_t n, Stream stream);
KernelCharacterization gemv(ExecutionUnit unit, Precision precision, std::uint64_t m, std::uint64_t n,
                            const double* A, const double* x, double* y, Stream stream);
KernelCharacterization spmv_csr(ExecutionUnit unit, Precision precision,
                                const SparseMatrixStats& stats, const std::int32_t* row_ptr,
                                const std::int32_t* col, const double* val, const double* x,
                                double* y, Stream stream);
// long_rows: -1 = unknown (rows longer than the tuning key spmv_long_min are
// diverted on the device to a load-balanced second kernel), 0 = the caller
// knows there are none, 1 = present.
void spmv_csr_rows(ExecutionUnit unit, Precision precision, std::uint64_t row_begin,
                   std::uint64_t row_end, const std::int32_t* row_ptr, const std::int32_t* col,
                   const double* val, const double* x, std::int64_t col_base, double* y,
                   Stream stream, int long_rows = -1);
KernelCharacterization stencil(ExecutionUnit unit, Precision precision, const StencilShape& shape,
                               const std::uint64_t dims[3], const double* weights,
                               std::uint64_t steps, double* u, double* v, Stream stream);
void stencil_sweep(ExecutionUnit unit, Precision precision, const StencilShape& shape,
                   const std::uint64_t dims[3], const double* weights, std::uint64_t o_begin,
                   std::uint64_t o_end, const double* u, double* v, Stream stream);

// Matrix Market (matrix_market.cpp:126-201) + CSR materialisation.
SparseMatrixStats mtx_stats(const std::string& path);
SparseMatrixStats mtx_read_csr(const std::string& path, std::vector<std::int32_t>& row_ptr,
                               std::vector<std::int32_t>& col, std::vector<double>& val);

// Hardware spec (hardware.hpp:43-89).  The reference's map<(unit,
// precision), peak> is a fixed [unit][precision] table here (0 = absent).
struct HardwareSpec {
    std::string name;
    double memory_bandwidth = 0.0;  // B/s
    double l2_cache_bytes = 0.0;
    double peaks[2][3] = {};        // flops/s by [ExecutionUnit][Precision], 0 = absent
    bool has_peak(ExecutionUnit u, Precision p) const;
    double peak(ExecutionUnit u, Precision p) const;  // throws MissingPeak
    void validate() const;  // hardware.cpp:91-110, including the peak table
};
HardwareSpec load_spec(const std::string& json_text);
HardwareSpec load_spec_file(const std::string& path);    // hardware.cpp:239-247
std::string serialize_spec(const HardwareSpec& spec);    // hardware.cpp:249-264
const HardwareSpec& builtin_spec(std::string_view name);
double machine_balance(const HardwareSpec& spec, ExecutionUnit unit, Precision precision);
double tensor_alpha(const HardwareSpec& spec, Precision precision);

// Roofline (roofline.cpp:21-34).
enum class Boundedness { MemoryBound, ComputeBound, Balanced };
double attainable(const HardwareSpec& spec, ExecutionUnit unit, Precision precision,
                  double intensity);
Boundedness classify(double intensity, double balance);
// ridge_point / sample_curve (roofline.cpp:36-79): (intensity, attainable) pairs.
double ridge_point(const HardwareSpec& spec, ExecutionUnit unit, Precision precision);
std::vector<std::pair<double, double>> sample_curve(const HardwareSpec& spec, ExecutionUnit unit,
                                                    Precision precision, double i_min, double i_max,
                                                    std::size_t n_points);

// Bounds (bounds.cpp:56-135).
double mem_cmp_ratio(double balance, double intensity);
double overlapped_total(double t_cmp, double t_mem, double t_others);
double unoverlapped_speedup(double t_cmp, double t_mem, double t_others, double alpha);
double kernel_speedup_ceiling(double alpha, double balance, double intensity, int* n_warnings);
double tensor_core_ceiling(double alpha);
double workload_ceiling(double intensity, double balance);
std::uint64_t min_temporal_depth(double balance, double single_step_intensity);
double tc_scale_trick_throughput(double peak_tc, std::uint64_t m, std::uint64_t n);

// Bounds as reportable objects (bounds.hpp:27-45, bounds.cpp:64-108): the
// value plus the assumption and warning strings the reference attaches.
enum class BoundKind { ExactUnoverlapped, KernelCeiling, TensorCoreCeiling, WorkloadCeiling };
const char* to_string(BoundKind kind);  // bounds.cpp:27-35
struct SpeedupBound {
    double value = 1.0;
    BoundKind kind = BoundKind::ExactUnoverlapped;
    std::vector<std::string> assumptions;
    std::vector<std::string> warnings;
};
SpeedupBound unoverlapped_bound(double t_cmp, double t_mem, double t_others, double alpha);
SpeedupBound kernel_ceiling_bound(double alpha, double balance, double intensity);
SpeedupBound tensor_core_bound(double alpha);
SpeedupBound workload_bound(double intensity, double balance);

// Analysis report (report.hpp:19-48; declared by the reference, implemented
// here from SPEC.md cli_report): classification, every applicable ceiling,
// the temporal-depth section for stencils, and the one-line verdict.
struct AnalysisReport {
    HardwareSpec machine;
    Precision precision = Precision::FP64;
    double balance = 0.0;
    bool balance_overridden = false;
    std::optional<double> alpha;  // absent when the spec has no tensor-core peak at `precision`
    KernelCharacterization kernel;
    Boundedness boundedness = Boundedness::MemoryBound;
    double attainable_flops = 0.0;  // CUDA-core roofline at the kernel's intensity
    std::vector<SpeedupBound> bounds;
    std::optional<double> single_step_intensity;
    std::optional<std::uint64_t> min_depth;
    std::vector<std::string> notes;
    std::string verdict;
};
AnalysisReport build_analysis(const HardwareSpec& spec, Precision precision,
                              const KernelCharacterization& kernel,
                              std::optional<double> balance_override = {},
                              std::optional<double> single_step_intensity = {});
std::string render_text(const AnalysisReport& report);  // 4 significant digits
std::string render_json(const AnalysisReport& report);  // full precision
std::string render_csv(const AnalysisReport& report);   // full precision

}  // namespace rooflens::b200
