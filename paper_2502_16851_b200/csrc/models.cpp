// models.cpp -- host-side accounting, hardware spec, roofline and speedup
// bounds of the B200 framework.  Restates the reference's documented models
// (they are the byte/flop accounting the kernels are judged against) in new
// code; tests/test_accounting.py pins every value against the reference
// library itself (oracle/_ref).
//
//   scale / gemv / spmv / stencil models   reference kernels.cpp:74-155
//   presets                                reference kernels.cpp:54-68
//   HardwareSpec, load_spec, built-ins     reference hardware.cpp:81-237
//   attainable / classify                  reference roofline.cpp:21-34
//   bounds                                 reference bounds.cpp:56-135
#include <algorithm>
#include <cmath>
#include <fstream>
#include <sstream>
#include <map>
#include <numeric>

#include <json.hpp>

#include "../../include/rooflens_b200.hpp"

namespace rooflens::b200 {

namespace {
using u128 = unsigned __int128;

std::uint64_t checked(u128 v, const char* what) {
    if (v >> 64) throw Error(ErrorKind::InvalidRange, std::string(what) + " overflows 64-bit count");
    return static_cast<std::uint64_t>(v);
}

bool is_width(std::uint64_t b) { return b == 1 || b == 2 || b == 4 || b == 8; }

void require_width(std::uint64_t b, bool zero_ok, const char* what) {
    if ((zero_ok && b == 0) || is_width(b)) return;
    throw Error(ErrorKind::InvalidIndexSize, std::string(what) + " must be one of {" +
                                                 (zero_ok ? "0," : "") + "1,2,4,8}, got " +
                                                 std::to_string(b));
}

constexpr double kTera = 1e12, kMega = 1e6;
}  // namespace

const char* to_string(ErrorKind k) {
    static const char* names[] = {
        "MissingPeak", "ParseError", "ValidationError", "MissingField", "UnknownHardware",
        "InvalidCount", "InvalidIndexSize", "ZeroIntensity", "InvalidAlpha", "ZeroBalance",
        "InvalidRange", "BadBanner", "UnsupportedFormat", "MalformedEntry", "IndexOutOfRange",
        "TruncatedFile", "IoError"};
    const int i = static_cast<int>(k);
    return (i >= 0 && i < 17) ? names[i] : "Error";
}

std::size_t element_bytes(Precision p) {
    return p == Precision::FP64 ? 8 : p == Precision::FP32 ? 4 : 2;
}

// ---------------------------------------------------------------------------
// Problem descriptors
// ---------------------------------------------------------------------------
void SparseMatrixStats::validate() const {
    if (!rows || !cols) throw Error(ErrorKind::ValidationError, "matrix dimensions must be >= 1");
    if (!nnz) throw Error(ErrorKind::ValidationError, "nnz must be >= 1");
    if (u128(nnz) > u128(rows) * cols)
        throw Error(ErrorKind::ValidationError, "nnz " + std::to_string(nnz) + " exceeds rows*cols");
}

void SparseMetadataTraffic::validate() const {
    require_width(index_entry_bytes, true, "index_entry_bytes");
    require_width(packed_entry_bytes, true, "packed_entry_bytes");
}

const std::vector<StencilShape>& stencil_presets() {
    static const std::vector<StencilShape> all = {
        {"2d5pt", 2, 5, 1},   {"2d9pt", 2, 9, 1}, {"2d13pt", 2, 13, 3},
        {"2d49pt", 2, 49, 3}, {"3d7pt", 3, 7, 1}, {"3d27pt", 3, 27, 1},
    };
    return all;
}

const StencilShape& stencil_preset(std::string_view name) {
    const auto& all = stencil_presets();
    auto it = std::find_if(all.begin(), all.end(), [&](const StencilShape& s) { return s.name == name; });
    if (it == all.end())
        throw Error(ErrorKind::ValidationError, "unknown stencil preset '" + std::string(name) + "'");
    return *it;
}

std::vector<double> stencil_default_weights(std::string_view name) {
    const StencilShape& s = stencil_preset(name);
    if (s.name == "2d5pt") return {0.5, 0.125, 0.125, 0.125, 0.125};
    if (s.name == "3d7pt") return {0.4, 0.1, 0.1, 0.1, 0.1, 0.1, 0.1};
    // raw = 1/(1 + |dx|+|dy|+|dz|) in canonical offset order, normalised by its sum.
    std::vector<int> manhattan;
    if (s.name == "3d27pt") {
        for (int dz = -1; dz <= 1; ++dz)
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) manhattan.push_back(std::abs(dz) + std::abs(dy) + std::abs(dx));
    } else if (s.name == "2d13pt") {
        manhattan.push_back(0);
        for (int d = 1; d <= 3; ++d)
            for (int k = 0; k < 4; ++k) manhattan.push_back(d);
    } else {
        const int r = s.radius;
        for (int dy = -r; dy <= r; ++dy)
            for (int dx = -r; dx <= r; ++dx) manhattan.push_back(std::abs(dy) + std::abs(dx));
    }
    std::vector<double> w(manhattan.size());
    double sum = 0.0;
    for (std::size_t i = 0; i < w.size(); ++i) {
        w[i] = 1.0 / double(1 + manhattan[i]);
        sum = sum + w[i];
    }
    for (double& x : w) x = x / sum;
    return w;
}

// ---------------------------------------------------------------------------
// Models
// ---------------------------------------------------------------------------
KernelCharacterization scale_model(std::uint64_t n, Precision p) {
    if (!n) throw Error(ErrorKind::InvalidCount, "scale: n_elements must be >= 1");
    return {"scale", n, checked(u128(n) * 2 * element_bytes(p), "scale traffic")};
}

KernelCharacterization gemv_model(std::uint64_t m, std::uint64_t n, Precision p) {
    if (!m || !n) throw Error(ErrorKind::InvalidCount, "gemv: m and n must be >= 1");
    const u128 mn = u128(m) * n;
    return {"gemv", checked(mn * 2, "gemv work"),
            checked((mn + m + n) * element_bytes(p), "gemv traffic")};
}

KernelCharacterization spmv_generic_model(const SparseMatrixStats& s,
                                          const SparseMetadataTraffic& meta, Precision p) {
    s.validate();
    meta.validate();
    const u128 dense = (u128(s.nnz) + s.rows + s.cols) * element_bytes(p);
    const u128 idx = u128(meta.index_entry_count) * meta.index_entry_bytes;
    const u128 packed = u128(meta.packed_entry_count) * meta.packed_entry_bytes;
    return {"spmv", checked(u128(s.nnz) * 2, "spmv work"), checked(dense + idx + packed, "spmv traffic")};
}

KernelCharacterization spmv_csr_model(const SparseMatrixStats& s, std::uint64_t index_bytes,
                                      Precision p) {
    s.validate();
    require_width(index_bytes, false, "csr index_bytes");
    SparseMetadataTraffic meta;
    meta.index_entry_count = checked(u128(s.nnz) + s.rows + 1, "csr index count");
    meta.index_entry_bytes = index_bytes;
    KernelCharacterization k = spmv_generic_model(s, meta, p);
    k.kernel_name = "spmv-csr";
    return k;
}

KernelCharacterization stencil_model(const StencilShape& shape, Precision p, std::uint64_t t) {
    if (!t) throw Error(ErrorKind::InvalidCount, "stencil: temporal depth must be >= 1");
    if (!shape.point_count) throw Error(ErrorKind::InvalidCount, "stencil: point count must be >= 1");
    return {shape.name.empty() ? "stencil" : shape.name,
            checked(u128(t) * 2 * shape.point_count, "stencil work"), 2 * element_bytes(p)};
}

// ---------------------------------------------------------------------------
// Hardware spec
// ---------------------------------------------------------------------------
namespace {
const char* const kUnitName[] = {"CudaCore", "TensorCore"};
const char* const kPrecName[] = {"FP64", "FP32", "FP16"};
const char* const kPrecKey[] = {"fp64", "fp32", "fp16"};
}  // namespace

bool HardwareSpec::has_peak(ExecutionUnit u, Precision p) const {
    return peaks[static_cast<int>(u)][static_cast<int>(p)] != 0.0;
}

double HardwareSpec::peak(ExecutionUnit u, Precision p) const {
    if (!has_peak(u, p))
        throw Error(ErrorKind::MissingPeak, "'" + name + "' has no " + kUnitName[static_cast<int>(u)] +
                                                " peak at " + kPrecName[static_cast<int>(p)]);
    return peaks[static_cast<int>(u)][static_cast<int>(p)];
}

namespace {
// hardware.cpp:91-110 in the reference's order: name, bandwidth, L2, an empty
// table, then each present entry in (unit, precision) map order.
void validate_spec(const std::string& name, double bw, double l2, const double (&peaks)[2][3],
                   const bool (&present)[2][3]) {
    if (name.empty()) throw Error(ErrorKind::ValidationError, "spec name is empty");
    if (!(bw > 0.0)) throw Error(ErrorKind::ValidationError, "'" + name + "': memory_bandwidth must be > 0");
    if (l2 < 0.0) throw Error(ErrorKind::ValidationError, "'" + name + "': l2_cache_bytes must be >= 0");
    bool any = false;
    for (int u = 0; u < 2; ++u)
        for (int p = 0; p < 3; ++p) any = any || present[u][p];
    if (!any) throw Error(ErrorKind::ValidationError, "'" + name + "': peaks table is empty");
    for (int u = 0; u < 2; ++u)
        for (int p = 0; p < 3; ++p) {
            if (!present[u][p]) continue;
            if (!(peaks[u][p] > 0.0))
                throw Error(ErrorKind::ValidationError, "'" + name + "': peak for " + kUnitName[u] + " " +
                                                            kPrecName[p] + " must be > 0");
            if (u == 1 && !present[0][p])
                throw Error(ErrorKind::ValidationError, "'" + name + "': TensorCore peak at " + kPrecName[p] +
                                                            " has no CudaCore counterpart");
        }
}
}  // namespace

void HardwareSpec::validate() const {
    bool present[2][3];
    for (int u = 0; u < 2; ++u)
        for (int p = 0; p < 3; ++p) present[u][p] = peaks[u][p] != 0.0;
    validate_spec(name, memory_bandwidth, l2_cache_bytes, peaks, present);
}

namespace {
double number_field(const nlohmann::json& j, const std::string& key) {
    if (!j.is_number()) throw Error(ErrorKind::ParseError, "'" + key + "' must be a number");
    return j.get<double>();
}

void only_keys(const nlohmann::json& obj, std::initializer_list<std::string_view> allowed,
               const std::string& where) {
    for (auto it = obj.begin(); it != obj.end(); ++it)
        if (std::find(allowed.begin(), allowed.end(), it.key()) == allowed.end())
            throw Error(ErrorKind::ParseError, "unknown key '" + it.key() + "' in " + where);
}

int precision_index(std::string key) {
    std::transform(key.begin(), key.end(), key.begin(), [](unsigned char c) { return std::tolower(c); });
    for (int p = 0; p < 3; ++p)
        if (key == kPrecKey[p]) return p;
    return -1;
}
}  // namespace

HardwareSpec load_spec(const std::string& text) {
    nlohmann::json doc;
    try {
        doc = nlohmann::json::parse(text);
    } catch (const nlohmann::json::exception& e) {
        throw Error(ErrorKind::ParseError, e.what());
    }
    if (!doc.is_object()) throw Error(ErrorKind::ParseError, "spec document must be a JSON object");
    only_keys(doc, {"name", "memory_bandwidth_tbps", "l2_cache_mb", "peaks"}, "spec document");
    for (const char* k : {"name", "memory_bandwidth_tbps", "l2_cache_mb", "peaks"})
        if (!doc.contains(k)) throw Error(ErrorKind::MissingField, std::string("'") + k + "' is required");
    if (!doc["name"].is_string()) throw Error(ErrorKind::ParseError, "'name' must be a string");
    if (!doc["peaks"].is_object()) throw Error(ErrorKind::ParseError, "'peaks' must be a table");

    HardwareSpec s;
    s.name = doc["name"].get<std::string>();
    s.memory_bandwidth = number_field(doc["memory_bandwidth_tbps"], "memory_bandwidth_tbps") * kTera;
    s.l2_cache_bytes = number_field(doc["l2_cache_mb"], "l2_cache_mb") * kMega;
    bool present[2][3] = {};
    for (auto it = doc["peaks"].begin(); it != doc["peaks"].end(); ++it) {
        const int pi = precision_index(it.key());
        if (pi < 0) throw Error(ErrorKind::ParseError, "unknown precision '" + it.key() + "' in peaks");
        if (!it->is_object()) throw Error(ErrorKind::ParseError, "peaks." + it.key() + " must be a table");
        only_keys(*it, {"cuda_core_tflops", "tensor_core_tflops"}, "peaks." + it.key());
        static const char* const field[] = {"cuda_core_tflops", "tensor_core_tflops"};
        for (int u = 0; u < 2; ++u) {
            if (!it->contains(field[u])) continue;
            s.peaks[u][pi] = number_field((*it)[field[u]], "peaks." + it.key() + "." + field[u]) * kTera;
            present[u][pi] = true;
        }
    }
    validate_spec(s.name, s.memory_bandwidth, s.l2_cache_bytes, s.peaks, present);
    return s;
}

HardwareSpec load_spec_file(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw Error(ErrorKind::IoError, "cannot open spec file '" + path + "'");
    std::ostringstream text;
    text << in.rdbuf();
    return load_spec(text.str());
}

std::string serialize_spec(const HardwareSpec& s) {
    nlohmann::json peaks = nlohmann::json::object();
    static const char* const field[] = {"cuda_core_tflops", "tensor_core_tflops"};
    for (int u = 0; u < 2; ++u)
        for (int p = 0; p < 3; ++p)
            if (s.peaks[u][p] != 0.0) peaks[kPrecKey[p]][field[u]] = s.peaks[u][p] / kTera;
    const nlohmann::json doc = {{"name", s.name},
                                {"memory_bandwidth_tbps", s.memory_bandwidth / kTera},
                                {"l2_cache_mb", s.l2_cache_bytes / kMega},
                                {"peaks", peaks}};
    return doc.dump(2) + "\n";
}

const HardwareSpec& builtin_spec(std::string_view name) {
    // Table 1 of the paper, value * unit factor.
    static const HardwareSpec a100 = [] {
        HardwareSpec s;
        s.name = "A100-80GB";
        s.memory_bandwidth = 1.94 * kTera;
        s.l2_cache_bytes = 40.0 * kMega;
        s.peaks[0][0] = 9.7 * kTera;
        s.peaks[1][0] = 19.5 * kTera;
        return s;
    }();
    static const HardwareSpec gh200 = [] {
        HardwareSpec s;
        s.name = "GH200";
        s.memory_bandwidth = 4.00 * kTera;
        s.l2_cache_bytes = 50.0 * kMega;
        s.peaks[0][0] = 34.0 * kTera;
        s.peaks[1][0] = 67.0 * kTera;
        return s;
    }();
    if (name == a100.name) return a100;
    if (name == gh200.name) return gh200;
    throw Error(ErrorKind::UnknownHardware, "no built-in spec named '" + std::string(name) + "'");
}

double machine_balance(const HardwareSpec& s, ExecutionUnit u, Precision p) {
    return s.peak(u, p) / s.memory_bandwidth;
}

double tensor_alpha(const HardwareSpec& s, Precision p) {
    return s.peak(ExecutionUnit::TensorCore, p) / s.peak(ExecutionUnit::CudaCore, p);
}

// ---------------------------------------------------------------------------
// Roofline
// ---------------------------------------------------------------------------
double attainable(const HardwareSpec& s, ExecutionUnit u, Precision p, double intensity) {
    if (intensity < 0.0) throw Error(ErrorKind::InvalidRange, "intensity must be >= 0");
    return std::min(s.peak(u, p), s.memory_bandwidth * intensity);
}

Boundedness classify(double intensity, double balance) {
    return intensity < balance ? Boundedness::MemoryBound
           : intensity > balance ? Boundedness::ComputeBound
                                 : Boundedness::Balanced;
}

// ridge_point / sample_curve (reference roofline.cpp:36-79): n log-spaced
// intensities from i_min to i_max (endpoints exact), the ridge inserted in
// order when it lies inside and is not already a sample.
double ridge_point(const HardwareSpec& s, ExecutionUnit u, Precision p) { return machine_balance(s, u, p); }

std::vector<std::pair<double, double>> sample_curve(const HardwareSpec& s, ExecutionUnit u, Precision p,
                                                    double i_min, double i_max, std::size_t n_points) {
    if (!(i_min > 0.0) || !(i_min < i_max)) throw Error(ErrorKind::InvalidRange, "need 0 < i_min < i_max");
    if (n_points < 2) throw Error(ErrorKind::InvalidRange, "need n_points >= 2");
    std::vector<double> xs;
    xs.reserve(n_points + 1);
    const double lo = std::log(i_min), hi = std::log(i_max);
    for (std::size_t k = 0; k < n_points; ++k) {
        if (k == 0)
            xs.push_back(i_min);
        else if (k == n_points - 1)
            xs.push_back(i_max);
        else
            xs.push_back(std::exp(lo + (static_cast<double>(k) / static_cast<double>(n_points - 1)) * (hi - lo)));
    }
    const double ridge = ridge_point(s, u, p);
    if (ridge >= i_min && ridge <= i_max && std::find(xs.begin(), xs.end(), ridge) == xs.end())
        xs.insert(std::upper_bound(xs.begin(), xs.end(), ridge), ridge);
    std::vector<std::pair<double, double>> out;
    out.reserve(xs.size());
    for (double i : xs) out.emplace_back(i, attainable(s, u, p, i));
    return out;
}

// ---------------------------------------------------------------------------
// Bounds
// ---------------------------------------------------------------------------
namespace {
void need_alpha(double a) {
    if (!(a >= 1.0)) throw Error(ErrorKind::InvalidAlpha, "alpha must be >= 1");
}
void need_intensity(double i) {
    if (!(i > 0.0)) throw Error(ErrorKind::ZeroIntensity, "intensity must be > 0");
}
}  // namespace

static void need_breakdown(double t_cmp, double t_mem, double t_others) {
    if (t_cmp < 0.0 || t_mem < 0.0 || t_others < 0.0)
        throw Error(ErrorKind::ValidationError, "time components must be >= 0");
    if (t_cmp == 0.0 && t_mem == 0.0 && t_others == 0.0)
        throw Error(ErrorKind::ValidationError, "time breakdown is all zero");
}

// mem_cmp_ratio (bounds.cpp:45-48): T_mem / T_cmp = B / I.
double mem_cmp_ratio(double balance, double intensity) {
    need_intensity(intensity);
    return balance / intensity;
}

// overlapped_total (bounds.cpp:50-53): the fully overlapped time.
double overlapped_total(double t_cmp, double t_mem, double t_others) {
    need_breakdown(t_cmp, t_mem, t_others);
    return std::max({t_cmp, t_mem, t_others});
}

double unoverlapped_speedup(double t_cmp, double t_mem, double t_others, double alpha) {
    need_breakdown(t_cmp, t_mem, t_others);
    need_alpha(alpha);
    if (t_cmp == 0.0) return 1.0;
    return (t_cmp + t_mem + t_others) / (t_cmp / alpha + t_mem + t_others);
}

double kernel_speedup_ceiling(double alpha, double balance, double intensity, int* n_warnings) {
    need_alpha(alpha);
    need_intensity(intensity);
    if (n_warnings) *n_warnings = intensity >= balance ? 1 : 0;
    return 1.0 + (alpha - 1.0) / (1.0 + alpha * (balance / intensity));
}

double tensor_core_ceiling(double alpha) {
    need_alpha(alpha);
    return 1.0 + (alpha - 1.0) / (1.0 + alpha);  // lands exactly on 4/3 at alpha = 2
}

double workload_ceiling(double intensity, double balance) {
    need_intensity(intensity);
    if (!(balance > 0.0)) throw Error(ErrorKind::ZeroBalance, "balance must be > 0");
    return 1.0 + intensity / balance;
}

std::uint64_t min_temporal_depth(double balance, double i1) {
    need_intensity(i1);
    if (balance < i1) return 1;
    const double ratio = balance / i1;
    if (!std::isfinite(ratio) || ratio >= 1e18)
        throw Error(ErrorKind::InvalidRange, "balance/intensity ratio too large");
    // smallest t with t * i1 > balance, decided by the multiplication itself
    std::uint64_t t = static_cast<std::uint64_t>(ratio);
    if (t == 0) t = 1;
    while (t > 1 && double(t - 1) * i1 > balance) --t;
    while (!(double(t) * i1 > balance)) ++t;
    return t;
}

double tc_scale_trick_throughput(double peak_tc, std::uint64_t m, std::uint64_t n) {
    if (!m || !n) throw Error(ErrorKind::InvalidCount, "engine dimensions must be >= 1");
    if (!(peak_tc > 0.0)) throw Error(ErrorKind::ValidationError, "peak_tc must be > 0");
    return peak_tc / double(std::max(m, n));
}

}  // namespace rooflens::b200
