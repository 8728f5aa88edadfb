// report.cpp -- reportable speedup bounds and the per-kernel analysis report.
//
//   SpeedupBound objects      reference bounds.hpp:27-45, bounds.cpp:23-108
//                             (same value, kind, assumption and warning text)
//   AnalysisReport            reference report.hpp:19-48 declares
//   build_analysis/render_*   build_analysis and render_text/json/csv but
//                             ships no implementation; the behaviour follows
//                             SPEC.md cli_report (verdict = min applicable
//                             bound to 3 significant digits; text 4
//                             significant digits, json/csv full precision;
//                             byte-deterministic output).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <sstream>

#include <json.hpp>

#include "../../include/rooflens_b200.hpp"

namespace rooflens::b200 {

namespace {
const char* kOpenBound = "open bound: stored value is the supremum";

const char* precision_name(Precision p) {
    return p == Precision::FP64 ? "FP64" : p == Precision::FP32 ? "FP32" : "FP16";
}
const char* unit_name(ExecutionUnit u) { return u == ExecutionUnit::CudaCore ? "CudaCore" : "TensorCore"; }
const char* boundedness_name(Boundedness b) {
    return b == Boundedness::MemoryBound ? "memory-bound"
           : b == Boundedness::ComputeBound ? "compute-bound"
                                            : "balanced";
}

std::string sig(double v, int digits) {
    char buf[64];
    std::snprintf(buf, sizeof buf, "%.*g", digits, v);
    return buf;
}
// Shortest "%.Ng" that reads back as the same double.
std::string full(double v) {
    for (int d = 15; d < 17; ++d) {
        std::string t = sig(v, d);
        if (std::strtod(t.c_str(), nullptr) == v) return t;
    }
    return sig(v, 17);
}
}  // namespace

const char* to_string(BoundKind kind) {
    switch (kind) {
        case BoundKind::ExactUnoverlapped: return "exact un-overlapped";
        case BoundKind::KernelCeiling: return "kernel ceiling";
        case BoundKind::TensorCoreCeiling: return "tensor-core ceiling";
        case BoundKind::WorkloadCeiling: return "workload ceiling";
    }
    return "?";
}

SpeedupBound unoverlapped_bound(double t_cmp, double t_mem, double t_others, double alpha) {
    SpeedupBound b;
    b.value = unoverlapped_speedup(t_cmp, t_mem, t_others, alpha);
    b.kind = BoundKind::ExactUnoverlapped;
    b.assumptions = {"fully un-overlapped", "exact speedup for this breakdown"};
    return b;
}

SpeedupBound kernel_ceiling_bound(double alpha, double balance, double intensity) {
    SpeedupBound b;
    int nw = 0;
    b.value = kernel_speedup_ceiling(alpha, balance, intensity, &nw);
    b.kind = BoundKind::KernelCeiling;
    b.assumptions = {"fully un-overlapped", "T_others >= 0", "T_mem = T_cmp * B/I (throughput-bound)",
                     kOpenBound};
    if (nw)
        b.warnings.push_back("intensity >= machine balance: kernel is not memory-bound, ceiling is not meaningful");
    return b;
}

SpeedupBound tensor_core_bound(double alpha) {
    SpeedupBound b;
    b.value = tensor_core_ceiling(alpha);
    b.kind = BoundKind::TensorCoreCeiling;
    b.assumptions = {"fully un-overlapped", "memory-bound premise: T_cmp -> T_mem", kOpenBound};
    return b;
}

SpeedupBound workload_bound(double intensity, double balance) {
    SpeedupBound b;
    b.value = workload_ceiling(intensity, balance);
    b.kind = BoundKind::WorkloadCeiling;
    b.assumptions = {"alpha -> infinity", "fully un-overlapped", kOpenBound};
    return b;
}

// The classification balance is the CUDA-core balance at `precision` (or the
// override); the tensor-core bounds need a tensor-core peak at `precision`
// and are evaluated at max(alpha, 1) (a slower matrix engine is not an
// accelerator; the note says so).  The verdict's X is the minimum over the
// bounds in the report.
AnalysisReport build_analysis(const HardwareSpec& spec, Precision precision, const KernelCharacterization& kernel,
                              std::optional<double> balance_override, std::optional<double> single_step_intensity) {
    spec.validate();
    if (!kernel.traffic_bytes) throw Error(ErrorKind::ValidationError, "kernel traffic_bytes must be > 0");
    AnalysisReport r;
    r.machine = spec;
    r.precision = precision;
    r.kernel = kernel;
    if (balance_override) {
        if (!(*balance_override > 0.0) || !std::isfinite(*balance_override))
            throw Error(ErrorKind::ZeroBalance, "balance override must be a finite value > 0");
        r.balance = *balance_override;
        r.balance_overridden = true;
    } else {
        r.balance = machine_balance(spec, ExecutionUnit::CudaCore, precision);
    }
    const double I = kernel.intensity();
    r.boundedness = classify(I, r.balance);
    r.attainable_flops = attainable(spec, ExecutionUnit::CudaCore, precision, I);
    if (spec.peaks[1][static_cast<int>(precision)] > 0.0) {
        const double alpha = tensor_alpha(spec, precision);
        r.alpha = alpha;
        const double a = std::max(alpha, 1.0);
        if (alpha < 1.0) r.notes.push_back("alpha < 1: tensor-core ceilings evaluated at alpha = 1");
        r.bounds.push_back(kernel_ceiling_bound(a, r.balance, I));
        r.bounds.push_back(tensor_core_bound(a));
    } else {
        r.notes.push_back(std::string("no ") + precision_name(precision) +
                          " tensor-core peak in the spec: kernel and tensor-core ceilings omitted");
    }
    r.bounds.push_back(workload_bound(I, r.balance));
    if (single_step_intensity) {
        r.single_step_intensity = *single_step_intensity;
        r.min_depth = min_temporal_depth(r.balance, *single_step_intensity);
        r.notes.push_back("temporal depth is a lower bound: register and shared-memory pressure limit the "
                          "practical depth (PAPER.md section 3.3)");
    }
    double x = r.bounds.front().value;
    for (const SpeedupBound& b : r.bounds) x = std::min(x, b.value);
    r.notes.push_back("partial overlap is not modelled: measured speedups lie in [1, " + sig(x, 3) + "]");
    r.verdict = "tensor cores cannot exceed " + sig(x, 3) + "x on this kernel/machine";
    return r;
}

namespace {
// (field, value) rows shared by the text and csv encodings; `fmt` renders a
// double (4 significant digits for text, round-trip for csv).
template <class Fmt>
std::vector<std::pair<std::string, std::string>> report_rows(const AnalysisReport& r, Fmt fmt) {
    std::vector<std::pair<std::string, std::string>> rows = {
        {"machine", r.machine.name},
        {"precision", precision_name(r.precision)},
        {"kernel", r.kernel.kernel_name},
        {"work_flops", std::to_string(r.kernel.work_flops)},
        {"traffic_bytes", std::to_string(r.kernel.traffic_bytes)},
        {"intensity", fmt(r.kernel.intensity())},
        {"balance", fmt(r.balance)},
        {"balance_overridden", r.balance_overridden ? "true" : "false"},
        {"boundedness", boundedness_name(r.boundedness)},
        {"attainable_flops", fmt(r.attainable_flops)},
    };
    if (r.alpha) rows.emplace_back("alpha", fmt(*r.alpha));
    for (const SpeedupBound& b : r.bounds) rows.emplace_back(to_string(b.kind), fmt(b.value));
    if (r.single_step_intensity) rows.emplace_back("single_step_intensity", fmt(*r.single_step_intensity));
    if (r.min_depth) rows.emplace_back("min_temporal_depth", std::to_string(*r.min_depth));
    for (const SpeedupBound& b : r.bounds)
        for (const std::string& w : b.warnings) rows.emplace_back("warning", std::string(to_string(b.kind)) + ": " + w);
    for (const std::string& n : r.notes) rows.emplace_back("note", n);
    rows.emplace_back("verdict", r.verdict);
    return rows;
}

std::string csv_field(const std::string& s) {
    if (s.find_first_of(",\"\n") == std::string::npos) return s;
    std::string out = "\"";
    for (char c : s) {
        if (c == '"') out += '"';
        out += c;
    }
    return out + "\"";
}
}  // namespace

std::string render_text(const AnalysisReport& r) {
    auto rows = report_rows(r, [](double v) { return sig(v, 4); });
    std::size_t w = 0;
    for (auto& kv : rows) w = std::max(w, kv.first.size());
    std::ostringstream os;
    for (auto& kv : rows) os << kv.first << std::string(w - kv.first.size() + 2, ' ') << kv.second << '\n';
    return os.str();
}

std::string render_csv(const AnalysisReport& r) {
    std::ostringstream os;
    os << "field,value\n";
    for (auto& kv : report_rows(r, full)) os << csv_field(kv.first) << ',' << csv_field(kv.second) << '\n';
    return os.str();
}

std::string render_json(const AnalysisReport& r) {
    using nlohmann::ordered_json;
    ordered_json m;
    m["name"] = r.machine.name;
    m["memory_bandwidth"] = r.machine.memory_bandwidth;
    m["l2_cache_bytes"] = r.machine.l2_cache_bytes;
    ordered_json peaks = ordered_json::object();
    for (int u = 0; u < 2; ++u)
        for (int p = 0; p < 3; ++p)
            if (r.machine.peaks[u][p] > 0.0)
                peaks[std::string(unit_name(ExecutionUnit(u))) + "/" + precision_name(Precision(p))] =
                    r.machine.peaks[u][p];
    m["peaks"] = peaks;
    ordered_json j;
    j["machine"] = m;
    j["precision"] = precision_name(r.precision);
    j["balance"] = r.balance;
    j["balance_overridden"] = r.balance_overridden;
    if (r.alpha) j["alpha"] = *r.alpha;
    j["kernel"] = {{"name", r.kernel.kernel_name},
                   {"work_flops", r.kernel.work_flops},
                   {"traffic_bytes", r.kernel.traffic_bytes},
                   {"intensity", r.kernel.intensity()}};
    j["boundedness"] = boundedness_name(r.boundedness);
    j["attainable_flops"] = r.attainable_flops;
    ordered_json bounds = ordered_json::array();
    for (const SpeedupBound& b : r.bounds)
        bounds.push_back({{"kind", to_string(b.kind)},
                          {"value", b.value},
                          {"assumptions", b.assumptions},
                          {"warnings", b.warnings}});
    j["bounds"] = bounds;
    if (r.single_step_intensity) j["single_step_intensity"] = *r.single_step_intensity;
    if (r.min_depth) j["min_temporal_depth"] = *r.min_depth;
    j["notes"] = r.notes;
    j["verdict"] = r.verdict;
    return j.dump(1) + "\n";
}

}  // namespace rooflens::b200
