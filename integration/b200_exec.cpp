// b200_exec.cpp -- the rooflens-side adapter over librooflens_b200.so
// (INTEGRATION.md §1): C statuses back into rooflens::Error, rl_kchar back
// into KernelCharacterization.  Needs no CUDA headers, nlohmann or torch:
// streams travel as void*.  The reference's ExecutionUnit / Precision
// (hardware.hpp:19-21) have rl_unit / rl_precision's ordinals.
#include "b200_exec.hpp"

#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "rooflens/error.hpp"
#include "rooflens/report.hpp"
#include "rooflens_b200.h"

namespace rooflens {
namespace {

void check(int rc) {
    if (rc == RL_OK) return;
    if (rc >= RL_ERR_KIND_BASE && rc < RL_ERR_KIND_BASE + 17) {
        // strip the "<Kind>: " prefix: rooflens::Error re-adds it
        std::string msg = rl_last_error();
        const auto p = msg.find(": ");
        if (p != std::string::npos) msg = msg.substr(p + 2);
        throw Error(static_cast<ErrorKind>(rc - RL_ERR_KIND_BASE), msg);
    }
    throw std::runtime_error(rl_last_error());  // CUDA (100 + cudaError_t) or NCCL (200 + ncclResult_t)
}

KernelCharacterization kc(const std::string& name, const rl_kchar& k) {
    KernelCharacterization c;
    c.kernel_name = name;
    c.work_flops = k.work_flops;
    c.traffic_bytes = k.traffic_bytes;
    return c;
}

rl_unit U(ExecutionUnit u) { return static_cast<rl_unit>(u); }
rl_precision Pr(Precision p) { return static_cast<rl_precision>(p); }

}  // namespace

KernelCharacterization scale(ExecutionUnit unit, Precision precision, double* a, const double* b, double q,
                             std::uint64_t n, void* stream) {
    rl_kchar k{};
    check(rl_scale(U(unit), Pr(precision), a, b, q, n, stream, &k));
    return kc("scale", k);
}

KernelCharacterization spmv_csr(ExecutionUnit unit, Precision precision, const SparseMatrixStats& s,
                                const std::int32_t* rp, const std::int32_t* col, const double* val,
                                const double* x, double* y, void* stream) {
    rl_kchar k{};
    check(rl_spmv_csr(U(unit), Pr(precision), s.rows, s.cols, s.nnz, rp, col, val, x, y, stream, &k));
    return kc("spmv-csr", k);
}

KernelCharacterization stencil(ExecutionUnit unit, Precision precision, const StencilShape& shape,
                               const std::uint64_t dims[3], const double* weights, std::uint64_t steps, double* u,
                               double* v, void* stream) {
    rl_kchar k{};
    check(rl_stencil(U(unit), Pr(precision), shape.name.c_str(), dims, weights, steps, u, v, stream, &k));
    return kc(shape.name, k);
}

KernelCharacterization stencil_temporal(ExecutionUnit unit, Precision precision, const StencilShape& shape,
                                        const std::uint64_t dims[3], const double* weights, std::uint64_t steps,
                                        std::uint64_t t, double* u, double* v, void* stream, bool* result_in_v) {
    rl_kchar k{};
    int in_v = 0;
    check(rl_stencil_temporal(U(unit), Pr(precision), shape.name.c_str(), dims, weights, steps, t, u, v, stream,
                              &in_v, &k));
    if (result_in_v) *result_in_v = in_v != 0;
    return kc(shape.name, k);
}

SpmvPlan::SpmvPlan(ExecutionUnit unit, Precision precision, const SparseMatrixStats& s, const std::int32_t* rp,
                   const std::int32_t* col, const double* val) {
    rl_spmv_plan p = nullptr;
    check(rl_spmv_plan_create(U(unit), Pr(precision), s.rows, s.cols, s.nnz, rp, col, val, &p));
    h_ = p;
}
SpmvPlan::~SpmvPlan() {
    if (h_) rl_spmv_plan_destroy(static_cast<rl_spmv_plan>(h_));
}
KernelCharacterization SpmvPlan::execute_host(const double* x, double* y) {
    rl_kchar k{};
    check(rl_spmv_plan_execute_host(static_cast<rl_spmv_plan>(h_), x, y, &k));
    return kc("spmv-csr", k);
}
KernelCharacterization SpmvPlan::execute(const double* x, double* y, void* stream) {
    rl_kchar k{};
    check(rl_spmv_plan_execute(static_cast<rl_spmv_plan>(h_), x, y, stream, &k));
    return kc("spmv-csr", k);
}
std::string SpmvPlan::layout() const {
    int l = 0;
    check(rl_spmv_plan_info(static_cast<rl_spmv_plan>(h_), &l, nullptr));
    return l == 4 ? "colsort" : "csr";
}

void B200Comm::unique_id(std::uint8_t id[128]) { check(rl_dist_unique_id(id)); }

B200Comm::B200Comm(int world, int rank, const std::uint8_t id[128]) {
    rl_dist d = nullptr;
    check(rl_dist_init(world, rank, id, &d));
    h_ = d;
}

B200Comm::~B200Comm() {
    if (h_) rl_dist_destroy(static_cast<rl_dist>(h_));
}

KernelCharacterization dist_scale(const B200Comm& comm, ExecutionUnit unit, Precision precision, double* a,
                                  const double* b, double q, std::uint64_t n_global, void* stream) {
    rl_kchar k{};
    check(rl_dist_scale(static_cast<rl_dist>(comm.handle()), U(unit), Pr(precision), a, b, q, n_global, stream, &k));
    return kc("scale", k);
}

DistSpmv::DistSpmv(const B200Comm& comm, ExecutionUnit unit, Precision precision, std::uint64_t n, std::uint64_t hb,
                   const std::int32_t* rp, const std::int32_t* col, const double* val, double* x, double* y) {
    rl_dist_spmv p = nullptr;
    check(rl_dist_spmv_create(static_cast<rl_dist>(comm.handle()), U(unit), Pr(precision), n, hb, 1, &rp, &col, &val,
                              &x, &y, &p));
    h_ = p;
}
DistSpmv::~DistSpmv() {
    if (h_) rl_dist_spmv_destroy(static_cast<rl_dist_spmv>(h_));
}
KernelCharacterization DistSpmv::execute(void* stream) {
    rl_kchar k{};
    check(rl_dist_spmv_execute(static_cast<rl_dist_spmv>(h_), stream, &k));
    return kc("spmv-csr", k);
}

DistStencil::DistStencil(const B200Comm& comm, ExecutionUnit unit, Precision precision, const StencilShape& shape,
                         const std::uint64_t dims[3], const double* weights, double* u, double* v)
    : name_(shape.name) {
    rl_dist_stencil p = nullptr;
    check(rl_dist_stencil_create(static_cast<rl_dist>(comm.handle()), U(unit), Pr(precision), shape.name.c_str(), dims,
                                 weights, 1, &u, &v, &p));
    h_ = p;
}
DistStencil::~DistStencil() {
    if (h_) rl_dist_stencil_destroy(static_cast<rl_dist_stencil>(h_));
}
KernelCharacterization DistStencil::run(std::uint64_t steps, void* stream, bool* result_in_v) {
    rl_kchar k{};
    int in_v = 0;
    check(rl_dist_stencil_run(static_cast<rl_dist_stencil>(h_), steps, stream, &in_v, &k));
    if (result_in_v) *result_in_v = in_v != 0;
    return kc(name_, k);
}

// ---------------------------------------------------------------------------
// report.hpp:40-48.  The reference declares build_analysis / render_* without
// defining them; librooflens_b200.so implements them (csrc/report.cpp) and
// this adapter supplies the reference's symbols over it.
// ---------------------------------------------------------------------------
namespace {

rl_hw_spec c_spec(const HardwareSpec& h) {
    rl_hw_spec s{};
    std::strncpy(s.name, h.name.c_str(), sizeof s.name - 1);
    s.memory_bandwidth = h.memory_bandwidth;
    s.l2_cache_bytes = h.l2_cache_bytes;
    for (const auto& [key, peak] : h.peaks)
        s.peaks[static_cast<int>(key.first)][static_cast<int>(key.second)] = peak;
    return s;
}

template <class F>
SpeedupBound bound_of(F&& call) {
    rl_speedup_bound b{};
    uint64_t n = 0;
    check(call(&b, nullptr, 0, &n));
    std::string text(n + 1, '\0');
    check(call(&b, text.data(), n + 1, nullptr));
    SpeedupBound r;
    r.value = b.value;
    r.kind = static_cast<BoundKind>(b.kind);
    std::size_t at = 0;
    for (int i = 0; i < b.n_assumptions + b.n_warnings; ++i) {
        const std::size_t nl = text.find('\n', at);
        (i < b.n_assumptions ? r.assumptions : r.warnings).push_back(text.substr(at, nl - at));
        at = nl + 1;
    }
    return r;
}

std::string render(const AnalysisReport& r, int format) {
    const rl_hw_spec s = c_spec(r.machine);
    const double* bo = r.balance_overridden ? &r.balance : nullptr;
    const double* si = r.single_step_intensity ? &*r.single_step_intensity : nullptr;
    uint64_t n = 0;
    auto call = [&](char* buf, uint64_t cap, uint64_t* len) {
        return rl_analysis_render(&s, Pr(r.precision), r.kernel.kernel_name.c_str(), r.kernel.work_flops,
                                  r.kernel.traffic_bytes, bo, si, format, buf, cap, len);
    };
    check(call(nullptr, 0, &n));
    std::string out(n + 1, '\0');
    check(call(out.data(), n + 1, nullptr));
    out.resize(n);
    return out;
}

// (field, value) rows of the csv encoding (RFC-4180 quoting).
std::vector<std::pair<std::string, std::string>> csv_rows(const std::string& text) {
    std::vector<std::pair<std::string, std::string>> rows;
    std::vector<std::string> cells;
    std::string cell;
    bool quoted = false;
    for (std::size_t i = 0; i < text.size(); ++i) {
        const char c = text[i];
        if (quoted) {
            if (c == '"' && i + 1 < text.size() && text[i + 1] == '"') cell += '"', ++i;
            else if (c == '"') quoted = false;
            else cell += c;
        } else if (c == '"') {
            quoted = true;
        } else if (c == ',') {
            cells.push_back(cell), cell.clear();
        } else if (c == '\n') {
            cells.push_back(cell), cell.clear();
            if (cells.size() == 2) rows.emplace_back(cells[0], cells[1]);
            cells.clear();
        } else {
            cell += c;
        }
    }
    return rows;
}

}  // namespace

AnalysisReport build_analysis(const HardwareSpec& spec, Precision precision, const KernelCharacterization& kernel,
                              std::optional<double> balance_override, std::optional<double> single_step_intensity) {
    const rl_hw_spec s = c_spec(spec);
    AnalysisReport r;
    r.machine = spec;
    r.precision = precision;
    r.kernel = kernel;
    r.balance_overridden = balance_override.has_value();
    r.single_step_intensity = single_step_intensity;
    if (balance_override) r.balance = *balance_override;
    // the library validates everything (spec, intensity, override) and
    // carries the notes and verdict; the numbers come from the same C-ABI
    for (const auto& [field, value] : csv_rows(render(r, RL_REPORT_CSV))) {
        if (field == "note") r.notes.push_back(value);
        else if (field == "verdict") r.verdict = value;
    }
    if (!balance_override) check(rl_machine_balance(&s, RL_CUDA_CORE, Pr(precision), &r.balance));
    const double I = kernel.intensity();
    r.boundedness = static_cast<Boundedness>(rl_classify(I, r.balance));
    if (spec.has_peak(ExecutionUnit::TensorCore, precision)) {
        check(rl_tensor_alpha(&s, Pr(precision), &r.alpha));
        const double a = r.alpha < 1.0 ? 1.0 : r.alpha;
        const double B = r.balance;
        r.bounds.push_back(bound_of([&](rl_speedup_bound* b, char* t, uint64_t c, uint64_t* l) {
            return rl_kernel_ceiling_bound(a, B, I, b, t, c, l);
        }));
        r.bounds.push_back(bound_of([&](rl_speedup_bound* b, char* t, uint64_t c, uint64_t* l) {
            return rl_tensor_core_bound(a, b, t, c, l);
        }));
    }
    r.bounds.push_back(bound_of([&](rl_speedup_bound* b, char* t, uint64_t c, uint64_t* l) {
        return rl_workload_bound(I, r.balance, b, t, c, l);
    }));
    if (single_step_intensity) {
        std::uint64_t t = 0;
        check(rl_min_temporal_depth(r.balance, *single_step_intensity, &t));
        r.min_depth = t;
    }
    return r;
}

std::string render_text(const AnalysisReport& r) { return render(r, RL_REPORT_TEXT); }
std::string render_json(const AnalysisReport& r) { return render(r, RL_REPORT_JSON); }
std::string render_csv(const AnalysisReport& r) { return render(r, RL_REPORT_CSV); }

}  // namespace rooflens
