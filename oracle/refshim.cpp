// refshim.cpp -- extern "C" shim over the UNMODIFIED reference library
// (rooflens, /root/reference/proj/src/*.cpp), compiled together with it by
// oracle/Makefile into oracle/_ref/librooflens_ref.so.
//
// TEST INFRASTRUCTURE ONLY: the reference's symbols are C++-mangled and return
// std::string/std::map-owning structs, so ctypes cannot call them directly.
// This shim flattens them for tests/ (accounting parity of the product's
// rl_kchar against the reference's own models) and for tests/golden/make_golden.py.
// It contains no arithmetic of its own: every value comes from the reference.
//
// Return convention mirrors the product C-ABI: 0 = OK, 1 + ErrorKind ordinal
// (reference error.hpp:10-32) on a rooflens::Error.
#include <cstdint>
#include <cstring>
#include <string>

#include "rooflens/bounds.hpp"
#include "rooflens/error.hpp"
#include "rooflens/hardware.hpp"
#include "rooflens/kernels.hpp"
#include "rooflens/matrix_market.hpp"
#include "rooflens/roofline.hpp"

using namespace rooflens;

namespace {
thread_local std::string g_last;

template <class F>
int guarded(F&& f) {
    try {
        f();
        g_last.clear();
        return 0;
    } catch (const Error& e) {
        g_last = e.what();
        return 1 + static_cast<int>(e.kind());
    } catch (const std::exception& e) {
        g_last = e.what();
        return 99;
    }
}

Precision prec_of(int p) { return static_cast<Precision>(p); }
ExecutionUnit unit_of(int u) { return static_cast<ExecutionUnit>(u); }

void out_kc(const KernelCharacterization& k, uint64_t* w, uint64_t* q) {
    *w = k.work_flops;
    *q = k.traffic_bytes;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_last.c_str(); }

int ref_scale_model(uint64_t n, int prec, uint64_t* w, uint64_t* q) {
    return guarded([&] { out_kc(scale_model(n, prec_of(prec)), w, q); });
}

int ref_gemv_model(uint64_t m, uint64_t n, int prec, uint64_t* w, uint64_t* q) {
    return guarded([&] { out_kc(gemv_model(m, n, prec_of(prec)), w, q); });
}

int ref_spmv_generic_model(uint64_t m, uint64_t n, uint64_t nnz, uint64_t idx_count,
                           uint64_t idx_bytes, uint64_t packed_count, uint64_t packed_bytes,
                           int prec, uint64_t* w, uint64_t* q) {
    return guarded([&] {
        SparseMatrixStats s{m, n, nnz};
        SparseMetadataTraffic meta{idx_count, idx_bytes, packed_count, packed_bytes};
        out_kc(spmv_generic_model(s, meta, prec_of(prec)), w, q);
    });
}

int ref_spmv_csr_model(uint64_t m, uint64_t n, uint64_t nnz, uint64_t index_bytes, int prec,
                       uint64_t* w, uint64_t* q) {
    return guarded([&] {
        SparseMatrixStats s{m, n, nnz};
        out_kc(spmv_csr_model(s, index_bytes, prec_of(prec)), w, q);
    });
}

int ref_stencil_model(const char* preset, int prec, uint64_t t, uint64_t* w, uint64_t* q,
                      uint64_t* points) {
    return guarded([&] {
        const StencilShape& s = stencil_preset(preset);
        *points = s.point_count;
        out_kc(stencil_model(s, prec_of(prec), t), w, q);
    });
}

int ref_intensity_ratio(uint64_t w, uint64_t q, uint64_t* num, uint64_t* den) {
    return guarded([&] {
        Ratio r = Ratio::of(w, q);
        *num = r.num;
        *den = r.den;
    });
}

// Spec from a JSON document (reference hardware.cpp:183-237); returns the
// FP64 figures (0 where absent) in SI units.
int ref_load_spec(const char* text, double* bw, double* l2, double* p_cc, double* p_tc) {
    return guarded([&] {
        HardwareSpec s = load_spec(text);
        *bw = s.memory_bandwidth;
        *l2 = s.l2_cache_bytes;
        *p_cc = s.has_peak(ExecutionUnit::CudaCore, Precision::FP64)
                    ? s.peak(ExecutionUnit::CudaCore, Precision::FP64) : 0.0;
        *p_tc = s.has_peak(ExecutionUnit::TensorCore, Precision::FP64)
                    ? s.peak(ExecutionUnit::TensorCore, Precision::FP64) : 0.0;
    });
}

int ref_builtin_spec(const char* name, double* bw, double* l2, double* p_cc, double* p_tc) {
    return guarded([&] {
        const HardwareSpec& s = builtin_spec(name);
        *bw = s.memory_bandwidth;
        *l2 = s.l2_cache_bytes;
        *p_cc = s.peak(ExecutionUnit::CudaCore, Precision::FP64);
        *p_tc = s.peak(ExecutionUnit::TensorCore, Precision::FP64);
    });
}

// Balance / alpha / roofline on an FP64 spec built from explicit SI figures.
static HardwareSpec mk(double bw, double p_cc, double p_tc) {
    HardwareSpec s;
    s.name = "probe";
    s.memory_bandwidth = bw;
    s.l2_cache_bytes = 0.0;
    s.peaks[{ExecutionUnit::CudaCore, Precision::FP64}] = p_cc;
    if (p_tc > 0.0) s.peaks[{ExecutionUnit::TensorCore, Precision::FP64}] = p_tc;
    return s;
}

int ref_machine_balance(double bw, double p_cc, double p_tc, int unit, double* out) {
    return guarded([&] { *out = machine_balance(mk(bw, p_cc, p_tc), unit_of(unit), Precision::FP64); });
}

int ref_tensor_alpha(double bw, double p_cc, double p_tc, double* out) {
    return guarded([&] { *out = tensor_alpha(mk(bw, p_cc, p_tc), Precision::FP64); });
}

int ref_attainable(double bw, double p_cc, double p_tc, int unit, double intensity, double* out) {
    return guarded([&] {
        *out = attainable(mk(bw, p_cc, p_tc), unit_of(unit), Precision::FP64, intensity);
    });
}

// Any (unit, precision) on a spec loaded from a JSON document (the full
// reference peak table): what 0 machine_balance, 1 tensor_alpha, 2 attainable
// at `intensity`, 3 ridge_point.
int ref_spec_eval(const char* doc, int what, int unit, int prec, double intensity, double* out) {
    return guarded([&] {
        const HardwareSpec s = load_spec(doc);
        if (what == 0) *out = machine_balance(s, unit_of(unit), prec_of(prec));
        else if (what == 1) *out = tensor_alpha(s, prec_of(prec));
        else if (what == 2) *out = attainable(s, unit_of(unit), prec_of(prec), intensity);
        else *out = ridge_point(s, unit_of(unit), prec_of(prec));
    });
}

// serialize_spec(load_spec(doc)) into buf (cap bytes incl. NUL).
int ref_serialize_spec(const char* doc, char* buf, uint64_t cap) {
    return guarded([&] {
        const std::string t = serialize_spec(load_spec(doc));
        if (t.size() + 1 > cap) throw Error(ErrorKind::InvalidRange, "capacity");
        std::memcpy(buf, t.c_str(), t.size() + 1);
    });
}

int ref_load_spec_file(const char* path, double* bw) {
    return guarded([&] { *bw = load_spec_file(path).memory_bandwidth; });
}

int ref_classify(double intensity, double balance) {
    return static_cast<int>(classify(intensity, balance));
}

// sample_curve (roofline.cpp:40-79) into caller arrays of `cap` entries.
int ref_sample_curve(double bw, double p_cc, double p_tc, int unit, double i_min, double i_max,
                     uint64_t n, double* xs, double* ys, uint64_t cap, uint64_t* count) {
    return guarded([&] {
        const auto pts = sample_curve(mk(bw, p_cc, p_tc), unit_of(unit), Precision::FP64, i_min, i_max,
                                      (std::size_t)n);
        if (pts.size() > cap) throw Error(ErrorKind::InvalidRange, "capacity");
        for (std::size_t k = 0; k < pts.size(); ++k) {
            xs[k] = pts[k].intensity;
            ys[k] = pts[k].attainable;
        }
        *count = pts.size();
    });
}

int ref_kernel_speedup_ceiling(double alpha, double balance, double intensity, double* out,
                               int* n_warnings) {
    return guarded([&] {
        SpeedupBound b = kernel_speedup_ceiling(alpha, balance, intensity);
        *out = b.value;
        *n_warnings = static_cast<int>(b.warnings.size());
    });
}

// The reference's SpeedupBound for bound `kind` (0 unoverlapped(t_cmp=a,
// t_mem=b, t_others=c, alpha=d), 1 kernel ceiling(a=alpha, b=balance,
// c=intensity), 2 tensor-core ceiling(a=alpha), 3 workload ceiling(a=I,
// b=balance)): value, BoundKind, to_string(kind) and its assumption and
// warning lines ('\n'-terminated) into text.
int ref_bound_text(int kind, double a, double b, double c, double d, double* value, int* bkind,
                   int* n_assumptions, int* n_warnings, char* text, uint64_t cap, char* kind_name,
                   uint64_t kind_cap) {
    return guarded([&] {
        SpeedupBound r = kind == 0   ? unoverlapped_bound(TimeBreakdown{a, b, c}, d)
                         : kind == 1 ? kernel_speedup_ceiling(a, b, c)
                         : kind == 2 ? tensor_core_ceiling(a)
                                     : workload_ceiling(a, b);
        *value = r.value;
        *bkind = static_cast<int>(r.kind);
        *n_assumptions = static_cast<int>(r.assumptions.size());
        *n_warnings = static_cast<int>(r.warnings.size());
        std::string t;
        for (auto& x : r.assumptions) t += x + "\n";
        for (auto& x : r.warnings) t += x + "\n";
        if (t.size() + 1 > cap) throw Error(ErrorKind::InvalidRange, "capacity");
        std::memcpy(text, t.c_str(), t.size() + 1);
        std::string kn = to_string(r.kind);
        if (kn.size() + 1 > kind_cap) throw Error(ErrorKind::InvalidRange, "capacity");
        std::memcpy(kind_name, kn.c_str(), kn.size() + 1);
    });
}

int ref_tensor_core_ceiling(double alpha, double* out) {
    return guarded([&] { *out = tensor_core_ceiling(alpha).value; });
}

int ref_workload_ceiling(double intensity, double balance, double* out) {
    return guarded([&] { *out = workload_ceiling(intensity, balance).value; });
}

int ref_unoverlapped_speedup(double t_cmp, double t_mem, double t_others, double alpha,
                             double* out) {
    return guarded([&] { *out = unoverlapped_speedup(TimeBreakdown{t_cmp, t_mem, t_others}, alpha); });
}

int ref_mem_cmp_ratio(double balance, double intensity, double* out) {
    return guarded([&] { *out = mem_cmp_ratio(balance, intensity); });
}

int ref_overlapped_total(double t_cmp, double t_mem, double t_others, double* out) {
    return guarded([&] { *out = overlapped_total(TimeBreakdown{t_cmp, t_mem, t_others}); });
}

int ref_min_temporal_depth(double balance, double intensity, uint64_t* out) {
    return guarded([&] { *out = min_temporal_depth(balance, intensity); });
}

int ref_tc_scale_trick_throughput(double peak_tc, uint64_t m, uint64_t n, double* out) {
    return guarded([&] { *out = tc_scale_trick_throughput(peak_tc, m, n); });
}

int ref_parse_stats_file(const char* path, uint64_t* rows, uint64_t* cols, uint64_t* nnz) {
    return guarded([&] {
        SparseMatrixStats s = parse_stats_file(path);
        *rows = s.rows;
        *cols = s.cols;
        *nnz = s.nnz;
    });
}

// stats_to_report on an FP64 spec built from SI figures.
int ref_stats_to_report(uint64_t rows, uint64_t cols, uint64_t nnz, double bw, double l2, double p_cc,
                        double p_tc, uint64_t* w, uint64_t* q, int* bound, double* kceil, int* kwarn,
                        double* wceil, uint64_t* csr_bytes, int* fits) {
    return guarded([&] {
        HardwareSpec s = mk(bw, p_cc, p_tc);
        s.l2_cache_bytes = l2;
        MatrixAnalysis a = stats_to_report(SparseMatrixStats{rows, cols, nnz}, s, Precision::FP64);
        *w = a.kernel.work_flops;
        *q = a.kernel.traffic_bytes;
        *bound = static_cast<int>(a.boundedness);
        *kceil = a.kernel_ceiling.value;
        *kwarn = static_cast<int>(a.kernel_ceiling.warnings.size());
        *wceil = a.workload_ceiling.value;
        *csr_bytes = a.csr_bytes;
        *fits = a.fits_in_l2 ? 1 : 0;
    });
}

}  // extern "C"
