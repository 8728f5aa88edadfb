// integration_main.cpp -- drives integration/b200_exec.cpp compiled against
// the reference's headers (tests/test_integration.py).  Prints one line per
// probe: "<probe> <outcome>" where outcome is ok:<W>/<Q>, the rooflens
// ErrorKind ordinal as kind:<k>, or runtime:<text> for a CUDA / NCCL status.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <string>

#include "b200_exec.hpp"
#include "rooflens/bounds.hpp"
#include "rooflens/error.hpp"
#include "rooflens/report.hpp"

using namespace rooflens;

static void probe(const char* name, const std::function<KernelCharacterization()>& f) {
    try {
        const KernelCharacterization k = f();
        std::printf("%s ok:%llu/%llu:%s\n", name, (unsigned long long)k.work_flops,
                    (unsigned long long)k.traffic_bytes, k.kernel_name.c_str());
    } catch (const Error& e) {
        std::printf("%s kind:%d:%s\n", name, static_cast<int>(e.kind()), e.what());
    } catch (const std::exception& e) {
        std::printf("%s runtime:%s\n", name, e.what());
    }
}

int main() {
    double a[8] = {}, b[8] = {1, 2, 3, 4, 5, 6, 7, 8};
    // precision the B200 kernels do not run: rooflens::Error(ValidationError)
    probe("scale_fp32", [&] { return scale(ExecutionUnit::CudaCore, Precision::FP32, a, b, 3.0, 8, nullptr); });
    // a null buffer: ValidationError before any device work
    probe("scale_null", [&] { return scale(ExecutionUnit::TensorCore, Precision::FP64, nullptr, b, 3.0, 8, nullptr); });
    // model validation the reference itself would raise (nnz > rows*cols): ValidationError
    SparseMatrixStats bad{2, 2, 5};
    probe("spmv_bad_stats", [&] {
        return spmv_csr(ExecutionUnit::CudaCore, Precision::FP64, bad, nullptr, nullptr, nullptr, nullptr, nullptr,
                        nullptr);
    });
    // unknown stencil preset name
    StencilShape odd;
    odd.name = "9d99pt";
    std::uint64_t dims[3] = {8, 8, 8};
    probe("stencil_unknown", [&] {
        return stencil(ExecutionUnit::CudaCore, Precision::FP64, odd, dims, nullptr, 1, a, b, nullptr);
    });
    // the reference's own models on the same arguments (same kind and text)
    probe("ref_spmv_bad_stats", [&] { return spmv_csr_model(bad, 4, Precision::FP64); });
    probe("ref_stencil_unknown", [&] { return stencil_model(stencil_preset("9d99pt"), Precision::FP64, 1); });
    // valid arguments: executes on a GPU; on a machine without one it is a
    // CUDA status (std::runtime_error), never a CPU fallback.  Host buffers
    // here, so only probed when the caller says no device is present.
    if (std::getenv("RL_PROBE_NO_DEVICE"))
        probe("scale_exec", [&] { return scale(ExecutionUnit::CudaCore, Precision::FP64, a, b, 3.0, 8, nullptr); });
    // SpMV plan: host-side validation before any device allocation
    {
        const std::int32_t rp[3] = {0, 1, 2}, colbad[2] = {0, 7};
        const double vv[2] = {1.0, 2.0};
        SparseMatrixStats s2{2, 2, 2};
        probe("plan_bad_column", [&] {
            SpmvPlan p(ExecutionUnit::CudaCore, Precision::FP64, s2, rp, colbad, vv);
            return KernelCharacterization{};
        });
        const std::int32_t rpdec[3] = {0, 2, 1}, colok[2] = {0, 1};
        probe("plan_decreasing_rows", [&] {
            SpmvPlan p(ExecutionUnit::CudaCore, Precision::FP64, SparseMatrixStats{2, 2, 1}, rpdec, colok, vv);
            return KernelCharacterization{};
        });
    }
    // temporal depth past 8: InvalidRange before any device work
    {
        std::uint64_t d3[3] = {8, 8, 8};
        probe("temporal_depth_9", [&] {
            return stencil_temporal(ExecutionUnit::CudaCore, Precision::FP64, stencil_preset("3d7pt"), d3, nullptr, 18,
                                    9, a, b, nullptr, nullptr);
        });
    }
    // report.hpp through the adapter: the bounds equal the reference's own
    // bounds.cpp objects (value, kind, assumption and warning text)
    try {
        const HardwareSpec& gh = builtin_spec("GH200");
        KernelCharacterization k = stencil_model(stencil_preset("3d27pt"), Precision::FP64, 1);
        const AnalysisReport r = build_analysis(gh, Precision::FP64, k, 9.99, k.intensity());
        const double a = tensor_alpha(gh, Precision::FP64);
        const SpeedupBound want[3] = {kernel_speedup_ceiling(a, 9.99, k.intensity()), tensor_core_ceiling(a),
                                      workload_ceiling(k.intensity(), 9.99)};
        bool same = r.bounds.size() == 3;
        for (int i = 0; same && i < 3; ++i)
            same = r.bounds[i].value == want[i].value && r.bounds[i].kind == want[i].kind &&
                   r.bounds[i].assumptions == want[i].assumptions && r.bounds[i].warnings == want[i].warnings;
        std::printf("report_bounds %s\n", same ? "same" : "differ");
        std::printf("report_alpha %s\n", r.alpha == a ? "same" : "differ");
        std::printf("report_min_depth %llu\n", (unsigned long long)r.min_depth.value_or(0));
        std::printf("report_verdict %s\n", r.verdict.c_str());
        std::printf("report_notes %zu\n", r.notes.size());
        const std::string j = render_json(r);
        std::printf("render_json %s\n", j.find("\"verdict\"") != std::string::npos ? "has_verdict" : "no_verdict");
        const KernelCharacterization c = scale_model(4, Precision::FP64);
        const AnalysisReport w = build_analysis(builtin_spec("A100-80GB"), Precision::FP64,
                                                gemv_model(100000, 100000, Precision::FP64));
        std::printf("report_gemv_workload %.6f\n", w.bounds.back().value);
        const std::string txt = render_text(w);
        std::printf("render_text_lines %zu\n", (size_t)std::count(txt.begin(), txt.end(), '\n'));
        (void)c;
    } catch (const Error& e) {
        std::printf("report_bounds kind:%d:%s\n", static_cast<int>(e.kind()), e.what());
    }
    try {
        build_analysis(builtin_spec("A100-80GB"), Precision::FP64, scale_model(4, Precision::FP64), 0.0);
        std::printf("report_zero_balance ok\n");
    } catch (const Error& e) {
        std::printf("report_zero_balance kind:%d\n", static_cast<int>(e.kind()));
    }
    return 0;
}
