// integration_main.cpp -- drives integration/b200_exec.cpp compiled against
// the reference's headers (tests/test_integration.py).  Prints one line per
// probe: "<probe> <outcome>" where outcome is ok:<W>/<Q>, the rooflens
// ErrorKind ordinal as kind:<k>, or runtime:<text> for a CUDA / NCCL status.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <string>

#include "b200_exec.hpp"
#include "rooflens/error.hpp"

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
    return 0;
}
