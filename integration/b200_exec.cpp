// b200_exec.cpp -- the rooflens-side adapter over librooflens_b200.so
// (INTEGRATION.md §1): C statuses back into rooflens::Error, rl_kchar back
// into KernelCharacterization.  Needs no CUDA headers, nlohmann or torch:
// streams travel as void*.  The reference's ExecutionUnit / Precision
// (hardware.hpp:19-21) have rl_unit / rl_precision's ordinals.
#include "b200_exec.hpp"

#include <stdexcept>
#include <string>

#include "rooflens/error.hpp"
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

}  // namespace rooflens
