// b200_exec.hpp -- what a rooflens maintainer adds to the reference tree
// (proj/include/rooflens/b200_exec.hpp) to execute the kernels its models
// describe on a B200: the reference's own types in, the reference's own
// types and exceptions out, librooflens_b200.so underneath.
// Compiled against /root/reference/proj/include by tests/test_integration.py.
#pragma once

#include <cstdint>
#include <string>

#include "rooflens/hardware.hpp"
#include "rooflens/kernels.hpp"

namespace rooflens {

// a = q*b on the GPU; returns scale_model(n, precision) (kernels.cpp:74-86)
KernelCharacterization scale(ExecutionUnit unit, Precision precision, double* a, const double* b, double q,
                             std::uint64_t n, void* stream);
// y = A*x (CSR, int32 indices); returns spmv_csr_model(stats, 4, precision) (kernels.cpp:123-135)
KernelCharacterization spmv_csr(ExecutionUnit unit, Precision precision, const SparseMatrixStats& stats,
                                const std::int32_t* row_ptr, const std::int32_t* col, const double* val,
                                const double* x, double* y, void* stream);
// `steps` Jacobi sweeps; returns stencil_model(shape, precision, 1) x points x steps (kernels.cpp:137-155)
KernelCharacterization stencil(ExecutionUnit unit, Precision precision, const StencilShape& shape,
                               const std::uint64_t dims[3], const double* weights, std::uint64_t steps, double* u,
                               double* v, void* stream);

// `steps` timesteps as steps/t fused sweeps of depth t (plus steps%t single
// sweeps); returns stencil_model(shape, precision, t) accounting
// (kernels.cpp:137-155).  *result_in_v: where the final field is.
KernelCharacterization stencil_temporal(ExecutionUnit unit, Precision precision, const StencilShape& shape,
                                        const std::uint64_t dims[3], const double* weights, std::uint64_t steps,
                                        std::uint64_t t, double* u, double* v, void* stream, bool* result_in_v);

// A matrix uploaded once (host CSR in), re-laid for the B200 SpMV kernels;
// each execute returns spmv_csr_model(stats, 4, precision).
class SpmvPlan {
public:
    SpmvPlan(ExecutionUnit unit, Precision precision, const SparseMatrixStats& stats, const std::int32_t* row_ptr,
             const std::int32_t* col, const double* val);
    ~SpmvPlan();
    SpmvPlan(const SpmvPlan&) = delete;
    SpmvPlan& operator=(const SpmvPlan&) = delete;
    KernelCharacterization execute_host(const double* x, double* y);                  // host x, y
    KernelCharacterization execute(const double* x_dev, double* y_dev, void* stream);  // device x, y
    std::string layout() const;  // "csr" or "colsort"

private:
    void* h_ = nullptr;
};

// Multi-GPU: one communicator per process (NCCL underneath).
class B200Comm {
public:
    // rank 0 calls unique_id() and ships the 128 bytes to every rank
    static void unique_id(std::uint8_t id[128]);
    B200Comm(int world, int rank, const std::uint8_t id[128]);
    ~B200Comm();
    B200Comm(const B200Comm&) = delete;
    B200Comm& operator=(const B200Comm&) = delete;
    void* handle() const { return h_; }

private:
    void* h_ = nullptr;
};
// STREAM Scale on this rank's chunk of n_global; returns scale_model(n_global)
KernelCharacterization dist_scale(const B200Comm& comm, ExecutionUnit unit, Precision precision, double* a,
                                  const double* b, double q, std::uint64_t n_global, void* stream);

// Row-partitioned SpMV of an n x n band matrix (half-bandwidth hb), one part
// per rank: device CSR of the rank's rows (global columns), x window and y
// (rl_dist_spmv_part).  execute returns spmv_csr_model of the global matrix.
class DistSpmv {
public:
    DistSpmv(const B200Comm& comm, ExecutionUnit unit, Precision precision, std::uint64_t n, std::uint64_t hb,
             const std::int32_t* row_ptr, const std::int32_t* col, const double* val, double* x, double* y);
    ~DistSpmv();
    DistSpmv(const DistSpmv&) = delete;
    DistSpmv& operator=(const DistSpmv&) = delete;
    KernelCharacterization execute(void* stream);

private:
    void* h_ = nullptr;
};

// Slab-decomposed stencil, one slab per rank (rl_dist_stencil_part buffers).
class DistStencil {
public:
    DistStencil(const B200Comm& comm, ExecutionUnit unit, Precision precision, const StencilShape& shape,
                const std::uint64_t dims[3], const double* weights, double* u, double* v);
    ~DistStencil();
    DistStencil(const DistStencil&) = delete;
    DistStencil& operator=(const DistStencil&) = delete;
    KernelCharacterization run(std::uint64_t steps, void* stream, bool* result_in_v);

private:
    void* h_ = nullptr;
    std::string name_;
};

}  // namespace rooflens
