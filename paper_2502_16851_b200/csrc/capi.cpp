// capi.cpp -- the executing C++ entry points (rooflens_b200.hpp) and the
// extern "C" boundary (rooflens_b200.h).
//
// Each executing call validates its arguments the way the reference model it
// sits behind does (same ErrorKind, same message format), launches the sm_100a
// kernel(s) on the caller's stream, and returns the reference model's W/Q for
// the call.  There is no CPU path: a missing/unusable device surfaces as a
// CUDA error code (RL_ERR_CUDA_BASE + cudaError_t).
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <vector>
#include <mutex>
#include <string>

#include <cuda_runtime.h>

#include "../../include/rooflens_b200.h"
#include "../../include/rooflens_b200.hpp"
#include "boundary.h"
#include "kernels.h"

namespace rlb {
Tuning& tuning() {
    static Tuning t;
    return t;
}
std::atomic<uint64_t> g_launches{0};
void note_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
}  // namespace rlb

namespace rooflens::b200 {
std::string& last_error_slot() {
    static thread_local std::string slot;
    return slot;
}
namespace {

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw CudaError(static_cast<int>(e), std::string("CudaError: ") + what + ": " +
                                                 cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")");
}

void require_fp64(Precision p) {
    if (p != Precision::FP64)
        throw Error(ErrorKind::ValidationError,
                    std::string("precision ") + (p == Precision::FP32 ? "FP32" : "FP16") +
                        " is not supported by the B200 kernels (FP64 only)");
}

void require_ptr(const void* p, const char* what) {
    if (!p) throw Error(ErrorKind::ValidationError, std::string(what) + " must not be null");
}

int preset_id(const std::string& n) {
    if (n == "2d5pt") return rlb::kP2d5;
    if (n == "2d9pt") return rlb::kP2d9;
    if (n == "2d13pt") return rlb::kP2d13;
    if (n == "2d49pt") return rlb::kP2d49;
    if (n == "3d7pt") return rlb::kP3d7;
    return rlb::kP3d27;
}

rlb::StencilDesc make_desc(const StencilShape& shape, const std::uint64_t dims[3],
                           const double* weights) {
    rlb::StencilDesc d{};
    d.preset = preset_id(shape.name);
    d.dim = shape.dimensionality;
    d.radius = shape.radius;
    d.npts = static_cast<int>(shape.point_count);
    d.nx = dims[0];
    d.ny = dims[1];
    d.nz = shape.dimensionality == 3 ? dims[2] : 1;
    const std::uint64_t need = 2ull * shape.radius + 1;
    if (d.nx < need || d.ny < need || (d.dim == 3 && d.nz < need))
        throw Error(ErrorKind::InvalidCount, "stencil: every grid extent must be >= " +
                                                 std::to_string(need) + " for " + shape.name);
    if (weights) {
        std::memcpy(d.w, weights, sizeof(double) * shape.point_count);
    } else {
        const auto w = stencil_default_weights(shape.name);
        std::memcpy(d.w, w.data(), sizeof(double) * w.size());
    }
    return d;
}

std::uint64_t interior_points(const rlb::StencilDesc& d) {
    const std::uint64_t r2 = 2ull * d.radius;
    std::uint64_t p = (d.nx - r2) * (d.ny - r2);
    if (d.dim == 3) p *= (d.nz - r2);
    return p;
}

void sweep(ExecutionUnit unit, const rlb::StencilDesc& d, std::uint64_t o0, std::uint64_t o1,
           const double* u, double* v, cudaStream_t s) {
    const std::uint64_t outer = d.dim == 3 ? d.nz : d.ny;
    const std::uint64_t lo = std::max<std::uint64_t>(o0, d.radius);
    const std::uint64_t hi = std::min<std::uint64_t>(o1, outer - d.radius);
    if (lo >= hi) return;
    if (unit == ExecutionUnit::TensorCore && d.preset != rlb::kP2d5 && d.preset != rlb::kP3d7 &&
        d.preset != rlb::kP3d27) {
        if (!rlb::stencil_r_eligible(d, u, v))
            throw Error(ErrorKind::ValidationError,
                        "the tensor-core 2d9pt/2d13pt/2d49pt kernels need an even nx and 16-byte aligned "
                        "u and v");
        cuda_check(rlb::launch_stencil_r(1, d, lo, hi, u, v, s), "stencil (tensor core)");
        return;
    }
    if (unit == ExecutionUnit::TensorCore)
        cuda_check(rlb::launch_stencil_tc(d, lo, hi, u, v, s), "stencil (tensor core)");
    else
        cuda_check(rlb::launch_stencil_cc(d, lo, hi, u, v, s), "stencil (cuda core)");
}

}  // namespace

KernelCharacterization scale(ExecutionUnit unit, Precision p, double* a, const double* b, double q,
                             std::uint64_t n, Stream stream) {
    KernelCharacterization k = scale_model(n, p);
    require_fp64(p);
    require_ptr(a, "a");
    require_ptr(b, "b");
    cuda_check(rlb::launch_scale(unit == ExecutionUnit::TensorCore, a, b, q, n,
                                 static_cast<cudaStream_t>(stream)),
               "scale");
    return k;
}

KernelCharacterization gemv(ExecutionUnit unit, Precision p, std::uint64_t m, std::uint64_t n,
                            const double* A, const double* x, double* y, Stream stream) {
    KernelCharacterization k = gemv_model(m, n, p);
    require_fp64(p);
    require_ptr(A, "A");
    require_ptr(x, "x");
    require_ptr(y, "y");
    cuda_check(rlb::launch_gemv(unit == ExecutionUnit::TensorCore, m, n, A, x, y,
                                static_cast<cudaStream_t>(stream)),
               "gemv");
    return k;
}

void spmv_csr_rows(ExecutionUnit unit, Precision p, std::uint64_t r0, std::uint64_t r1,
                   const std::int32_t* rp, const std::int32_t* col, const double* val,
                   const double* x, std::int64_t col_base, double* y, Stream stream, int long_rows) {
    require_fp64(p);
    if (r1 < r0) throw Error(ErrorKind::InvalidRange, "row_end < row_begin");
    if (r1 == r0) return;
    require_ptr(rp, "row_ptr");
    require_ptr(col, "col");
    require_ptr(val, "val");
    require_ptr(x, "x");
    require_ptr(y, "y");
    // element alignment (the kernels pick vector loads only for 32-byte val /
    // 16-byte col bases, spmv.cu; an element-misaligned view is rejected)
    if ((reinterpret_cast<std::uintptr_t>(val) & 7) || (reinterpret_cast<std::uintptr_t>(x) & 7) ||
        (reinterpret_cast<std::uintptr_t>(y) & 7) || (reinterpret_cast<std::uintptr_t>(col) & 3) ||
        (reinterpret_cast<std::uintptr_t>(rp) & 3))
        throw Error(ErrorKind::ValidationError, "spmv_csr: val/x/y must be 8-byte and row_ptr/col 4-byte aligned");
    cuda_check(rlb::launch_spmv(unit == ExecutionUnit::TensorCore, r0, r1, rp, col, val, x, col_base,
                                y, long_rows, static_cast<cudaStream_t>(stream)),
               "spmv_csr");
}

KernelCharacterization spmv_csr(ExecutionUnit unit, Precision p, const SparseMatrixStats& s,
                                const std::int32_t* rp, const std::int32_t* col, const double* val,
                                const double* x, double* y, Stream stream) {
    KernelCharacterization k = spmv_csr_model(s, kDefaultIndexBytes, p);
    require_fp64(p);
    if (s.nnz > 0x7fffffffull || s.rows > 0x7fffffffull || s.cols > 0x7fffffffull)
        throw Error(ErrorKind::InvalidRange, "int32 CSR indices cannot address this matrix");
    require_ptr(col, "col");
    require_ptr(val, "val");
    require_ptr(x, "x");
    spmv_csr_rows(unit, p, 0, s.rows, rp, col, val, x, 0, y, stream);
    return k;
}

void stencil_sweep(ExecutionUnit unit, Precision p, const StencilShape& shape,
                   const std::uint64_t dims[3], const double* weights, std::uint64_t o0,
                   std::uint64_t o1, const double* u, double* v, Stream stream) {
    require_fp64(p);
    require_ptr(u, "u");
    require_ptr(v, "v");
    if (u == v) throw Error(ErrorKind::ValidationError, "u and v must be distinct buffers");
    const rlb::StencilDesc d = make_desc(shape, dims, weights);
    sweep(unit, d, o0, o1, u, v, static_cast<cudaStream_t>(stream));
}

KernelCharacterization stencil(ExecutionUnit unit, Precision p, const StencilShape& shape,
                               const std::uint64_t dims[3], const double* weights,
                               std::uint64_t steps, double* u, double* v, Stream stream) {
    KernelCharacterization per_point = stencil_model(shape, p, 1);
    require_fp64(p);
    if (!steps) throw Error(ErrorKind::InvalidCount, "stencil: steps must be >= 1");
    require_ptr(u, "u");
    require_ptr(v, "v");
    if (u == v) throw Error(ErrorKind::ValidationError, "u and v must be distinct buffers");
    const rlb::StencilDesc d = make_desc(shape, dims, weights);
    const unsigned __int128 pts = (unsigned __int128)interior_points(d) * steps;
    const unsigned __int128 w = pts * per_point.work_flops, q = pts * per_point.traffic_bytes;
    if ((w >> 64) || (q >> 64)) throw Error(ErrorKind::InvalidRange, "stencil accounting overflows 64-bit count");
    const std::uint64_t outer = d.dim == 3 ? d.nz : d.ny;
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    for (std::uint64_t t = 0; t < steps; ++t) {
        const double* src = (t & 1) ? v : u;
        double* dst = (t & 1) ? u : v;
        sweep(unit, d, 0, outer, src, dst, s);
    }
    return {shape.name, static_cast<std::uint64_t>(w), static_cast<std::uint64_t>(q)};
}

KernelCharacterization stencil_temporal(ExecutionUnit unit, Precision p, const StencilShape& shape,
                                        const std::uint64_t dims[3], const double* weights,
                                        std::uint64_t steps, std::uint64_t t, double* u, double* v,
                                        Stream stream, int* result_in_v) {
    const KernelCharacterization kt = stencil_model(shape, p, t);  // validates t >= 1
    const KernelCharacterization k1 = stencil_model(shape, p, 1);
    require_fp64(p);
    if (!steps) throw Error(ErrorKind::InvalidCount, "stencil: steps must be >= 1");
    require_ptr(u, "u");
    require_ptr(v, "v");
    if (u == v) throw Error(ErrorKind::ValidationError, "u and v must be distinct buffers");
    if (t > 8) throw Error(ErrorKind::InvalidRange, "temporal depth > 8 is not implemented");
    const rlb::StencilDesc d = make_desc(shape, dims, weights);
    const bool use_tb = t >= 2 && rlb::stencil_tb_supported(d, (int)t, u, v);
    // 3d7pt: the register-blocked TMA kernel; the z-column kernel covers the
    // shapes it refuses (odd nx, unaligned rows)
    const bool use_tb3r = t >= 2 && rlb::stencil_tb3r_supported(d, (int)t, u, v);
    const bool use_tb27r = t >= 2 && rlb::tuning().stencil_tb27r && rlb::stencil_tb27r_supported(d, (int)t, u, v);
    const bool use_tb3 = t >= 2 && (use_tb3r || rlb::stencil_tb3_supported(d, (int)t));
    const bool use_tbtc = t >= 2 && unit == ExecutionUnit::TensorCore && rlb::stencil_tbtc_supported(d, (int)t, u, v);
    const bool ok2d = d.preset == rlb::kP2d5 && use_tb;
    if (t >= 2 && !(unit == ExecutionUnit::CudaCore ? (ok2d || use_tb3) : use_tbtc))
        throw Error(ErrorKind::ValidationError,
                    "temporal depth >= 2 is implemented on the CUDA core for 2d5pt (t <= 8; even depths need "
                    "an even nx and 16-byte aligned rows), 3d7pt and 3d27pt (t <= 4), and on the tensor core "
                    "for 2d5pt (t <= 4, even nx, 16-byte aligned u and v)");
    const std::uint64_t fused = steps / t, rem = steps % t;
    const unsigned __int128 pts = interior_points(d);
    const unsigned __int128 w = pts * ((unsigned __int128)fused * kt.work_flops + (unsigned __int128)rem * k1.work_flops);
    const unsigned __int128 q = pts * ((unsigned __int128)fused * kt.traffic_bytes + (unsigned __int128)rem * k1.traffic_bytes);
    if ((w >> 64) || (q >> 64)) throw Error(ErrorKind::InvalidRange, "stencil accounting overflows 64-bit count");
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    const std::uint64_t outer = d.dim == 3 ? d.nz : d.ny;
    std::uint64_t sweeps = 0;
    for (std::uint64_t i = 0; i < fused + rem; ++i, ++sweeps) {
        const double* src = (sweeps & 1) ? v : u;
        double* dst = (sweeps & 1) ? u : v;
        if (i < fused && use_tbtc) {
            cuda_check(rlb::launch_stencil_tbtc(d, (int)t, src, dst, s), "stencil (tensor-core temporal blocking)");
        } else if (i < fused && use_tb27r) {
            cuda_check(rlb::launch_stencil_tb27r(d, (int)t, 1, outer - 1, src, dst, s), "stencil (3D temporal blocking)");
        } else if (i < fused && use_tb3r) {
            cuda_check(rlb::launch_stencil_tb3r(d, (int)t, 1, outer - 1, src, dst, s), "stencil (3D temporal blocking)");
        } else if (i < fused && use_tb3) {
            cuda_check(rlb::launch_stencil_tb3(d, (int)t, 1, outer - 1, src, dst, s), "stencil (3D temporal blocking)");
        } else if (i < fused && use_tb) {
            cuda_check(rlb::launch_stencil_tb(d, (int)t, 1, outer - 1, src, dst, s), "stencil (temporal blocking)");
        } else {
            sweep(unit, d, 0, outer, src, dst, s);
        }
    }
    if (result_in_v) *result_in_v = (int)(sweeps & 1);
    return {shape.name, static_cast<std::uint64_t>(w), static_cast<std::uint64_t>(q)};
}

}  // namespace rooflens::b200

// ===========================================================================
// Host-buffer end-to-end paths: cached device workspace + two streams.
// ===========================================================================
namespace {
using namespace rooflens::b200;

struct Workspace {
    std::mutex mu;
    void* buf[6] = {};
    size_t cap[6] = {};
    cudaStream_t h2d = nullptr, comp = nullptr;
    cudaEvent_t ev[64] = {};

    void* get(int i, size_t bytes) {
        if (cap[i] < bytes) {
            if (buf[i]) cudaFree(buf[i]);
            buf[i] = nullptr;
            cap[i] = 0;
            if (cudaMalloc(&buf[i], bytes) != cudaSuccess) {
                cudaGetLastError();
                throw CudaError(cudaErrorMemoryAllocation, "CudaError: workspace allocation failed");
            }
            cap[i] = bytes;
        }
        return buf[i];
    }
    void streams() {
        if (!h2d) {
            cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking);
            cudaStreamCreateWithFlags(&comp, cudaStreamNonBlocking);
            for (auto& e : ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        }
    }
    void release() {
        for (int i = 0; i < 6; ++i) {
            if (buf[i]) cudaFree(buf[i]);
            buf[i] = nullptr;
            cap[i] = 0;
        }
        if (h2d) {
            cudaStreamDestroy(h2d);
            cudaStreamDestroy(comp);
            for (auto& e : ev) cudaEventDestroy(e);
            h2d = comp = nullptr;
        }
    }
};
Workspace& ws() {
    static Workspace w;
    return w;
}

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw CudaError(static_cast<int>(e), std::string("CudaError: ") + what + ": " + cudaGetErrorName(e));
}

constexpr uint64_t kChunk = 4ull << 20;  // doubles per pipelined chunk (32 MiB)

KernelCharacterization scale_host(ExecutionUnit unit, Precision p, double* a, const double* b, double q,
                                  uint64_t n) {
    KernelCharacterization k = scale_model(n, p);
    require_fp64(p);
    require_ptr(a, "a");
    require_ptr(b, "b");
    Workspace& w = ws();
    std::lock_guard<std::mutex> lock(w.mu);
    w.streams();
    double* db = static_cast<double*>(w.get(0, n * 8));
    double* da = static_cast<double*>(w.get(1, n * 8));
    const uint64_t nch = (n + kChunk - 1) / kChunk;
    for (uint64_t c = 0; c < nch; ++c) {
        const uint64_t o = c * kChunk, len = std::min(kChunk, n - o);
        cudaEvent_t e = w.ev[c % 64];
        ck(cudaMemcpyAsync(db + o, b + o, len * 8, cudaMemcpyHostToDevice, w.h2d), "H2D");
        ck(cudaEventRecord(e, w.h2d), "event");
        ck(cudaStreamWaitEvent(w.comp, e, 0), "wait");
        scale(unit, p, da + o, db + o, q, len, w.comp);
        ck(cudaMemcpyAsync(a + o, da + o, len * 8, cudaMemcpyDeviceToHost, w.comp), "D2H");
    }
    ck(cudaStreamSynchronize(w.comp), "sync");
    return k;
}

KernelCharacterization spmv_host(ExecutionUnit unit, Precision p, uint64_t m, uint64_t n, uint64_t nnz,
                                 const int32_t* rp, const int32_t* col, const double* val,
                                 const double* x, double* y) {
    KernelCharacterization k = spmv_csr_model({m, n, nnz}, kDefaultIndexBytes, p);
    require_fp64(p);
    require_ptr(rp, "row_ptr");
    require_ptr(col, "col");
    require_ptr(val, "val");
    require_ptr(x, "x");
    require_ptr(y, "y");
    if (nnz > 0x7fffffffull || m > 0x7fffffffull)
        throw Error(ErrorKind::InvalidRange, "int32 CSR indices cannot address this matrix");
    Workspace& w = ws();
    std::lock_guard<std::mutex> lock(w.mu);
    w.streams();
    int32_t* drp = static_cast<int32_t*>(w.get(0, (m + 1) * 4));
    int32_t* dcol = static_cast<int32_t*>(w.get(1, nnz * 4));
    double* dval = static_cast<double*>(w.get(2, nnz * 8));
    double* dx = static_cast<double*>(w.get(3, n * 8));
    double* dy = static_cast<double*>(w.get(4, m * 8));
    ck(cudaMemcpyAsync(dx, x, n * 8, cudaMemcpyHostToDevice, w.h2d), "H2D x");
    ck(cudaMemcpyAsync(drp, rp, (m + 1) * 4, cudaMemcpyHostToDevice, w.h2d), "H2D row_ptr");
    // Row chunks of ~kChunk nonzeros: copy col/val of the chunk, run its rows,
    // return its y while the next chunk is in flight.
    const uint64_t rows_per_chunk = std::max<uint64_t>(1, (uint64_t)((double)kChunk * m / (double)nnz));
    int c = 0;
    for (uint64_t r0 = 0; r0 < m; r0 += rows_per_chunk, ++c) {
        const uint64_t r1 = std::min(m, r0 + rows_per_chunk);
        const uint64_t k0 = (uint64_t)rp[r0], k1 = (uint64_t)rp[r1];
        if (k1 > k0) {
            ck(cudaMemcpyAsync(dcol + k0, col + k0, (k1 - k0) * 4, cudaMemcpyHostToDevice, w.h2d), "H2D col");
            ck(cudaMemcpyAsync(dval + k0, val + k0, (k1 - k0) * 8, cudaMemcpyHostToDevice, w.h2d), "H2D val");
        }
        cudaEvent_t e = w.ev[c % 64];
        ck(cudaEventRecord(e, w.h2d), "event");
        ck(cudaStreamWaitEvent(w.comp, e, 0), "wait");
        spmv_csr_rows(unit, p, r0, r1, drp, dcol, dval, dx, 0, dy, w.comp);
        ck(cudaMemcpyAsync(y + r0, dy + r0, (r1 - r0) * 8, cudaMemcpyDeviceToHost, w.comp), "D2H y");
    }
    ck(cudaStreamSynchronize(w.comp), "sync");
    return k;
}

KernelCharacterization stencil_host(ExecutionUnit unit, Precision p, const char* preset,
                                    const uint64_t* dims, const double* weights, uint64_t steps,
                                    double* u, double* v) {
    require_ptr(preset, "preset");
    require_ptr(dims, "dims");
    const StencilShape& shape = stencil_preset(preset);
    require_ptr(u, "u");
    require_ptr(v, "v");
    const uint64_t n = dims[0] * dims[1] * (shape.dimensionality == 3 ? dims[2] : 1);
    Workspace& w = ws();
    std::lock_guard<std::mutex> lock(w.mu);
    w.streams();
    double* du = static_cast<double*>(w.get(0, n * 8));
    double* dv = static_cast<double*>(w.get(1, n * 8));
    ck(cudaMemcpyAsync(du, u, n * 8, cudaMemcpyHostToDevice, w.comp), "H2D u");
    // v's Dirichlet ring must equal u's (contract): replicate on the device.
    ck(cudaMemcpyAsync(dv, du, n * 8, cudaMemcpyDeviceToDevice, w.comp), "D2D v");
    KernelCharacterization k = stencil(unit, p, shape, dims, weights, steps, du, dv, w.comp);
    double* res_host = (steps & 1) ? v : u;
    const double* res_dev = (steps & 1) ? dv : du;
    ck(cudaMemcpyAsync(res_host, res_dev, n * 8, cudaMemcpyDeviceToHost, w.comp), "D2H result");
    ck(cudaStreamSynchronize(w.comp), "sync");
    return k;
}

// ---------------------------------------------------------------------------
// SpMV plan
// ---------------------------------------------------------------------------
}  // namespace

struct rl_spmv_plan_s {
    ExecutionUnit unit;
    uint64_t m = 0, n = 0, nnz = 0;
    int32_t *rp = nullptr, *col = nullptr;
    double *val = nullptr, *x = nullptr, *y = nullptr;
    // column-sorted row blocks (K17, spmv_colsort.cu)
    bool colsort = false;
    int krb = 0, krows = 0, kvec = 1;
    rlb::SpmvKBlock* kblk = nullptr;
    double* kval = nullptr;
    unsigned* kmeta = nullptr;
    std::vector<uint32_t> kblk_r0;
    rlb::ColsortRun krun{};  // fixed-point mode state (null grid: FP64 atomics)
    rlb::ColsortRun colsort_run() const {
        rlb::ColsortRun r = krun;
        r.rp = rp, r.col = col, r.val = val, r.col_base = 0;
        r.fuse = rlb::tuning().spmv_colsort_fuse;
        return r;
    }
    uint64_t layout_bytes = 0;
    std::vector<uint64_t> chunk_row;   // chunk c = rows [chunk_row[c], chunk_row[c+1])
    std::vector<uint64_t> chunk_xend;  // x prefix [0, chunk_xend[c]) chunk c reads
    std::vector<uint64_t> xpiece;      // x upload pieces: [xpiece[i], xpiece[i+1])
    std::vector<char> ycut;            // chunk c ends a y copy group
    cudaStream_t s_in = nullptr, s_out = nullptr;
    // compute streams: one for CSR; several for the column-sorted layout, whose
    // per-chunk kernels (a few blocks each) run concurrently as x arrives
    std::vector<cudaStream_t> s_cmp;
    int long_rows = 0;  // the CSR has rows the per-row kernels divert (spmv.cu)
    std::vector<cudaEvent_t> ev_x, ev_y;
    std::vector<cudaEvent_t> ev_join;  // one per compute stream + s_out
    cudaEvent_t ev_fork = nullptr;  // s_cmp / s_out join s_in at the start of every call (and capture)
    // execute_host_async: calls rotate over kSlots device x / y buffer slots
    // (slot 0 = x / y above, the others allocated on first use); a call reuses
    // a slot only after the slot's previous call has finished computing from
    // its x (ev_cdone) and downloading its y (ev_ydone)
    static constexpr int kSlots = 3;
    double *xs[kSlots] = {}, *ys[kSlots] = {};  // slot 0 = x / y above
    uint64_t async_calls = 0;
    cudaEvent_t ev_cdone[kSlots] = {}, ev_ydone[kSlots] = {}, ev_xall[kSlots] = {};
    // execute_host as a CUDA graph, captured for the last (x, y) host pair
    cudaGraphExec_t gexec = nullptr;
    const double* gx = nullptr;
    double* gy = nullptr;
    uint64_t graph_launches = 0;
    KernelCharacterization kc;
    ~rl_spmv_plan_s() {
        if (rp) cudaFree(rp);
        if (col) cudaFree(col);
        if (val) cudaFree(val);
        if (x) cudaFree(x);
        if (y) cudaFree(y);
        for (int i = 1; i < kSlots; ++i) {
            if (xs[i]) cudaFree(xs[i]);
            if (ys[i]) cudaFree(ys[i]);
        }
        for (int i = 0; i < kSlots; ++i)
            for (auto e : {ev_cdone[i], ev_ydone[i], ev_xall[i]})
                if (e) cudaEventDestroy(e);
        for (void* p : {(void*)kblk, (void*)kval, (void*)kmeta, (void*)krun.grid, (void*)krun.list, (void*)krun.count})
            if (p) cudaFree(p);
        if (gexec) cudaGraphExecDestroy(gexec);
        for (auto e : ev_x) cudaEventDestroy(e);
        for (auto e : ev_y) cudaEventDestroy(e);
        for (auto e : ev_join)
            if (e) cudaEventDestroy(e);
        if (ev_fork) cudaEventDestroy(ev_fork);
        if (s_in) cudaStreamDestroy(s_in);
        for (auto st : s_cmp) cudaStreamDestroy(st);
        if (s_out) cudaStreamDestroy(s_out);
    }
};

namespace {

// Row blocks of a plan's K17 layout: spmv_plan_colsort_blocks blocks over
// all rows (0: the builder's default, 4 x 148); spmv_plan_edge_blocks > 0
// cuts the first and last of the execute_host pipeline's chunks into that
// many blocks each, so those chunks run on every SM (the pipeline's head
// and tail wait on them).
std::vector<rlb::ColsortSegment> plan_segments(uint64_t m) {
    const auto& t = rlb::tuning();
    const uint64_t nb = t.spmv_plan_colsort_blocks > 0 ? (uint64_t)t.spmv_plan_colsort_blocks : 4 * (uint64_t)rlb::kNumSMsHost;
    const uint64_t eb = (uint64_t)std::max(0, t.spmv_plan_edge_blocks);
    const uint64_t nch = (uint64_t)std::max(1, t.spmv_plan_colsort_chunks);
    if (eb == 0 || nch < 3) return {{m, nb}};
    // rows of an edge chunk: the chunk weights of plan_create (taper k: edge
    // chunks weigh 1, the others k + 1)
    const uint64_t tk = (uint64_t)std::max(0, t.spmv_plan_taper);
    const uint64_t wsum = tk ? (tk + 1) * (nch - 2) + 2 : nch;
    const uint64_t e = m / wsum;
    const uint64_t mid = nb - std::min(nb - 1, 2 * nb / wsum);
    return {{e, eb}, {m - e, std::max<uint64_t>(1, mid)}, {m, eb}};
}

rl_spmv_plan_s* plan_create(ExecutionUnit unit, Precision p, uint64_t m, uint64_t n, uint64_t nnz,
                            const int32_t* rp, const int32_t* col, const double* val) {
    KernelCharacterization k = spmv_csr_model({m, n, nnz}, kDefaultIndexBytes, p);
    require_fp64(p);
    require_ptr(rp, "row_ptr");
    require_ptr(col, "col");
    require_ptr(val, "val");
    if (nnz > 0x7fffffffull || m > 0x7fffffffull || n > 0x7fffffffull)
        throw Error(ErrorKind::InvalidRange, "int32 CSR indices cannot address this matrix");
    if ((uint64_t)rp[m] != nnz) throw Error(ErrorKind::ValidationError, "row_ptr[m] != nnz");
    // host-side validation first: nothing is allocated for a malformed CSR
    if (rp[0] != 0) throw Error(ErrorKind::ValidationError, "row_ptr[0] != 0");
    for (uint64_t i = 0; i < m; ++i)
        if (rp[i + 1] < rp[i]) throw Error(ErrorKind::ValidationError, "row_ptr decreases at row " + std::to_string(i));
    for (uint64_t j = 0; j < nnz; ++j)
        if (col[j] < 0 || (uint64_t)col[j] >= n)
            throw Error(ErrorKind::IndexOutOfRange, "column index " + std::to_string(col[j]) + " outside [0, " +
                                                        std::to_string(n) + ")");
    auto pl = std::make_unique<rl_spmv_plan_s>();
    pl->unit = unit;
    pl->m = m;
    pl->n = n;
    pl->nnz = nnz;
    pl->kc = k;
    ck(cudaMalloc(&pl->x, std::max<uint64_t>(n, 2) * 8), "plan alloc");
    ck(cudaMalloc(&pl->y, m * 8), "plan alloc");
    {
        // the column-sorted row-block layout (K17, spmv_colsort.cu) when the
        // matrix is eligible (rows <= kColsortMaxRowLen nonzeros, block column
        // spans fit); else the caller's CSR with the long-row path
        rlb::SpmvColsortLayout L;
        if (rlb::tuning().spmv_plan_colsort && nnz > 0 &&
            rlb::spmv_colsort_build(m, n, rp, col, val, L, plan_segments(m), rlb::colsort_classes(unit == ExecutionUnit::TensorCore),
                                    unit == ExecutionUnit::TensorCore, rlb::tuning().spmv_colsort_vec)) {
            pl->colsort = true;
            pl->krb = L.rb;
            pl->kvec = L.vec;
            pl->krows = L.rows;
            auto up = [&](auto*& dst, const auto& v) {
                using T = std::remove_reference_t<decltype(*dst)>;
                ck(cudaMalloc(&dst, std::max<size_t>(v.size(), 1) * sizeof(T)), "plan alloc");
                if (!v.empty()) ck(cudaMemcpy(dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "plan upload");
            };
            up(pl->kblk, L.blocks);
            up(pl->kval, L.val);
            up(pl->kmeta, L.meta);
            for (const auto& k : L.blocks) pl->kblk_r0.push_back(k.row0);
            pl->layout_bytes = L.val.size() * 12 + L.blocks.size() * sizeof(rlb::SpmvKBlock);
            if (rlb::colsort_fixed_for(unit == ExecutionUnit::TensorCore)) {
                // fixed-point rows: per-block grid, the flagged-row list and the
                // CSR the FP64 row kernel reads for the rows it hands over
                std::vector<int> g;
                for (const auto& k : L.blocks) g.push_back(rlb::colsort_initial_grid(k));
                up(pl->krun.grid, g);
                ck(cudaMalloc(&pl->krun.list, std::max<uint64_t>(m, 1) * sizeof(int)), "plan alloc");
                ck(cudaMalloc(&pl->krun.count, 2 * sizeof(unsigned)), "plan alloc");
                ck(cudaMemset(pl->krun.count, 0, 2 * sizeof(unsigned)), "plan alloc");
                pl->krun.done = pl->krun.count + 1;
                pl->krun.rows = (unsigned)m;
            }
        }
        if (!pl->colsort || pl->krun.grid) {
            ck(cudaMalloc(&pl->rp, (m + 1) * 4), "plan alloc");
            ck(cudaMemcpy(pl->rp, rp, (m + 1) * 4, cudaMemcpyHostToDevice), "plan upload");
            ck(cudaMalloc(&pl->col, std::max<uint64_t>(nnz, 1) * 4), "plan alloc");
            ck(cudaMalloc(&pl->val, std::max<uint64_t>(nnz, 1) * 8), "plan alloc");
            ck(cudaMemcpy(pl->col, col, nnz * 4, cudaMemcpyHostToDevice), "plan upload");
            ck(cudaMemcpy(pl->val, val, nnz * 8, cudaMemcpyHostToDevice), "plan upload");
            if (!pl->colsort) pl->layout_bytes = (m + 1) * 4 + nnz * 12;  // (a K17 plan keeps the CSR only for re-summed rows)
        }
    }
    const uint64_t unitrows = 1;
    const uint64_t units = m;
    if (!pl->colsort) {
        int64_t maxlen = 0;
        for (uint64_t i = 0; i < m; ++i) maxlen = std::max<int64_t>(maxlen, (int64_t)rp[i + 1] - rp[i]);
        pl->long_rows = (maxlen > rlb::tuning().spmv_long_min && rlb::tuning().spmv_long_rows) ? 1 : 0;
    }
    uint64_t nch = std::min<uint64_t>(
        (uint64_t)(pl->colsort ? rlb::tuning().spmv_plan_colsort_chunks : rlb::tuning().spmv_plan_chunks), units);
    // Chunk c covers weight w_c of the rows: with spmv_plan_taper = k > 0 the
    // first and last chunks weigh 1 and the others k + 1, so the pipeline's
    // head (the first x prefix) and tail (the last compute + y copy) are short
    // while the middle copies stay large; k = 0: equal chunks.
    const uint64_t tk = (uint64_t)std::max(0, rlb::tuning().spmv_plan_taper);
    const bool taper = tk > 0 && nch >= 3;
    const uint64_t wmid = taper ? tk + 1 : 1;
    const uint64_t wsum = taper ? wmid * (nch - 2) + 2 : nch;
    uint64_t acc = 0;
    for (uint64_t c = 0; c <= nch; ++c) {
        pl->chunk_row.push_back(std::min<uint64_t>(m, units * acc / wsum * unitrows));
        if (c < nch) acc += (taper && (c == 0 || c == nch - 1)) ? 1 : wmid;
    }
    pl->chunk_row.back() = m;
    if (pl->colsort) {  // chunk boundaries on block starts
        for (size_t c = 1; c + 1 < pl->chunk_row.size(); ++c) {
            auto it = std::lower_bound(pl->kblk_r0.begin(), pl->kblk_r0.end(), (uint32_t)pl->chunk_row[c]);
            pl->chunk_row[c] = it == pl->kblk_r0.end() ? m : *it;
        }
        pl->chunk_row.erase(std::unique(pl->chunk_row.begin(), pl->chunk_row.end()), pl->chunk_row.end());
        nch = pl->chunk_row.size() - 1;
    }
    for (uint64_t c = 0; c < nch; ++c) {
        uint64_t mx = 0;
        for (int64_t j = rp[pl->chunk_row[c]]; j < rp[pl->chunk_row[c + 1]]; ++j)
            mx = std::max<uint64_t>(mx, (uint64_t)col[j] + 1);
        pl->chunk_xend.push_back(mx);
    }
    // x upload pieces end exactly where a chunk's column prefix ends, so
    // chunk c waits for no byte of x it does not read
    pl->xpiece.push_back(0);
    uint64_t run = 0;
    for (uint64_t c = 0; c < nch; ++c) {
        run = std::max(run, pl->chunk_xend[c]);
        if (run > pl->xpiece.back()) pl->xpiece.push_back(run);
    }
    if (pl->xpiece.back() < n) pl->xpiece.push_back(n);
    // Fewer, larger copies (spmv_plan_xpieces / spmv_plan_ygroups): with both
    // PCIe directions busy every extra copy pair costs ~8-17 us
    // (tools/micro/pcie_multi.cu: 64 MiB moves in 0.675 ms as 1+1 copies,
    // 0.925 ms as 16+16).  The first x piece stays the first chunk's prefix so
    // compute and the y stream start early; the later boundaries are thinned
    // to at most `xpieces` pieces.
    if (const int xp = rlb::tuning().spmv_plan_xpieces; xp >= 2 && pl->xpiece.size() - 1 > (size_t)xp) {
        std::vector<uint64_t> b(pl->xpiece.begin() + 1, pl->xpiece.end());  // piece ends, last == n
        std::vector<uint64_t> keep{0, b[0]};
        const size_t rest = b.size() - 1;  // ends after the first piece
        for (int j = 1; j < xp; ++j) {
            const uint64_t e = b[std::min(rest, (size_t)((uint64_t)rest * j / (xp - 1)))];
            if (e > keep.back()) keep.push_back(e);
        }
        if (keep.back() < n) keep.push_back(n);
        pl->xpiece = keep;
    }
    // y copies: one per group of consecutive chunks (0: one per chunk)
    {
        const int yg = rlb::tuning().spmv_plan_ygroups;
        for (uint64_t c = 0; c < nch; ++c) {
            const bool last = c + 1 == nch;
            const bool cut = yg <= 0 || last || (uint64_t)((c + 1) * (uint64_t)yg / nch) != (uint64_t)(c * (uint64_t)yg / nch);
            pl->ycut.push_back(cut ? 1 : 0);
        }
    }
    const uint64_t npc = pl->xpiece.size() - 1;
    ck(cudaStreamCreateWithFlags(&pl->s_in, cudaStreamNonBlocking), "stream");
    pl->s_cmp.resize(pl->colsort && !pl->krun.grid ? (size_t)std::max(1, rlb::tuning().spmv_plan_streams) : 1);
    for (auto& st : pl->s_cmp) ck(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
    pl->ev_join.resize(pl->s_cmp.size() + 1);
    ck(cudaStreamCreateWithFlags(&pl->s_out, cudaStreamNonBlocking), "stream");
    pl->ev_x.resize(npc);
    pl->ev_y.resize(nch * pl->s_cmp.size());
    for (auto& e : pl->ev_x) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    for (auto& e : pl->ev_y) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    for (auto& e : pl->ev_join) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    ck(cudaEventCreateWithFlags(&pl->ev_fork, cudaEventDisableTiming), "event");
    if (pl->long_rows) {  // reserve the diversion buffers now: execute_host runs under graph capture
        rlb::LongRows lr{};
        ck(rlb::spmv_long_workspace(pl->s_cmp[0], m, lr), "plan long-row workspace");
    }
    return pl.release();
}

// Rows [r0, r1) of y = A x on the plan's layout (r0/r1 block-aligned for the block layouts).
void plan_rows(rl_spmv_plan_s* pl, uint64_t r0, uint64_t r1, const double* x, double* y, cudaStream_t s) {
    if (pl->colsort) {  // r0 / r1 on block starts
        const auto& v = pl->kblk_r0;
        const int b0 = (int)(std::lower_bound(v.begin(), v.end(), (uint32_t)r0) - v.begin());
        const int b1 = r1 >= pl->m ? (int)v.size() : (int)(std::lower_bound(v.begin(), v.end(), (uint32_t)r1) - v.begin());
        ck(rlb::launch_spmv_colsort(pl->unit == ExecutionUnit::TensorCore, pl->kvec, pl->kblk, b0, b1, pl->krb, pl->krows,
                                    pl->kval, pl->kmeta, x, y, pl->colsort_run(), s),
           "spmv (column-sorted plan)");
        return;
    }
    {
        spmv_csr_rows(pl->unit, Precision::FP64, r0, r1, pl->rp, pl->col, pl->val, x, 0, y, s, pl->long_rows);
    }
}

// Enqueue one pipelined call on the plan's streams (x pieces on s_in, row
// chunks on s_cmp as their x prefix lands, y chunks on s_out).  `mark`
// records trace events.
template <class Mark>
void plan_enqueue(rl_spmv_plan_s* pl, const double* x, double* y, double* y_direct, Mark&& mark, double* dx = nullptr,
                  double* dy = nullptr, bool fork = true) {
    if (!dx) dx = pl->x;
    if (!dy) dy = pl->y;
    // Fork: the compute and output streams join s_in before anything else, so
    // under graph capture every chunk is inside the graph even when a chunk
    // waits on no x piece (a leading run of empty rows), and eagerly no
    // chunk of this call overtakes the previous call's y copies.  (The async
    // calls order their slots with events instead and let calls overlap.)
    if (fork) {
        ck(cudaEventRecord(pl->ev_fork, pl->s_in), "event");
        for (auto st : pl->s_cmp) ck(cudaStreamWaitEvent(st, pl->ev_fork, 0), "wait");
        ck(cudaStreamWaitEvent(pl->s_out, pl->ev_fork, 0), "wait");
    }
    mark(pl->s_in);
    const size_t npc = pl->ev_x.size();
    for (size_t i = 0; i < npc; ++i) {
        const uint64_t a = pl->xpiece[i], b = pl->xpiece[i + 1];
        ck(cudaMemcpyAsync(dx + a, x + a, (b - a) * 8, cudaMemcpyHostToDevice, pl->s_in), "H2D x");
        ck(cudaEventRecord(pl->ev_x[i], pl->s_in), "event");
        mark(pl->s_in);
    }
    // x pieces land in order on s_in, so chunk c waits on the event of the
    // last piece its column prefix reaches
    std::vector<size_t> waited(pl->s_cmp.size(), 0);  // pieces each compute stream already waits for
    uint64_t ystart = 0;   // first row of the pending y group
    for (size_t c = 0; c + 1 < pl->chunk_row.size(); ++c) {
        const size_t si = c % pl->s_cmp.size();
        cudaStream_t sc = pl->s_cmp[si];
        size_t need = waited[si];
        while (need < npc && pl->xpiece[need] < pl->chunk_xend[c]) ++need;
        if (need > waited[si]) {
            ck(cudaStreamWaitEvent(sc, pl->ev_x[need - 1], 0), "wait");
            waited[si] = need;
        }
        const uint64_t r0 = pl->chunk_row[c], r1 = pl->chunk_row[c + 1];
        mark(sc);
        if (!rlb::tuning().spmv_plan_probe_nocompute)  // developer probe: the copy pipeline alone
            plan_rows(pl, r0, r1, dx, y_direct ? y_direct : dy, sc);
        mark(sc);
        if (!y_direct && pl->ycut[c]) {
            // the y group [ystart, r1) may span chunks of every compute
            // stream: s_out waits on each (all their work so far is chunks <= c)
            const size_t K = pl->s_cmp.size();
            for (size_t k = 0; k < K && k <= c; ++k) {
                cudaEvent_t ev = pl->ev_y[c * K + k];
                ck(cudaEventRecord(ev, pl->s_cmp[k]), "event");
                ck(cudaStreamWaitEvent(pl->s_out, ev, 0), "wait");
            }
            ck(cudaMemcpyAsync(y + ystart, dy + ystart, (r1 - ystart) * 8, cudaMemcpyDeviceToHost, pl->s_out),
               "D2H y");
            mark(pl->s_out);
            ystart = r1;
        }
    }
}

bool pinned_host(const void* p) {
    cudaPointerAttributes a{};
    const bool ok = cudaPointerGetAttributes(&a, p) == cudaSuccess && a.type == cudaMemoryTypeHost;
    cudaGetLastError();
    return ok;
}

// Wait for every execute_host_async call of the plan.
void plan_wait(rl_spmv_plan_s* pl) {
    ck(cudaStreamSynchronize(pl->s_in), "sync");
    for (auto st : pl->s_cmp) ck(cudaStreamSynchronize(st), "sync");
    ck(cudaStreamSynchronize(pl->s_out), "sync");
}

// One call that returns after enqueueing: x is read and y written
// asynchronously (valid after rl_spmv_plan_wait).  Consecutive calls
// overlap -- call k + 1's x upload runs beside call k's compute and y
// download -- on two device buffer slots.
void plan_execute_host_async(rl_spmv_plan_s* pl, const double* x, double* y) {
    require_ptr(pl, "plan");
    require_ptr(x, "x");
    require_ptr(y, "y");
    const int b = (int)(pl->async_calls % rl_spmv_plan_s::kSlots);
    pl->xs[0] = pl->x;
    pl->ys[0] = pl->y;
    if (!pl->xs[b]) {
        ck(cudaMalloc(&pl->xs[b], std::max<uint64_t>(pl->n, 2) * 8), "plan alloc");
        ck(cudaMalloc(&pl->ys[b], std::max<uint64_t>(pl->m, 1) * 8), "plan alloc");
    }
    if (!pl->ev_cdone[b]) {
        for (auto* e : {&pl->ev_cdone[b], &pl->ev_ydone[b], &pl->ev_xall[b]})
            ck(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event");
    } else {  // the slot's previous call: its compute read x, its y went down
        ck(cudaStreamWaitEvent(pl->s_in, pl->ev_cdone[b], 0), "wait");
        ck(cudaStreamWaitEvent(pl->s_cmp[0], pl->ev_ydone[b], 0), "wait");
    }
    // Whole-vector copies: the overlap comes from consecutive calls (call k +
    // 1's x upload beside call k's y download), so the per-call pipeline
    // chunks, whose copy pieces and cross-stream waits cost more than they
    // hide (tools/micro/plan_stream.py: 8 chunks 1.035 ms per call, 2 chunks
    // 0.809), are not needed.
    double* dx = pl->xs[b];
    double* dy = pl->ys[b];
    cudaStream_t sc = pl->s_cmp[0];
    ck(cudaMemcpyAsync(dx, x, pl->n * 8, cudaMemcpyHostToDevice, pl->s_in), "H2D x");
    ck(cudaEventRecord(pl->ev_xall[b], pl->s_in), "event");
    ck(cudaStreamWaitEvent(sc, pl->ev_xall[b], 0), "wait");
    plan_rows(pl, 0, pl->m, dx, dy, sc);
    ck(cudaEventRecord(pl->ev_cdone[b], sc), "event");
    ck(cudaStreamWaitEvent(pl->s_out, pl->ev_cdone[b], 0), "wait");
    ck(cudaMemcpyAsync(y, dy, pl->m * 8, cudaMemcpyDeviceToHost, pl->s_out), "D2H y");
    ck(cudaEventRecord(pl->ev_ydone[b], pl->s_out), "event");
    ++pl->async_calls;
}

void plan_execute_host(rl_spmv_plan_s* pl, const double* x, double* y) {
    require_ptr(pl, "plan");
    if (pl->async_calls) plan_wait(pl);  // a synchronous call after async ones
    require_ptr(x, "x");
    require_ptr(y, "y");
    static const bool trace = getenv("RL_PLAN_TRACE") != nullptr;
    // y: when the host buffer is pinned and mapped (cudaHostAlloc / registered,
    // UVA), the kernels can store y straight into it over PCIe (tuning key
    // spmv_plan_zero_copy; measured slower than the D2H copies).
    double* y_direct = nullptr;
    if (rlb::tuning().spmv_plan_zero_copy) {
        cudaPointerAttributes ay{};
        if (cudaPointerGetAttributes(&ay, y) == cudaSuccess && ay.type == cudaMemoryTypeHost &&
            ay.devicePointer != nullptr)
            y_direct = static_cast<double*>(ay.devicePointer);
        cudaGetLastError();
    }
    // Pinned x and y: the whole call is one CUDA graph (captured once per
    // (x, y) pair), so the ~60 copies, waits and launches cost one launch of
    // host time instead of pacing the copy engines.
    if (!trace && !y_direct && rlb::tuning().spmv_plan_graph) {
        // the cached graph is replayed only for the same pointers, still
        // page-locked (a buffer freed and re-allocated pageable at the same
        // address takes the eager path)
        const bool pinned = pinned_host(x) && pinned_host(y);
        if (pl->gexec && (pl->gx != x || pl->gy != y || !pinned)) {
            cudaGraphExecDestroy(pl->gexec);
            pl->gexec = nullptr;
        }
        if (!pl->gexec && pinned) {
            const uint64_t before = rlb::g_launches.load();
            ck(cudaStreamBeginCapture(pl->s_in, cudaStreamCaptureModeThreadLocal), "graph capture");
            cudaGraph_t g = nullptr;
            try {
                plan_enqueue(pl, x, y, nullptr, [](cudaStream_t) {});
                for (size_t k = 0; k < pl->s_cmp.size(); ++k)
                    ck(cudaEventRecord(pl->ev_join[k], pl->s_cmp[k]), "event");
                ck(cudaEventRecord(pl->ev_join.back(), pl->s_out), "event");
                for (auto e : pl->ev_join) ck(cudaStreamWaitEvent(pl->s_in, e, 0), "wait");
            } catch (...) {
                cudaStreamEndCapture(pl->s_in, &g);
                if (g) cudaGraphDestroy(g);
                throw;
            }
            ck(cudaStreamEndCapture(pl->s_in, &g), "graph capture");
            const cudaError_t e = cudaGraphInstantiate(&pl->gexec, g, 0);
            cudaGraphDestroy(g);
            ck(e, "graph instantiate");
            pl->graph_launches = rlb::g_launches.load() - before;
            rlb::g_launches.fetch_sub(pl->graph_launches);  // counted per replay below
            pl->gx = x;
            pl->gy = y;
        }
        if (pl->gexec) {
            ck(cudaGraphLaunch(pl->gexec, pl->s_in), "graph launch");
            rlb::note_launch(pl->graph_launches);
            ck(cudaStreamSynchronize(pl->s_in), "sync");
            return;
        }
    }
    std::vector<cudaEvent_t> tev;
    auto mark = [&](cudaStream_t st) {
        if (!trace) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, st);
        tev.push_back(e);
    };
    plan_enqueue(pl, x, y, y_direct, mark);
    ck(cudaStreamSynchronize(pl->s_out), "sync");
    for (auto st : pl->s_cmp) ck(cudaStreamSynchronize(st), "sync");
    ck(cudaStreamSynchronize(pl->s_in), "sync");
    if (trace && !tev.empty()) {
        fprintf(stderr, "plan trace (us from start):");
        for (size_t i = 1; i < tev.size(); ++i) {
            float ms = 0;
            cudaEventElapsedTime(&ms, tev[0], tev[i]);
            fprintf(stderr, " %.0f", ms * 1e3);
        }
        fprintf(stderr, "\n");
        for (auto e : tev) cudaEventDestroy(e);
    }
}

// ---------------------------------------------------------------------------
// Error plumbing
// ---------------------------------------------------------------------------
void put(rl_kchar* out, const KernelCharacterization& k) {
    if (out) {
        out->work_flops = k.work_flops;
        out->traffic_bytes = k.traffic_bytes;
    }
}

ExecutionUnit unit_of(rl_unit u) {
    if (u != RL_CUDA_CORE && u != RL_TENSOR_CORE)
        throw Error(ErrorKind::ValidationError, "unknown execution unit " + std::to_string((int)u));
    return static_cast<ExecutionUnit>(u);
}
Precision prec_of(rl_precision p) {
    if (p != RL_FP64 && p != RL_FP32 && p != RL_FP16)
        throw Error(ErrorKind::ValidationError, "unknown precision " + std::to_string((int)p));
    return static_cast<Precision>(p);
}
const StencilShape& shape_of(const char* preset) {
    if (!preset) throw Error(ErrorKind::ValidationError, "preset must not be null");
    return stencil_preset(preset);
}
HardwareSpec spec_of(const rl_hw_spec* s) {
    require_ptr(s, "spec");
    HardwareSpec h;
    h.name = std::string(s->name, strnlen(s->name, sizeof s->name));
    h.memory_bandwidth = s->memory_bandwidth;
    h.l2_cache_bytes = s->l2_cache_bytes;
    std::memcpy(h.peaks, s->peaks, sizeof h.peaks);
    return h;
}
void spec_out(rl_hw_spec* o, const HardwareSpec& h) {
    require_ptr(o, "out");
    std::memset(o, 0, sizeof *o);
    std::strncpy(o->name, h.name.c_str(), sizeof o->name - 1);
    o->memory_bandwidth = h.memory_bandwidth;
    o->l2_cache_bytes = h.l2_cache_bytes;
    std::memcpy(o->peaks, h.peaks, sizeof o->peaks);
}
}  // namespace

// ===========================================================================
// extern "C"
// ===========================================================================
extern "C" {

const char* rl_last_error(void) { return last_error_slot().c_str(); }
const char* rl_version(void) { return "rooflens-b200 0.1.0 (sm_100a)"; }
uint64_t rl_kernel_launches(void) { return rlb::g_launches.load(); }

int rl_scale_model(uint64_t n, rl_precision p, rl_kchar* out) {
    return guarded([&] { put(out, scale_model(n, prec_of(p))); });
}
int rl_gemv_model(uint64_t m, uint64_t n, rl_precision p, rl_kchar* out) {
    return guarded([&] { put(out, gemv_model(m, n, prec_of(p))); });
}
int rl_spmv_generic_model(uint64_t rows, uint64_t cols, uint64_t nnz, uint64_t ic, uint64_t ib,
                          uint64_t pc, uint64_t pb, rl_precision p, rl_kchar* out) {
    return guarded([&] { put(out, spmv_generic_model({rows, cols, nnz}, {ic, ib, pc, pb}, prec_of(p))); });
}
int rl_spmv_csr_model(uint64_t rows, uint64_t cols, uint64_t nnz, uint64_t ib, rl_precision p,
                      rl_kchar* out) {
    return guarded([&] { put(out, spmv_csr_model({rows, cols, nnz}, ib, prec_of(p))); });
}
int rl_stencil_model(const char* preset, rl_precision p, uint64_t t, rl_kchar* out) {
    return guarded([&] { put(out, stencil_model(shape_of(preset), prec_of(p), t)); });
}
int rl_stencil_preset(const char* name, int* dim, uint64_t* points, int* radius) {
    return guarded([&] {
        const StencilShape& s = shape_of(name);
        if (dim) *dim = s.dimensionality;
        if (points) *points = s.point_count;
        if (radius) *radius = s.radius;
    });
}
int rl_stencil_default_weights(const char* name, double* w, uint64_t cap) {
    return guarded([&] {
        const auto v = stencil_default_weights(shape_of(name).name);
        if (cap < v.size()) throw Error(ErrorKind::InvalidCount, "weights capacity too small");
        require_ptr(w, "weights");
        std::memcpy(w, v.data(), v.size() * sizeof(double));
    });
}

int rl_scale(rl_unit u, rl_precision p, double* a, const double* b, double q, uint64_t n,
             rl_stream s, rl_kchar* out) {
    return guarded([&] { put(out, rooflens::b200::scale(unit_of(u), prec_of(p), a, b, q, n, s)); });
}
int rl_gemv(rl_unit u, rl_precision p, uint64_t m, uint64_t n, const double* A, const double* x, double* y,
            rl_stream s, rl_kchar* out) {
    return guarded([&] { put(out, rooflens::b200::gemv(unit_of(u), prec_of(p), m, n, A, x, y, s)); });
}
int rl_spmv_csr(rl_unit u, rl_precision p, uint64_t m, uint64_t n, uint64_t nnz, const int32_t* rp,
                const int32_t* col, const double* val, const double* x, double* y, rl_stream s,
                rl_kchar* out) {
    return guarded([&] {
        put(out, rooflens::b200::spmv_csr(unit_of(u), prec_of(p), {m, n, nnz}, rp, col, val, x, y, s));
    });
}
int rl_spmv_csr_rows(rl_unit u, rl_precision p, uint64_t r0, uint64_t r1, const int32_t* rp,
                     const int32_t* col, const double* val, const double* x, int64_t col_base,
                     double* y, rl_stream s) {
    return guarded([&] {
        rooflens::b200::spmv_csr_rows(unit_of(u), prec_of(p), r0, r1, rp, col, val, x, col_base, y, s);
    });
}
int rl_stencil(rl_unit u, rl_precision p, const char* preset, const uint64_t* dims,
               const double* weights, uint64_t steps, double* uu, double* v, rl_stream s,
               rl_kchar* out) {
    return guarded([&] {
        require_ptr(dims, "dims");
        put(out, rooflens::b200::stencil(unit_of(u), prec_of(p), shape_of(preset), dims, weights,
                                         steps, uu, v, s));
    });
}
int rl_stencil_temporal(rl_unit u, rl_precision p, const char* preset, const uint64_t* dims,
                        const double* weights, uint64_t steps, uint64_t t, double* uu, double* v,
                        rl_stream s, int* result_in_v, rl_kchar* out) {
    return guarded([&] {
        require_ptr(dims, "dims");
        put(out, rooflens::b200::stencil_temporal(unit_of(u), prec_of(p), shape_of(preset), dims, weights,
                                                  steps, t, uu, v, s, result_in_v));
    });
}
int rl_stencil_sweep(rl_unit u, rl_precision p, const char* preset, const uint64_t* dims,
                     const double* weights, uint64_t o0, uint64_t o1, const double* uu, double* v,
                     rl_stream s) {
    return guarded([&] {
        require_ptr(dims, "dims");
        rooflens::b200::stencil_sweep(unit_of(u), prec_of(p), shape_of(preset), dims, weights, o0,
                                      o1, uu, v, s);
    });
}

int rl_scale_host(rl_unit u, rl_precision p, double* a, const double* b, double q, uint64_t n,
                  rl_kchar* out) {
    return guarded([&] { put(out, scale_host(unit_of(u), prec_of(p), a, b, q, n)); });
}
int rl_spmv_csr_host(rl_unit u, rl_precision p, uint64_t m, uint64_t n, uint64_t nnz,
                     const int32_t* rp, const int32_t* col, const double* val, const double* x,
                     double* y, rl_kchar* out) {
    return guarded([&] { put(out, spmv_host(unit_of(u), prec_of(p), m, n, nnz, rp, col, val, x, y)); });
}
int rl_stencil_host(rl_unit u, rl_precision p, const char* preset, const uint64_t* dims,
                    const double* weights, uint64_t steps, double* uu, double* v, rl_kchar* out) {
    return guarded([&] {
        put(out, stencil_host(unit_of(u), prec_of(p), preset, dims, weights, steps, uu, v));
    });
}
int rl_spmv_plan_create(rl_unit u, rl_precision p, uint64_t m, uint64_t n, uint64_t nnz,
                        const int32_t* rp, const int32_t* col, const double* val, rl_spmv_plan* out) {
    return guarded([&] {
        require_ptr(out, "out");
        *out = nullptr;
        *out = plan_create(unit_of(u), prec_of(p), m, n, nnz, rp, col, val);
    });
}
int rl_spmv_plan_execute_host_async(rl_spmv_plan pl, const double* x, double* y, rl_kchar* out) {
    return guarded([&] {
        plan_execute_host_async(pl, x, y);
        put(out, pl->kc);
    });
}
int rl_spmv_plan_wait(rl_spmv_plan pl) {
    return guarded([&] {
        require_ptr(pl, "plan");
        plan_wait(pl);
    });
}
int rl_spmv_plan_execute_host(rl_spmv_plan pl, const double* x, double* y, rl_kchar* out) {
    return guarded([&] {
        plan_execute_host(pl, x, y);
        put(out, pl->kc);
    });
}
int rl_spmv_plan_execute(rl_spmv_plan pl, const double* x, double* y, rl_stream s, rl_kchar* out) {
    return guarded([&] {
        require_ptr(pl, "plan");
        require_ptr(x, "x");
        require_ptr(y, "y");
        if (rlb::tuning().spmv_plan_dev_chunks) {  // developer probe: the execute_host chunks, no copies
            for (size_t c = 0; c + 1 < pl->chunk_row.size(); ++c)
                plan_rows(pl, pl->chunk_row[c], pl->chunk_row[c + 1], x, y, static_cast<cudaStream_t>(s));
        } else {
            plan_rows(pl, 0, pl->m, x, y, static_cast<cudaStream_t>(s));
        }
        put(out, pl->kc);
    });
}
int rl_spmv_plan_info(rl_spmv_plan pl, int* tiled, uint64_t* layout_bytes) {
    return guarded([&] {
        require_ptr(pl, "plan");
        if (tiled) *tiled = pl->colsort ? 4 : 0;
        if (layout_bytes) *layout_bytes = pl->layout_bytes;
    });
}
int rl_spmv_plan_destroy(rl_spmv_plan pl) {
    return guarded([&] {
        if (pl && pl->async_calls) {  // async calls still in flight read / write the plan's buffers
            cudaStreamSynchronize(pl->s_in);
            for (auto st : pl->s_cmp) cudaStreamSynchronize(st);
            cudaStreamSynchronize(pl->s_out);
        }
        delete pl;
    });
}
int rl_host_workspace_release(void) {
    return guarded([&] {
        std::lock_guard<std::mutex> lock(ws().mu);
        ws().release();
    });
}

int rl_fill_uniform(double* out, uint64_t n, uint64_t seed, uint64_t sid, uint64_t idx0, int kind,
                    rl_stream s) {
    return guarded([&] {
        require_ptr(out, "out");
        ck(rlb::launch_fill_uniform(out, n, seed, sid, idx0, kind, static_cast<cudaStream_t>(s)),
           "fill_uniform");
    });
}
int rl_gen_band_csr(uint64_t m_local, uint64_t row0, uint64_t n, uint32_t k, uint64_t hb,
                    uint64_t seed, int32_t* rp, int32_t* col, double* val, rl_stream s) {
    return guarded([&] {
        if (k == 0 || k > 64 || n < k || hb + 1 < k)
            throw Error(ErrorKind::InvalidCount, "gen_band_csr: need 1 <= k <= 64, k <= n, k <= 2*hb+1");
        if ((unsigned __int128)(row0 + m_local) * k > 0x7fffffffull)
            throw Error(ErrorKind::InvalidRange, "gen_band_csr: nnz exceeds int32");
        require_ptr(rp, "row_ptr");
        ck(rlb::launch_gen_band_csr(m_local, row0, n, k, hb, seed, rp, col, val,
                                    static_cast<cudaStream_t>(s)),
           "gen_band_csr");
    });
}
int rl_stencil_init(double* u, const uint64_t* dims, int dim, uint64_t o0, uint64_t o1,
                    int radius, uint64_t seed, rl_stream s) {
    return guarded([&] {
        require_ptr(u, "u");
        require_ptr(dims, "dims");
        if (dim != 2 && dim != 3) throw Error(ErrorKind::ValidationError, "dim must be 2 or 3");
        const uint64_t outer = dim == 2 ? dims[1] : dims[2];
        if (o1 < o0 || o1 > outer) throw Error(ErrorKind::InvalidRange, "outer range outside the grid");
        ck(rlb::launch_stencil_init(u, dims[0], dims[1], dim == 3 ? dims[2] : 1, dim, o0, o1, radius,
                                    seed, static_cast<cudaStream_t>(s)),
           "stencil_init");
    });
}

int rl_mtx_stats(const char* path, uint64_t* rows, uint64_t* cols, uint64_t* nnz) {
    return guarded([&] {
        require_ptr(path, "path");
        const SparseMatrixStats s = mtx_stats(path);
        if (rows) *rows = s.rows;
        if (cols) *cols = s.cols;
        if (nnz) *nnz = s.nnz;
    });
}
int rl_mtx_read_csr(const char* path, uint64_t row_cap, uint64_t nnz_cap, int32_t* rp, int32_t* col,
                    double* val, uint64_t* rows, uint64_t* cols, uint64_t* nnz) {
    return guarded([&] {
        require_ptr(path, "path");
        std::vector<int32_t> vrp, vcol;
        std::vector<double> vval;
        const SparseMatrixStats s = mtx_read_csr(path, vrp, vcol, vval);
        if (row_cap < s.rows + 1 || nnz_cap < s.nnz)
            throw Error(ErrorKind::InvalidCount, "CSR buffers too small: need " + std::to_string(s.rows + 1) +
                                                     " row pointers and " + std::to_string(s.nnz) + " entries");
        require_ptr(rp, "row_ptr");
        require_ptr(col, "col");
        require_ptr(val, "val");
        std::memcpy(rp, vrp.data(), vrp.size() * 4);
        std::memcpy(col, vcol.data(), vcol.size() * 4);
        std::memcpy(val, vval.data(), vval.size() * 8);
        if (rows) *rows = s.rows;
        if (cols) *cols = s.cols;
        if (nnz) *nnz = s.nnz;
    });
}
int rl_matrix_analysis_of(uint64_t rows, uint64_t cols, uint64_t nnz, const rl_hw_spec* spec,
                          rl_precision p, rl_matrix_analysis* out) {
    return guarded([&] {
        require_ptr(out, "out");
        const HardwareSpec h = spec_of(spec);
        const Precision pr = prec_of(p);
        const KernelCharacterization k = spmv_csr_model({rows, cols, nnz}, kDefaultIndexBytes, pr);
        const double I = k.intensity();
        const double B = machine_balance(h, ExecutionUnit::CudaCore, pr);
        std::memset(out, 0, sizeof *out);
        out->work_flops = k.work_flops;
        out->traffic_bytes = k.traffic_bytes;
        out->boundedness = static_cast<int>(classify(I, B));
        out->kernel_ceiling = kernel_speedup_ceiling(tensor_alpha(h, pr), B, I, &out->kernel_ceiling_warnings);
        out->workload_ceiling = workload_ceiling(I, B);
        out->csr_bytes = k.traffic_bytes;
        out->fits_in_l2 = static_cast<double>(k.traffic_bytes) <= h.l2_cache_bytes;
    });
}
int rl_load_spec(const char* text, rl_hw_spec* out) {
    return guarded([&] {
        require_ptr(text, "json_text");
        spec_out(out, load_spec(text));
    });
}
int rl_load_spec_file(const char* path, rl_hw_spec* out) {
    return guarded([&] {
        require_ptr(path, "path");
        spec_out(out, load_spec_file(path));
    });
}
int rl_serialize_spec(const rl_hw_spec* s, char* buf, uint64_t cap, uint64_t* length) {
    return guarded([&] {
        const std::string text = serialize_spec(spec_of(s));
        if (length) *length = text.size();
        if (!buf) return;
        if (cap < text.size() + 1)
            throw Error(ErrorKind::InvalidRange, "serialize_spec: buffer of " + std::to_string(cap) +
                                                     " bytes cannot hold " + std::to_string(text.size() + 1));
        std::memcpy(buf, text.c_str(), text.size() + 1);
    });
}
int rl_builtin_spec(const char* name, rl_hw_spec* out) {
    return guarded([&] {
        require_ptr(name, "name");
        spec_out(out, builtin_spec(name));
    });
}
int rl_machine_balance(const rl_hw_spec* s, rl_unit u, rl_precision p, double* out) {
    return guarded([&] { *out = machine_balance(spec_of(s), unit_of(u), prec_of(p)); });
}
int rl_tensor_alpha(const rl_hw_spec* s, rl_precision p, double* out) {
    return guarded([&] { *out = tensor_alpha(spec_of(s), prec_of(p)); });
}
int rl_attainable(const rl_hw_spec* s, rl_unit u, rl_precision p, double i, double* out) {
    return guarded([&] { *out = attainable(spec_of(s), unit_of(u), prec_of(p), i); });
}
int rl_classify(double i, double b) { return static_cast<int>(classify(i, b)); }
int rl_ridge_point(const rl_hw_spec* s, rl_unit u, rl_precision p, double* out) {
    return guarded([&] {
        require_ptr(s, "spec");
        require_ptr(out, "out");
        *out = ridge_point(spec_of(s), unit_of(u), prec_of(p));
    });
}
int rl_sample_curve(const rl_hw_spec* s, rl_unit u, rl_precision p, double i_min, double i_max, uint64_t n,
                    double* xs, double* ys, uint64_t capacity, uint64_t* count) {
    return guarded([&] {
        require_ptr(s, "spec");
        require_ptr(count, "count");
        const auto pts = sample_curve(spec_of(s), unit_of(u), prec_of(p), i_min, i_max, (std::size_t)n);
        if (pts.size() > capacity) throw Error(ErrorKind::InvalidRange, "output capacity too small");
        require_ptr(xs, "intensity");
        require_ptr(ys, "attainable");
        for (std::size_t k = 0; k < pts.size(); ++k) {
            xs[k] = pts[k].first;
            ys[k] = pts[k].second;
        }
        *count = pts.size();
    });
}
int rl_mem_cmp_ratio(double b, double i, double* out) {
    return guarded([&] {
        require_ptr(out, "out");
        *out = mem_cmp_ratio(b, i);
    });
}
int rl_overlapped_total(double tc, double tm, double to, double* out) {
    return guarded([&] {
        require_ptr(out, "out");
        *out = overlapped_total(tc, tm, to);
    });
}
int rl_unoverlapped_speedup(double tc, double tm, double to, double a, double* out) {
    return guarded([&] { *out = unoverlapped_speedup(tc, tm, to, a); });
}
int rl_kernel_speedup_ceiling(double a, double b, double i, double* out, int* nw) {
    return guarded([&] { *out = kernel_speedup_ceiling(a, b, i, nw); });
}
int rl_tensor_core_ceiling(double a, double* out) {
    return guarded([&] { *out = tensor_core_ceiling(a); });
}
int rl_workload_ceiling(double i, double b, double* out) {
    return guarded([&] { *out = workload_ceiling(i, b); });
}
int rl_min_temporal_depth(double b, double i, uint64_t* out) {
    return guarded([&] { *out = min_temporal_depth(b, i); });
}
int rl_tc_scale_trick_throughput(double p, uint64_t m, uint64_t n, double* out) {
    return guarded([&] { *out = tc_scale_trick_throughput(p, m, n); });
}

namespace {
// Copy `text` (NUL-terminated) into a caller buffer: *length (optional) gets
// the full length; a null buffer only sizes; a short buffer is InvalidRange.
void text_out(const std::string& text, char* buf, uint64_t cap, uint64_t* length, const char* what) {
    if (length) *length = text.size();
    if (!buf) return;
    if (cap < text.size() + 1)
        throw Error(ErrorKind::InvalidRange, std::string(what) + ": buffer of " + std::to_string(cap) +
                                                 " bytes cannot hold " + std::to_string(text.size() + 1));
    std::memcpy(buf, text.c_str(), text.size() + 1);
}

void bound_out(const SpeedupBound& b, rl_speedup_bound* out, char* text, uint64_t cap, uint64_t* length) {
    require_ptr(out, "out");
    out->value = b.value;
    out->kind = static_cast<int>(b.kind);
    out->n_assumptions = static_cast<int>(b.assumptions.size());
    out->n_warnings = static_cast<int>(b.warnings.size());
    std::string t;
    for (const std::string& a : b.assumptions) t += a + "\n";
    for (const std::string& w : b.warnings) t += w + "\n";
    text_out(t, text, cap, length, "speedup bound text");
}
}  // namespace

const char* rl_bound_kind_name(int kind) {
    return (kind >= 0 && kind <= 3) ? to_string(static_cast<BoundKind>(kind)) : "?";
}
int rl_unoverlapped_bound(double tc, double tm, double to, double a, rl_speedup_bound* out, char* text,
                          uint64_t cap, uint64_t* length) {
    return guarded([&] { bound_out(unoverlapped_bound(tc, tm, to, a), out, text, cap, length); });
}
int rl_kernel_ceiling_bound(double a, double b, double i, rl_speedup_bound* out, char* text, uint64_t cap,
                            uint64_t* length) {
    return guarded([&] { bound_out(kernel_ceiling_bound(a, b, i), out, text, cap, length); });
}
int rl_tensor_core_bound(double a, rl_speedup_bound* out, char* text, uint64_t cap, uint64_t* length) {
    return guarded([&] { bound_out(tensor_core_bound(a), out, text, cap, length); });
}
int rl_workload_bound(double i, double b, rl_speedup_bound* out, char* text, uint64_t cap, uint64_t* length) {
    return guarded([&] { bound_out(workload_bound(i, b), out, text, cap, length); });
}

int rl_analysis_render(const rl_hw_spec* spec, rl_precision p, const char* kernel_name, uint64_t work_flops,
                       uint64_t traffic_bytes, const double* balance_override,
                       const double* single_step_intensity, int format, char* buf, uint64_t cap,
                       uint64_t* length) {
    return guarded([&] {
        require_ptr(spec, "spec");
        if (format < RL_REPORT_TEXT || format > RL_REPORT_CSV)
            throw Error(ErrorKind::ValidationError, "report format must be text, json or csv");
        KernelCharacterization k;
        k.kernel_name = kernel_name ? kernel_name : "";
        k.work_flops = work_flops;
        k.traffic_bytes = traffic_bytes;
        std::optional<double> bo, si;
        if (balance_override) bo = *balance_override;
        if (single_step_intensity) si = *single_step_intensity;
        const AnalysisReport r = build_analysis(spec_of(spec), prec_of(p), k, bo, si);
        text_out(format == RL_REPORT_TEXT ? render_text(r) : format == RL_REPORT_JSON ? render_json(r) : render_csv(r),
                 buf, cap, length, "analysis report");
    });
}

int rl_fp64_peak_launch(rl_unit u, uint64_t iters, rl_stream s, double* sink, double* flops) {
    return guarded([&] {
        require_ptr(sink, "sink");
        require_ptr(flops, "flops_out");
        ck(rlb::launch_fp64_peak(unit_of(u) == ExecutionUnit::TensorCore, iters, sink, flops,
                                 static_cast<cudaStream_t>(s)),
           "fp64_peak");
    });
}

// Tuning keys.  Product keys select a documented variant a caller may want
// (the tensor-core stencil form, plan layouts, graph replay, the long-row
// path); the rest are sweep knobs of the kernels' launch shapes, accepted
// only with RL_DEV_TUNING=1 in the environment (tests and tools/sweep.py).
int rl_tuning_set(const char* key, int64_t value, int64_t* previous) {
    return guarded([&] {
        require_ptr(key, "key");
        struct Key {
            const char* name;
            int rlb::Tuning::*field;
            bool product;
        };
        static const Key keys[] = {
        {"scale_blocks_per_sm", &rlb::Tuning::scale_blocks_per_sm, false},
        {"dist_graph", &rlb::Tuning::dist_graph, true},
        {"spmv_rows", &rlb::Tuning::spmv_rows, false},
        {"gemv_rows", &rlb::Tuning::gemv_rows, false},
        {"gemv_unroll", &rlb::Tuning::gemv_unroll, false},
        {"spmv_blocks_per_sm", &rlb::Tuning::spmv_blocks_per_sm, false},
        {"spmv_sched", &rlb::Tuning::spmv_sched, false},
        {"spmv_threads", &rlb::Tuning::spmv_threads, false},
        {"spmv_plan_chunks", &rlb::Tuning::spmv_plan_chunks, true},
        {"spmv_plan_zero_copy", &rlb::Tuning::spmv_plan_zero_copy, false},
        {"spmv_long_rows", &rlb::Tuning::spmv_long_rows, true},
        {"spmv_long_min", &rlb::Tuning::spmv_long_min, true},
        {"spmv_long_piece", &rlb::Tuning::spmv_long_piece, false},
        {"spmv_long_group", &rlb::Tuning::spmv_long_group, false},
        {"spmv_plan_graph", &rlb::Tuning::spmv_plan_graph, true},
        {"spmv_plan_taper", &rlb::Tuning::spmv_plan_taper, false},
        {"spmv_plan_xpieces", &rlb::Tuning::spmv_plan_xpieces, false},
        {"spmv_plan_colsort", &rlb::Tuning::spmv_plan_colsort, true},
        {"spmv_colsort_fixed", &rlb::Tuning::spmv_colsort_fixed, true},
        {"stencil_tb27r", &rlb::Tuning::stencil_tb27r, false},
        {"spmv_plan_streams", &rlb::Tuning::spmv_plan_streams, false},
        {"spmv_plan_colsort_chunks", &rlb::Tuning::spmv_plan_colsort_chunks, false},
        {"spmv_colsort_window", &rlb::Tuning::spmv_colsort_window, false},
        {"spmv_colsort_classes", &rlb::Tuning::spmv_colsort_classes, false},
        {"spmv_colsort_tc_shape", &rlb::Tuning::spmv_colsort_tc_shape, false},
        {"spmv_colsort_cc_shape", &rlb::Tuning::spmv_colsort_cc_shape, false},
        {"spmv_colsort_vec", &rlb::Tuning::spmv_colsort_vec, false},
        {"spmv_colsort_fuse", &rlb::Tuning::spmv_colsort_fuse, false},
        {"spmv_plan_colsort_blocks", &rlb::Tuning::spmv_plan_colsort_blocks, false},
        {"spmv_plan_edge_blocks", &rlb::Tuning::spmv_plan_edge_blocks, false},
        {"spmv_plan_dev_chunks", &rlb::Tuning::spmv_plan_dev_chunks, false},
        {"spmv_plan_probe_nocompute", &rlb::Tuning::spmv_plan_probe_nocompute, false},
        {"spmv_colsort_spread", &rlb::Tuning::spmv_colsort_spread, false},
        {"spmv_plan_ygroups", &rlb::Tuning::spmv_plan_ygroups, false},
        {"stencil_r_ctas_per_sm", &rlb::Tuning::stencil_r_ctas_per_sm, false},
        {"stencil_tb_waves", &rlb::Tuning::stencil_tb_waves, false},
        {"stencil_tb_tma", &rlb::Tuning::stencil_tb_tma, false},
        {"stencil_tb3_chunks", &rlb::Tuning::stencil_tb3_chunks, false},
        {"stencil_tb3_shape", &rlb::Tuning::stencil_tb3_shape, false},
        {"stencil_tb3_l2promo", &rlb::Tuning::stencil_tb3_l2promo, false},
        {"stencil3d_cc_stages", &rlb::Tuning::stencil3d_cc_stages, false},
        {"stencil_tc_concat", &rlb::Tuning::stencil_tc_concat, false},
        {"stencil_cc27x2", &rlb::Tuning::stencil_cc27x2, false},
        {"stencil_r_cc_stages", &rlb::Tuning::stencil_r_cc_stages, false},
        {"stencil_r_tc_stages", &rlb::Tuning::stencil_r_tc_stages, false},
        {"stencil_r_sym", &rlb::Tuning::stencil_r_sym, false},
        {"stencil_r_l2promo", &rlb::Tuning::stencil_r_l2promo, false},
        {"spmv_tc_blocks_per_sm", &rlb::Tuning::spmv_tc_blocks_per_sm, false},
        {"spmv_tc_threads", &rlb::Tuning::spmv_tc_threads, false},
        {"spmv_tc_rows", &rlb::Tuning::spmv_tc_rows, false},
        {"spmv_l1_carveout", &rlb::Tuning::spmv_l1_carveout, false},
        {"spmv_xhint", &rlb::Tuning::spmv_xhint, false},
        {"scale_unroll", &rlb::Tuning::scale_unroll, false},
        {"stencil2d_rows", &rlb::Tuning::stencil2d_rows, false},
        {"stencil3d_zchunk", &rlb::Tuning::stencil3d_zchunk, false},
        {"tc_stencil_zchunk", &rlb::Tuning::tc_stencil_zchunk, false},
        {"stencil_tma", &rlb::Tuning::stencil_tma, true},
        {"stencil_ctas_per_sm", &rlb::Tuning::stencil_ctas_per_sm, false},
        {"stencil_rows_per_thread", &rlb::Tuning::stencil_rows_per_thread, false},
        {"stencil2d_rows_per_thread", &rlb::Tuning::stencil2d_rows_per_thread, false},
        {"stencil_tc_ctas_per_sm", &rlb::Tuning::stencil_tc_ctas_per_sm, false},
        {"stencil_tc3d_ctas_per_sm", &rlb::Tuning::stencil_tc3d_ctas_per_sm, false},
        {"stencil_tc3d_mode", &rlb::Tuning::stencil_tc3d_mode, false},
        {"stencil_tc1_ctas_per_sm", &rlb::Tuning::stencil_tc1_ctas_per_sm, false},
        {"stencil_tc3d_hybrid", &rlb::Tuning::stencil_tc3d_hybrid, true},
        {"stencil_tch_ctas_per_sm", &rlb::Tuning::stencil_tch_ctas_per_sm, false},
        {"stencil_tch_k8", &rlb::Tuning::stencil_tch_k8, false},
        {"stencil_tch_stages", &rlb::Tuning::stencil_tch_stages, false},
        {"stencil3d_balance", &rlb::Tuning::stencil3d_balance, false},
        {"stencil_tc2d_hybrid", &rlb::Tuning::stencil_tc2d_hybrid, true},
        {"stencil_tch_tpw", &rlb::Tuning::stencil_tch_tpw, false},
        };
        static const bool dev = [] {
            const char* e = std::getenv("RL_DEV_TUNING");
            return e != nullptr && e[0] == '1';
        }();
        const std::string k(key);
        const Key* hit = nullptr;
        for (const Key& e : keys)
            if (k == e.name) hit = &e;
        if (!hit) throw Error(ErrorKind::ValidationError, "unknown tuning key '" + k + "'");
        if (!hit->product && !dev)
            throw Error(ErrorKind::ValidationError, "'" + k + "' is a developer sweep key (set RL_DEV_TUNING=1)");
        int* slot = &(rlb::tuning().*(hit->field));
        if (previous) *previous = *slot;
        if (value < -1) throw Error(ErrorKind::InvalidRange, "tuning values must be >= -1");
        *slot = static_cast<int>(value);
    });
}

}  // extern "C"
