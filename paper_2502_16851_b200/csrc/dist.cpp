// dist.cpp -- the sharded hot path (north_star): one process
// per GPU, NCCL point-to-point over NVLink/NVSwitch for the halo exchanges,
// the library's sm_100a kernels as the per-part compute.
//
//   STREAM Scale  contiguous chunks, no communication.
//   CSR SpMV      row blocks with x windows [r0 - hb, r1 + hb); per call the
//                 band halo of x (hb doubles per side) is exchanged with the
//                 neighbours in one NCCL group on a high-priority stream while
//                 the interior rows (band inside the owned x) run; the two edge
//                 row blocks follow.
//   Stencils      slabs of the outer axis with `radius` ghost layers; per
//                 timestep the ghosts are exchanged while the slab interior is
//                 swept, then the edge layers.  Timestep pairs (u->v->u) are
//                 captured once into a CUDA graph, so a timestep costs one
//                 graph launch of host time per two steps.
//
// Parts: a job has P = world * parts_local parts; rank r owns parts
// [r*L, (r+1)*L).  The exchange schedule (halo_schedule) lists, per rank and in
// posting order, the sends and receives of every part boundary; peers are
// ranks, so parts on the same rank exchange through NCCL self send/recv.  Both
// sides of a rank pair post their transfers in boundary order, which is what
// NCCL's in-order matching of sends and receives per peer needs.
//
// The reference has no multi-GPU form (reference SPEC.md:101 lists multi-GPU
// aggregation as a non-goal); the accounting each call returns is the
// reference model of the global problem (kernels.cpp:74-155).
#include <dlfcn.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime.h>
#include <nccl.h>  // types only: the library itself is dlopen'd (NcclApi)

#include "boundary.h"
#include "kernels.h"

using namespace rooflens::b200;

namespace {

// ---------------------------------------------------------------------------
// NCCL, loaded at the first rl_dist_unique_id / rl_dist_init.  Preference:
// the copy already mapped into the process (torch's, so one NCCL serves both),
// then $RL_NCCL_LIBRARY, then the loader's libnccl.so.2.
// ---------------------------------------------------------------------------
struct NcclApi {
    decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
    decltype(&ncclCommInitRank) CommInitRank = nullptr;
    decltype(&ncclCommDestroy) CommDestroy = nullptr;
    decltype(&ncclSend) Send = nullptr;
    decltype(&ncclRecv) Recv = nullptr;
    decltype(&ncclGroupStart) GroupStart = nullptr;
    decltype(&ncclGroupEnd) GroupEnd = nullptr;
    decltype(&ncclAllReduce) AllReduce = nullptr;
    decltype(&ncclGetErrorString) GetErrorString = nullptr;
    decltype(&ncclGetVersion) GetVersion = nullptr;
    std::string error;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h)
            if (const char* p = std::getenv("RL_NCCL_LIBRARY")) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char* e = dlerror();
            api.error = std::string("cannot load libnccl.so.2: ") + (e ? e : "unknown dlopen error");
            return;
        }
        bool ok = true;
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            ok = ok && fn != nullptr;
        };
        sym(api.GetUniqueId, "ncclGetUniqueId");
        sym(api.CommInitRank, "ncclCommInitRank");
        sym(api.CommDestroy, "ncclCommDestroy");
        sym(api.Send, "ncclSend");
        sym(api.Recv, "ncclRecv");
        sym(api.GroupStart, "ncclGroupStart");
        sym(api.GroupEnd, "ncclGroupEnd");
        sym(api.AllReduce, "ncclAllReduce");
        sym(api.GetErrorString, "ncclGetErrorString");
        sym(api.GetVersion, "ncclGetVersion");
        if (!ok) api.error = "libnccl.so.2 lacks a required symbol (NCCL >= 2.7 needed for send/recv)";
    });
    if (!api.error.empty()) throw NcclError(ncclSystemError, "NcclError: " + api.error);
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess && r != ncclInProgress)
        throw NcclError(static_cast<int>(r), std::string("NcclError: ") + what + ": " + nccl().GetErrorString(r));
}

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw CudaError(static_cast<int>(e), std::string("CudaError: ") + what + ": " + cudaGetErrorName(e) + " (" +
                                                 cudaGetErrorString(e) + ")");
}

void require(const void* p, const char* what) {
    if (!p) throw Error(ErrorKind::ValidationError, std::string(what) + " must not be null");
}

// ---------------------------------------------------------------------------
// Partitions and the exchange schedule (pure host; rl_dist_*_part/_schedule
// expose them so tests can drive the same schedule over gloo on the CPU).
// ---------------------------------------------------------------------------
struct Range {
    uint64_t b, e;
};

Range block(uint64_t n, uint64_t parts, uint64_t part) {
    if (!parts) throw Error(ErrorKind::InvalidCount, "parts must be >= 1");
    if (part >= parts)
        throw Error(ErrorKind::InvalidRange, "part " + std::to_string(part) + " outside [0, " + std::to_string(parts) + ")");
    const uint64_t base = n / parts, extra = n % parts;
    const uint64_t lo = part * base + std::min(part, extra);
    return {lo, lo + base + (part < extra ? 1 : 0)};
}

struct SpmvPart {
    uint64_t r0, r1, cb, ce;  // rows [r0, r1), x window [cb, ce)
};

SpmvPart spmv_part(uint64_t n, uint64_t hb, uint64_t parts, uint64_t part) {
    if (!n) throw Error(ErrorKind::InvalidCount, "spmv: n must be >= 1");
    if (n < parts) throw Error(ErrorKind::InvalidCount, "spmv: fewer rows than parts");
    if (parts > 1 && n / parts < hb)
        throw Error(ErrorKind::ValidationError, "spmv: band half-width " + std::to_string(hb) + " exceeds the " +
                                                    std::to_string(n / parts) +
                                                    " rows of the smallest part (the halo must come from the "
                                                    "neighbours only)");
    const Range r = block(n, parts, part);
    return {r.b, r.e, r.b > hb ? r.b - hb : 0, hb >= n - r.e ? n : r.e + hb};
}

struct SlabPart {
    uint64_t o0, o1, g0, g1;  // owned [o0, o1), buffer [g0, g1) of the outer axis
};

SlabPart slab_part(uint64_t n_outer, uint64_t radius, uint64_t parts, uint64_t part) {
    if (n_outer < parts) throw Error(ErrorKind::InvalidCount, "stencil: fewer layers than parts");
    if (parts > 1 && n_outer / parts < 2 * radius + 1)
        throw Error(ErrorKind::ValidationError, "stencil: a slab is thinner than its halo (" +
                                                    std::to_string(n_outer / parts) + " layers < 2 x radius " +
                                                    std::to_string(radius) + " + 1)");
    const Range o = block(n_outer, parts, part);
    return {o.b, o.e, o.b > radius ? o.b - radius : 0, std::min(n_outer, o.e + radius)};
}

// One boundary between parts b and b+1: transfer A (b's last owned layers ->
// b+1's low halo) and B (b+1's first owned layers -> b's high halo).
struct Boundary {
    uint64_t cnt_a, a_send, a_recv;  // a_send: offset in part b, a_recv: in part b+1
    uint64_t cnt_b, b_send, b_recv;  // b_send: offset in part b+1, b_recv: in part b
};

std::vector<rl_dist_op> halo_schedule(const std::vector<Boundary>& bnd, int world, int parts_local, int rank) {
    if (world < 1 || parts_local < 1) throw Error(ErrorKind::InvalidCount, "world and parts_local must be >= 1");
    if (rank < 0 || rank >= world) throw Error(ErrorKind::InvalidRange, "rank outside [0, world)");
    std::vector<rl_dist_op> ops;
    const auto owner = [&](uint64_t p) { return (int32_t)(p / parts_local); };
    const auto local = [&](uint64_t p) { return (int32_t)(p % parts_local); };
    for (uint64_t b = 0; b < bnd.size(); ++b) {
        const Boundary& x = bnd[b];
        const uint64_t lo = b, hi = b + 1;
        if (x.cnt_a) {
            if (owner(lo) == rank) ops.push_back({0, owner(hi), local(lo), 0, x.a_send, x.cnt_a});
            if (owner(hi) == rank) ops.push_back({1, owner(lo), local(hi), 0, x.a_recv, x.cnt_a});
        }
        if (x.cnt_b) {
            if (owner(hi) == rank) ops.push_back({0, owner(lo), local(hi), 0, x.b_send, x.cnt_b});
            if (owner(lo) == rank) ops.push_back({1, owner(hi), local(lo), 0, x.b_recv, x.cnt_b});
        }
    }
    return ops;
}

std::vector<Boundary> spmv_boundaries(uint64_t n, uint64_t hb, uint64_t parts) {
    std::vector<Boundary> v;
    for (uint64_t b = 0; b + 1 < parts; ++b) {
        const SpmvPart lo = spmv_part(n, hb, parts, b), hi = spmv_part(n, hb, parts, b + 1);
        Boundary x{};
        x.cnt_a = hi.r0 - hi.cb;
        x.a_send = (lo.r1 - x.cnt_a) - lo.cb;
        x.a_recv = 0;
        x.cnt_b = lo.ce - lo.r1;
        x.b_send = hi.r0 - hi.cb;
        x.b_recv = lo.r1 - lo.cb;
        v.push_back(x);
    }
    return v;
}

struct StencilGeom {
    const StencilShape* shape;
    uint64_t dims[3];
    uint64_t n_outer, layer;
};

StencilGeom stencil_geom(const char* preset, const uint64_t* dims) {
    require(preset, "preset");
    require(dims, "dims");
    StencilGeom g{};
    g.shape = &stencil_preset(preset);
    g.dims[0] = dims[0];
    g.dims[1] = dims[1];
    g.dims[2] = g.shape->dimensionality == 3 ? dims[2] : 1;
    const uint64_t need = 2ull * g.shape->radius + 1;
    if (g.dims[0] < need || g.dims[1] < need || (g.shape->dimensionality == 3 && g.dims[2] < need))
        throw Error(ErrorKind::InvalidCount, "stencil: every grid extent must be >= " + std::to_string(need) + " for " +
                                                 g.shape->name);
    g.n_outer = g.shape->dimensionality == 3 ? g.dims[2] : g.dims[1];
    g.layer = g.shape->dimensionality == 3 ? g.dims[0] * g.dims[1] : g.dims[0];
    return g;
}

std::vector<Boundary> stencil_boundaries(const StencilGeom& g, uint64_t parts) {
    const uint64_t r = g.shape->radius;
    std::vector<Boundary> v;
    for (uint64_t b = 0; b + 1 < parts; ++b) {
        const SlabPart lo = slab_part(g.n_outer, r, parts, b), hi = slab_part(g.n_outer, r, parts, b + 1);
        Boundary x{};
        x.cnt_a = (hi.o0 - hi.g0) * g.layer;
        x.a_send = (lo.o1 - lo.g0) * g.layer - x.cnt_a;
        x.a_recv = 0;
        x.cnt_b = (lo.g1 - lo.o1) * g.layer;
        x.b_send = (hi.o0 - hi.g0) * g.layer;
        x.b_recv = (lo.o1 - lo.g0) * g.layer;
        v.push_back(x);
    }
    return v;
}

void copy_ops(const std::vector<rl_dist_op>& v, rl_dist_op* ops, uint64_t cap, uint64_t* count) {
    if (count) *count = v.size();
    if (!ops) return;
    if (cap < v.size())
        throw Error(ErrorKind::InvalidRange, "schedule has " + std::to_string(v.size()) + " transfers, capacity " +
                                                 std::to_string(cap));
    std::copy(v.begin(), v.end(), ops);
}

}  // namespace

// ---------------------------------------------------------------------------
// Communicator
// ---------------------------------------------------------------------------
struct rl_dist_s {
    int world = 1, rank = 0, device = 0, version = 0;
    ncclComm_t comm = nullptr;
    cudaStream_t s_comm = nullptr;  // greatest priority: halo transfers overtake the interior sweep
    void* scratch = nullptr;        // 16 bytes for the scalar all-reduces
    ~rl_dist_s() {
        if (comm) nccl().CommDestroy(comm);
        if (s_comm) cudaStreamDestroy(s_comm);
        if (scratch) cudaFree(scratch);
    }
};

namespace {

rl_dist_s* dist_init(int world, int rank, const uint8_t* id) {
    require(id, "id");
    if (world < 1) throw Error(ErrorKind::InvalidCount, "world must be >= 1");
    if (rank < 0 || rank >= world) throw Error(ErrorKind::InvalidRange, "rank outside [0, world)");
    const NcclApi& api = nccl();
    auto d = std::make_unique<rl_dist_s>();
    d->world = world;
    d->rank = rank;
    ck(cudaGetDevice(&d->device), "cudaGetDevice");
    int lo = 0, hi = 0;
    ck(cudaDeviceGetStreamPriorityRange(&lo, &hi), "stream priorities");
    ck(cudaStreamCreateWithPriority(&d->s_comm, cudaStreamNonBlocking, hi), "stream");
    ck(cudaMalloc(&d->scratch, 16), "scratch");
    ncclUniqueId uid;
    static_assert(sizeof(uid) == RL_DIST_UNIQUE_ID_BYTES, "ncclUniqueId size");
    std::memcpy(&uid, id, sizeof uid);
    nccl_check(api.CommInitRank(&d->comm, world, uid, rank), "ncclCommInitRank");
    nccl_check(api.GetVersion(&d->version), "ncclGetVersion");
    return d.release();
}

template <class T>
void allreduce(rl_dist_s* d, T* value, ncclDataType_t type, ncclRedOp_t op) {
    require(d, "comm");
    require(value, "value");
    ck(cudaMemcpyAsync(d->scratch, value, sizeof(T), cudaMemcpyHostToDevice, d->s_comm), "H2D");
    nccl_check(nccl().AllReduce(d->scratch, d->scratch, 1, type, op, d->comm, d->s_comm), "ncclAllReduce");
    ck(cudaMemcpyAsync(value, d->scratch, sizeof(T), cudaMemcpyDeviceToHost, d->s_comm), "D2H");
    ck(cudaStreamSynchronize(d->s_comm), "sync");
}

// Post `ops` (one rank's schedule) as one NCCL group on the comm stream;
// buffer(part) is the base of that local part's x window / field.
template <class Buf>
void post_exchange(rl_dist_s* d, const std::vector<rl_dist_op>& ops, Buf&& buffer) {
    const NcclApi& api = nccl();
    nccl_check(api.GroupStart(), "ncclGroupStart");
    for (const rl_dist_op& o : ops) {
        double* base = buffer(o.part) + o.offset;
        const ncclResult_t r = o.kind == 0 ? api.Send(base, o.count, ncclFloat64, o.peer, d->comm, d->s_comm)
                                           : api.Recv(base, o.count, ncclFloat64, o.peer, d->comm, d->s_comm);
        if (r != ncclSuccess) {
            api.GroupEnd();
            nccl_check(r, o.kind == 0 ? "ncclSend" : "ncclRecv");
        }
    }
    nccl_check(api.GroupEnd(), "ncclGroupEnd");
}

// A replayable unit of work on the plan's own stream, bridged to the
// caller's stream by events: the first call runs eagerly (it also sets up
// NCCL's peer connections), later calls replay the captured graph.
struct Replay {
    cudaStream_t s = nullptr;
    cudaEvent_t ev_in = nullptr, ev_out = nullptr, ev_start = nullptr, ev_halo = nullptr;
    cudaGraphExec_t exec = nullptr;       // one call (SpMV) / two timesteps (stencil)
    cudaGraphExec_t exec_long = nullptr;  // stencil: kLongSteps timesteps
    uint64_t launches = 0, launches_long = 0;  // library kernels per replay
    bool warmed = false;
    void create() {
        ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
        for (cudaEvent_t* e : {&ev_in, &ev_out, &ev_start, &ev_halo})
            ck(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event");
    }
    void destroy() {
        if (exec) cudaGraphExecDestroy(exec);
        if (exec_long) cudaGraphExecDestroy(exec_long);
        for (cudaEvent_t e : {ev_in, ev_out, ev_start, ev_halo})
            if (e) cudaEventDestroy(e);
        if (s) cudaStreamDestroy(s);
    }
    template <class Body>
    void capture(Body&& body) {
        capture_into(exec, launches, body);
    }
    template <class Body>
    void capture_into(cudaGraphExec_t& out, uint64_t& nlaunch, Body&& body) {
        const uint64_t before = rl_kernel_launches();
        ck(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "graph capture");
        cudaGraph_t g = nullptr;
        try {
            body();
        } catch (...) {
            cudaStreamEndCapture(s, &g);
            if (g) cudaGraphDestroy(g);
            throw;
        }
        ck(cudaStreamEndCapture(s, &g), "graph capture");
        const cudaError_t e = cudaGraphInstantiate(&out, g, 0);
        cudaGraphDestroy(g);
        ck(e, "graph instantiate");
        nlaunch = rl_kernel_launches() - before;
    }
    // The instantiated graph carries its own fork/join between the plan's
    // stream and the comm stream, so a replay is ONE launch into the caller's
    // stream: ordered after the caller's prior work, before its later work.
    void replay(cudaStream_t caller) {
        ck(cudaGraphLaunch(exec, caller), "graph launch");
        rlb::note_launch(launches);
    }
    void replay_long(cudaStream_t caller) {
        ck(cudaGraphLaunch(exec_long, caller), "graph launch");
        rlb::note_launch(launches_long);
    }
    void enter(cudaStream_t caller) {
        ck(cudaEventRecord(ev_in, caller), "event");
        ck(cudaStreamWaitEvent(s, ev_in, 0), "wait");
    }
    void leave(cudaStream_t caller) {
        ck(cudaEventRecord(ev_out, s), "event");
        ck(cudaStreamWaitEvent(caller, ev_out, 0), "wait");
    }
};

bool graphs_on() { return rlb::tuning().dist_graph != 0; }
constexpr int kLongSteps = 10;  // even: a long graph starts and ends in u

}  // namespace

// ---------------------------------------------------------------------------
// SpMV plan
// ---------------------------------------------------------------------------
struct rl_dist_spmv_s {
    rl_dist_s* d = nullptr;
    ExecutionUnit unit = ExecutionUnit::CudaCore;
    struct Part {
        SpmvPart g;
        const int32_t* rp;
        const int32_t* col;
        const double* val;
        double* x;
        double* y;
        uint64_t i0, i1;  // interior local rows [i0, i1): the band stays inside the owned x
        // column-sorted row blocks (K17, spmv_colsort.cu) built from this part's
        // CSR at creation; blocks [kb0, kb1) are interior (rows inside [i0, i1))
        bool colsort = false;
        int krb = 0, krows = 0, kb0 = 0, kb1 = 0, knb = 0, kvec = 1;
        rlb::SpmvKBlock* kblk = nullptr;
        double* kval = nullptr;
        unsigned* kmeta = nullptr;
        rlb::ColsortRun krun{};  // fixed-point mode state (null grid: FP64 atomics)
        rlb::ColsortRun colsort_run() const {
            rlb::ColsortRun r = krun;
            r.rp = rp, r.col = col, r.val = val, r.col_base = (int64_t)g.cb;
            r.fuse = rlb::tuning().spmv_colsort_fuse;
            return r;
        }
    };
    std::vector<Part> parts;
    std::vector<rl_dist_op> ops;
    int long_rows = 0;
    KernelCharacterization kc;
    Replay rp;
    ~rl_dist_spmv_s() {
        rp.destroy();
        for (auto& q : parts)
            for (void* a : {(void*)q.kblk, (void*)q.kval, (void*)q.kmeta, (void*)q.krun.grid, (void*)q.krun.list, (void*)q.krun.count})
                if (a) cudaFree(a);
    }
};

namespace {

// The part's CSR through the column-sorted row-block layout (the single-GPU
// plan's default, K17): copied to the host once, columns made local to the
// part's x window, built, uploaded.  Ineligible matrices keep the CSR.
void colsort_part(rl_dist_spmv_s::Part& q, uint64_t rows, uint64_t nnz, bool tc) {
    std::vector<int32_t> hrp(rows + 1), hcol(nnz);
    std::vector<double> hval(nnz);
    ck(cudaMemcpy(hrp.data(), q.rp, (rows + 1) * 4, cudaMemcpyDeviceToHost), "D2H row_ptr");
    ck(cudaMemcpy(hcol.data(), q.col, nnz * 4, cudaMemcpyDeviceToHost), "D2H col");
    ck(cudaMemcpy(hval.data(), q.val, nnz * 8, cudaMemcpyDeviceToHost), "D2H val");
    for (auto& c : hcol) c -= (int32_t)q.g.cb;
    // the edge rows (whose band reaches the halo) in small blocks, two per SM,
    // so the launch after the exchange spreads over every SM; the interior in
    // the default two waves
    const uint64_t ne = q.i0 + (rows - q.i1), nin = q.i1 - q.i0;
    const uint64_t eb = std::max<uint64_t>(1, 2 * (uint64_t)rlb::kNumSMsHost * q.i0 / std::max<uint64_t>(1, ne));
    std::vector<rlb::ColsortSegment> segs = {{q.i0, eb}, {q.i1, std::max<uint64_t>(1, 4 * (uint64_t)rlb::kNumSMsHost * nin / rows)},
                                             {rows, std::max<uint64_t>(1, 2 * (uint64_t)rlb::kNumSMsHost - eb)}};
    rlb::SpmvColsortLayout L;
    if (!rlb::spmv_colsort_build(rows, q.g.ce - q.g.cb, hrp.data(), hcol.data(), hval.data(), L, segs,
                                 rlb::colsort_classes(tc), tc, rlb::tuning().spmv_colsort_vec))
        return;
    // block order: edge blocks first, then the interior, so each phase is one launch
    std::stable_partition(L.blocks.begin(), L.blocks.end(), [&](const rlb::SpmvKBlock& k) {
        return !(k.row0 >= q.i0 && k.row0 + k.rows <= q.i1);
    });
    auto up = [&](auto*& dst, const auto& v) {
        using T = std::remove_reference_t<decltype(*dst)>;
        ck(cudaMalloc(&dst, std::max<size_t>(v.size(), 1) * sizeof(T)), "alloc");
        if (!v.empty()) ck(cudaMemcpy(dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "upload");
    };
    up(q.kblk, L.blocks);
    up(q.kval, L.val);
    up(q.kmeta, L.meta);
    q.colsort = true;
    q.krb = L.rb;
    q.kvec = L.vec;
    q.krows = L.rows;
    if (rlb::colsort_fixed_for(tc)) {
        std::vector<int> g;
        for (const auto& k : L.blocks) g.push_back(rlb::colsort_initial_grid(k));
        up(q.krun.grid, g);
        ck(cudaMalloc(&q.krun.list, std::max<uint64_t>(rows, 1) * sizeof(int)), "alloc");
        ck(cudaMalloc(&q.krun.count, 2 * sizeof(unsigned)), "alloc");
        ck(cudaMemset(q.krun.count, 0, 2 * sizeof(unsigned)), "alloc");
        q.krun.done = q.krun.count + 1;
        q.krun.rows = (unsigned)rows;
    }
    q.knb = (int)L.blocks.size();
    q.kb1 = q.knb;  // interior blocks [kb0, knb), edge blocks [0, kb0)
    q.kb0 = 0;
    while (q.kb0 < q.knb && !(L.blocks[q.kb0].row0 >= q.i0 && L.blocks[q.kb0].row0 + L.blocks[q.kb0].rows <= q.i1))
        ++q.kb0;
}

void part_rows(const rl_dist_spmv_s* pl, const rl_dist_spmv_s::Part& q, int b0, int b1, uint64_t r0, uint64_t r1,
               cudaStream_t s) {
    if (q.colsort) {
        ck(rlb::launch_spmv_colsort(pl->unit == ExecutionUnit::TensorCore, q.kvec, q.kblk, b0, b1, q.krb, q.krows, q.kval,
                                    q.kmeta, q.x, q.y, q.colsort_run(), s),
           "spmv (column-sorted part)");
        return;
    }
    spmv_csr_rows(pl->unit, Precision::FP64, r0, r1, q.rp, q.col, q.val, q.x, (int64_t)q.g.cb, q.y, s, pl->long_rows);
}

rl_dist_spmv_s* spmv_create(rl_dist_s* d, ExecutionUnit unit, Precision p, uint64_t n, uint64_t hb, int L,
                            const int32_t* const* rp, const int32_t* const* col, const double* const* val,
                            double* const* x, double* const* y) {
    require(d, "comm");
    if (p != Precision::FP64) throw Error(ErrorKind::ValidationError, "the B200 kernels are FP64 only");
    if (L < 1) throw Error(ErrorKind::InvalidCount, "parts_local must be >= 1");
    for (const void* a : {(const void*)rp, (const void*)col, (const void*)val, (const void*)x, (const void*)y})
        require(a, "per-part pointer array");
    if (n > 0x7fffffffull) throw Error(ErrorKind::InvalidRange, "int32 CSR indices cannot address this matrix");
    const uint64_t P = (uint64_t)d->world * (uint64_t)L;
    auto pl = std::make_unique<rl_dist_spmv_s>();
    pl->d = d;
    pl->unit = unit;
    pl->rp.create();
    unsigned long long* chk = nullptr;
    ck(cudaMalloc(&chk, 3 * sizeof(unsigned long long)), "alloc");
    uint64_t nnz_local = 0;
    try {
        for (int i = 0; i < L; ++i) {
            rl_dist_spmv_s::Part q{};
            q.g = spmv_part(n, hb, P, (uint64_t)d->rank * L + i);
            require(rp[i], "row_ptr[i]");
            require(col[i], "col[i]");
            require(val[i], "val[i]");
            require(x[i], "x[i]");
            require(y[i], "y[i]");
            q.rp = rp[i];
            q.col = col[i];
            q.val = val[i];
            q.x = x[i];
            q.y = y[i];
            const uint64_t rows = q.g.r1 - q.g.r0;
            q.i0 = q.g.cb < q.g.r0 ? std::min(rows, hb) : 0;
            q.i1 = q.g.ce > q.g.r1 ? std::max(q.i0, rows > hb ? rows - hb : 0) : rows;
            // the CSR must stay inside the band (else the x window is too small)
            int32_t ends[2];
            ck(cudaMemcpy(&ends[0], q.rp, 4, cudaMemcpyDeviceToHost), "row_ptr read");
            ck(cudaMemcpy(&ends[1], q.rp + rows, 4, cudaMemcpyDeviceToHost), "row_ptr read");
            if (ends[0] != 0) throw Error(ErrorKind::ValidationError, "row_ptr[i][0] must be 0");
            if (ends[1] < 0) throw Error(ErrorKind::ValidationError, "row_ptr[i][rows] is negative");
            ck(rlb::launch_band_check(rows, q.rp, q.col, (int64_t)q.g.r0, (int64_t)n, chk, pl->rp.s), "band check");
            unsigned long long h[3];
            ck(cudaMemcpyAsync(h, chk, sizeof h, cudaMemcpyDeviceToHost, pl->rp.s), "D2H");
            ck(cudaStreamSynchronize(pl->rp.s), "sync");
            if (h[2]) throw Error(ErrorKind::ValidationError, "row_ptr[i] decreases");
            if (h[1])
                throw Error(ErrorKind::IndexOutOfRange, std::to_string(h[1]) + " column indices outside [0, " +
                                                            std::to_string(n) + ")");
            if (h[0] > hb)
                throw Error(ErrorKind::ValidationError, "a column lies " + std::to_string(h[0]) +
                                                            " from its row, outside the half-bandwidth " +
                                                            std::to_string(hb));
            nnz_local += (uint64_t)ends[1];
            pl->parts.push_back(q);
            if (rlb::tuning().spmv_plan_colsort && ends[1] > 0)
                colsort_part(pl->parts.back(), rows, (uint64_t)ends[1], unit == ExecutionUnit::TensorCore);
            if (!pl->parts.back().colsort && rlb::tuning().spmv_long_rows &&
                rlb::spmv_long_rows_probe(q.rp, q.col, q.val, 0, rows, pl->rp.s) != 0)
                pl->long_rows = 1;
        }
    } catch (...) {
        cudaFree(chk);
        throw;
    }
    cudaFree(chk);
    uint64_t nnz = nnz_local;
    allreduce(d, &nnz, ncclUint64, ncclSum);
    pl->kc = spmv_csr_model({n, n, nnz}, kDefaultIndexBytes, p);
    pl->ops = halo_schedule(spmv_boundaries(n, hb, P), d->world, L, d->rank);
    if (pl->long_rows) {  // reserved now: replays run under graph capture
        uint64_t mx = 0;
        for (const auto& q : pl->parts) mx = std::max(mx, q.g.r1 - q.g.r0);
        rlb::LongRows lr{};
        ck(rlb::spmv_long_workspace(pl->rp.s, mx, lr), "long-row workspace");
    }
    return pl.release();
}

void spmv_body(rl_dist_spmv_s* pl) {
    rl_dist_s* d = pl->d;
    Replay& r = pl->rp;
    const bool xchg = !pl->ops.empty();
    if (xchg) {
        ck(cudaEventRecord(r.ev_start, r.s), "event");
        ck(cudaStreamWaitEvent(d->s_comm, r.ev_start, 0), "wait");
        post_exchange(d, pl->ops, [&](int i) { return pl->parts[i].x; });
        ck(cudaEventRecord(r.ev_halo, d->s_comm), "event");
    }
    for (const auto& q : pl->parts) part_rows(pl, q, q.kb0, q.kb1, q.i0, q.i1, r.s);
    if (xchg) ck(cudaStreamWaitEvent(r.s, r.ev_halo, 0), "wait");
    for (const auto& q : pl->parts) {
        const uint64_t rows = q.g.r1 - q.g.r0;
        if (q.colsort) {
            part_rows(pl, q, 0, q.kb0, 0, 0, r.s);  // every edge block, one launch
        } else {
            part_rows(pl, q, 0, 0, 0, q.i0, r.s);
            part_rows(pl, q, 0, 0, q.i1, rows, r.s);
        }
    }
}

void spmv_execute(rl_dist_spmv_s* pl, cudaStream_t caller) {
    require(pl, "plan");
    Replay& r = pl->rp;
    if (!r.exec && r.warmed && graphs_on()) r.capture([&] { spmv_body(pl); });
    if (r.exec) {
        r.replay(caller);
        return;
    }
    r.enter(caller);
    spmv_body(pl);
    r.warmed = true;
    r.leave(caller);
}

}  // namespace

// ---------------------------------------------------------------------------
// Stencil plan
// ---------------------------------------------------------------------------
struct rl_dist_stencil_s {
    rl_dist_s* d = nullptr;
    ExecutionUnit unit = ExecutionUnit::CudaCore;
    const StencilShape* shape = nullptr;
    std::vector<double> weights;
    struct Part {
        SlabPart g;
        uint64_t dims[3];  // local buffer extents
        double* u;
        double* v;
        uint64_t a, b, i0, i1;  // local owned [a, b), interior [i0, i1)
    };
    std::vector<Part> parts;
    std::vector<rl_dist_op> ops;
    KernelCharacterization per_step;
    Replay rp;  // the graph holds two timesteps: u -> v -> u
    ~rl_dist_stencil_s() { rp.destroy(); }
};

namespace {

rl_dist_stencil_s* stencil_create(rl_dist_s* d, ExecutionUnit unit, Precision p, const char* preset,
                                  const uint64_t* dims, const double* weights, int L, double* const* u,
                                  double* const* v) {
    require(d, "comm");
    if (p != Precision::FP64) throw Error(ErrorKind::ValidationError, "the B200 kernels are FP64 only");
    if (L < 1) throw Error(ErrorKind::InvalidCount, "parts_local must be >= 1");
    require(u, "u");
    require(v, "v");
    const StencilGeom g = stencil_geom(preset, dims);
    const uint64_t P = (uint64_t)d->world * (uint64_t)L;
    const uint64_t r = g.shape->radius;
    auto pl = std::make_unique<rl_dist_stencil_s>();
    pl->d = d;
    pl->unit = unit;
    pl->shape = g.shape;
    if (weights) pl->weights.assign(weights, weights + g.shape->point_count);
    for (int i = 0; i < L; ++i) {
        rl_dist_stencil_s::Part q{};
        q.g = slab_part(g.n_outer, r, P, (uint64_t)d->rank * L + i);
        require(u[i], "u[i]");
        require(v[i], "v[i]");
        if (u[i] == v[i]) throw Error(ErrorKind::ValidationError, "u and v must be distinct buffers");
        q.u = u[i];
        q.v = v[i];
        q.dims[0] = g.dims[0];
        q.dims[1] = g.shape->dimensionality == 3 ? g.dims[1] : q.g.g1 - q.g.g0;
        q.dims[2] = g.shape->dimensionality == 3 ? q.g.g1 - q.g.g0 : 1;
        q.a = q.g.o0 - q.g.g0;
        q.b = q.g.o1 - q.g.g0;
        const bool lo_nbr = q.g.g0 < q.g.o0, hi_nbr = q.g.g1 > q.g.o1;
        q.i0 = std::min(q.b, q.a + (lo_nbr ? r : 0));
        q.i1 = std::max(q.i0, hi_nbr ? (q.b > r ? q.b - r : 0) : q.b);
        pl->parts.push_back(q);
    }
    // per timestep: the model per point x the global interior points
    const KernelCharacterization per_point = stencil_model(*g.shape, p, 1);
    unsigned __int128 pts = 1;
    for (int k = 0; k < g.shape->dimensionality; ++k) pts *= g.dims[k] - 2 * r;
    const unsigned __int128 w = pts * per_point.work_flops, q = pts * per_point.traffic_bytes;
    if ((w >> 64) || (q >> 64)) throw Error(ErrorKind::InvalidRange, "stencil accounting overflows 64-bit count");
    pl->per_step = {g.shape->name, (uint64_t)w, (uint64_t)q};
    pl->ops = halo_schedule(stencil_boundaries(g, P), d->world, L, d->rank);
    pl->rp.create();
    return pl.release();
}

void stencil_step(rl_dist_stencil_s* pl, bool from_u) {
    rl_dist_s* d = pl->d;
    Replay& r = pl->rp;
    const double* w = pl->weights.empty() ? nullptr : pl->weights.data();
    const bool xchg = !pl->ops.empty();
    if (xchg) {
        ck(cudaEventRecord(r.ev_start, r.s), "event");
        ck(cudaStreamWaitEvent(d->s_comm, r.ev_start, 0), "wait");
        post_exchange(d, pl->ops, [&](int i) { return from_u ? pl->parts[i].u : pl->parts[i].v; });
        ck(cudaEventRecord(r.ev_halo, d->s_comm), "event");
    }
    for (const auto& q : pl->parts)
        if (q.i1 > q.i0)
            stencil_sweep(pl->unit, Precision::FP64, *pl->shape, q.dims, w, q.i0, q.i1, from_u ? q.u : q.v,
                          from_u ? q.v : q.u, r.s);
    if (xchg) ck(cudaStreamWaitEvent(r.s, r.ev_halo, 0), "wait");
    for (const auto& q : pl->parts) {
        const double* src = from_u ? q.u : q.v;
        double* dst = from_u ? q.v : q.u;
        if (q.i0 > q.a) stencil_sweep(pl->unit, Precision::FP64, *pl->shape, q.dims, w, q.a, q.i0, src, dst, r.s);
        if (q.b > q.i1) stencil_sweep(pl->unit, Precision::FP64, *pl->shape, q.dims, w, q.i1, q.b, src, dst, r.s);
    }
}

KernelCharacterization stencil_run(rl_dist_stencil_s* pl, uint64_t steps, cudaStream_t caller, int* result_in_v) {
    require(pl, "plan");
    if (!steps) throw Error(ErrorKind::InvalidCount, "stencil: steps must be >= 1");
    const unsigned __int128 w = (unsigned __int128)pl->per_step.work_flops * steps;
    const unsigned __int128 q = (unsigned __int128)pl->per_step.traffic_bytes * steps;
    if ((w >> 64) || (q >> 64)) throw Error(ErrorKind::InvalidRange, "stencil accounting overflows 64-bit count");
    Replay& r = pl->rp;
    uint64_t t = 0;
    if (!r.exec && r.warmed && graphs_on() && steps >= 2)
        r.capture([&] {
            stencil_step(pl, true);
            stencil_step(pl, false);
        });
    // long runs: kLongSteps timesteps per graph launch (host cost per
    // timestep ~ one graph launch / kLongSteps)
    if (r.exec && !r.exec_long && steps >= kLongSteps)
        r.capture_into(r.exec_long, r.launches_long, [&] {
            for (int i = 0; i < kLongSteps; ++i) stencil_step(pl, (i & 1) == 0);
        });
    if (r.exec_long)
        for (; t + kLongSteps <= steps; t += kLongSteps) r.replay_long(caller);
    if (r.exec)
        for (; t + 2 <= steps; t += 2) r.replay(caller);
    if (t < steps) {  // eager: the first call, or the odd last timestep
        r.enter(caller);
        for (; t < steps; ++t) stencil_step(pl, (t & 1) == 0);
        r.leave(caller);
    }
    r.warmed = true;
    if (result_in_v) *result_in_v = (int)(steps & 1);
    return {pl->per_step.kernel_name, (uint64_t)w, (uint64_t)q};
}

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

}  // namespace

// ===========================================================================
// extern "C"
// ===========================================================================
extern "C" {

int rl_dist_unique_id(uint8_t* id) {
    return guarded([&] {
        require(id, "id");
        ncclUniqueId uid;
        nccl_check(nccl().GetUniqueId(&uid), "ncclGetUniqueId");
        std::memcpy(id, &uid, sizeof uid);
    });
}
int rl_dist_init(int world, int rank, const uint8_t* id, rl_dist* out) {
    return guarded([&] {
        require(out, "out");
        *out = nullptr;
        *out = dist_init(world, rank, id);
    });
}
int rl_dist_destroy(rl_dist d) {
    return guarded([&] { delete d; });
}
int rl_dist_info(rl_dist d, int* world, int* rank, int* device, int* version) {
    return guarded([&] {
        require(d, "comm");
        if (world) *world = d->world;
        if (rank) *rank = d->rank;
        if (device) *device = d->device;
        if (version) *version = d->version;
    });
}
int rl_dist_allreduce_u64(rl_dist d, uint64_t* v) {
    return guarded([&] { allreduce(d, v, ncclUint64, ncclSum); });
}
int rl_dist_allreduce_max(rl_dist d, double* v) {
    return guarded([&] { allreduce(d, v, ncclFloat64, ncclMax); });
}

int rl_dist_block(uint64_t n, uint64_t parts, uint64_t part, uint64_t* begin, uint64_t* end) {
    return guarded([&] {
        const Range r = block(n, parts, part);
        if (begin) *begin = r.b;
        if (end) *end = r.e;
    });
}
int rl_dist_spmv_part(uint64_t n, uint64_t hb, uint64_t parts, uint64_t part, uint64_t* r0, uint64_t* r1,
                      uint64_t* cb, uint64_t* ce) {
    return guarded([&] {
        const SpmvPart q = spmv_part(n, hb, parts, part);
        if (r0) *r0 = q.r0;
        if (r1) *r1 = q.r1;
        if (cb) *cb = q.cb;
        if (ce) *ce = q.ce;
    });
}
int rl_dist_stencil_part(const char* preset, const uint64_t* dims, uint64_t parts, uint64_t part, uint64_t* o0,
                         uint64_t* o1, uint64_t* g0, uint64_t* g1) {
    return guarded([&] {
        const StencilGeom g = stencil_geom(preset, dims);
        const SlabPart q = slab_part(g.n_outer, g.shape->radius, parts, part);
        if (o0) *o0 = q.o0;
        if (o1) *o1 = q.o1;
        if (g0) *g0 = q.g0;
        if (g1) *g1 = q.g1;
    });
}
int rl_dist_spmv_schedule(uint64_t n, uint64_t hb, int world, int L, int rank, rl_dist_op* ops, uint64_t cap,
                          uint64_t* count) {
    return guarded([&] {
        if (world < 1 || L < 1) throw Error(ErrorKind::InvalidCount, "world and parts_local must be >= 1");
        copy_ops(halo_schedule(spmv_boundaries(n, hb, (uint64_t)world * L), world, L, rank), ops, cap, count);
    });
}
int rl_dist_stencil_schedule(const char* preset, const uint64_t* dims, int world, int L, int rank, rl_dist_op* ops,
                             uint64_t cap, uint64_t* count) {
    return guarded([&] {
        if (world < 1 || L < 1) throw Error(ErrorKind::InvalidCount, "world and parts_local must be >= 1");
        copy_ops(halo_schedule(stencil_boundaries(stencil_geom(preset, dims), (uint64_t)world * L), world, L, rank),
                 ops, cap, count);
    });
}

int rl_dist_scale(rl_dist d, rl_unit u, rl_precision p, double* a, const double* b, double q, uint64_t n_global,
                  rl_stream s, rl_kchar* out) {
    return guarded([&] {
        require(d, "comm");
        const KernelCharacterization k = scale_model(n_global, prec_of(p));
        const Range c = block(n_global, (uint64_t)d->world, (uint64_t)d->rank);
        if (c.e > c.b) scale(unit_of(u), prec_of(p), a, b, q, c.e - c.b, s);
        put(out, k);
    });
}

int rl_dist_spmv_create(rl_dist d, rl_unit u, rl_precision p, uint64_t n, uint64_t hb, int L,
                        const int32_t* const* rp, const int32_t* const* col, const double* const* val,
                        double* const* x, double* const* y, rl_dist_spmv* out) {
    return guarded([&] {
        require(out, "out");
        *out = nullptr;
        *out = spmv_create(d, unit_of(u), prec_of(p), n, hb, L, rp, col, val, x, y);
    });
}
int rl_dist_spmv_execute(rl_dist_spmv pl, rl_stream s, rl_kchar* out) {
    return guarded([&] {
        spmv_execute(pl, static_cast<cudaStream_t>(s));
        put(out, pl->kc);
    });
}
int rl_dist_spmv_destroy(rl_dist_spmv pl) {
    return guarded([&] { delete pl; });
}

int rl_dist_stencil_create(rl_dist d, rl_unit u, rl_precision p, const char* preset, const uint64_t* dims,
                           const double* weights, int L, double* const* uu, double* const* v, rl_dist_stencil* out) {
    return guarded([&] {
        require(out, "out");
        *out = nullptr;
        *out = stencil_create(d, unit_of(u), prec_of(p), preset, dims, weights, L, uu, v);
    });
}
int rl_dist_stencil_run(rl_dist_stencil pl, uint64_t steps, rl_stream s, int* result_in_v, rl_kchar* out) {
    return guarded([&] { put(out, stencil_run(pl, steps, static_cast<cudaStream_t>(s), result_in_v)); });
}
int rl_dist_stencil_destroy(rl_dist_stencil pl) {
    return guarded([&] { delete pl; });
}

}  // extern "C"
