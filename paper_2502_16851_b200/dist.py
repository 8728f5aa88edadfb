"""Multi-GPU decomposition of the three kernels (one process per GPU).

The sharded path lives in the C-ABI (csrc/dist.cpp, ``rl_dist_*``): NCCL
point-to-point on a high-priority stream carries the halos, the library's
sm_100a kernels do the per-part compute, and steady-state calls replay CUDA
graphs.  This module is its Python face:

* ``Comm``       an NCCL communicator (``rl_dist_init``); ``Comm.from_env()``
                 shares the unique id over torch.distributed (rank 0 creates it).
* ``dist_scale`` STREAM Scale on this rank's contiguous chunk, no communication.
* ``DistSpmv``   row-partitioned CSR SpMV; per call the x band halo (hb doubles
                 per side) is exchanged while the interior rows run.
* ``DistStencil`` slab-decomposed Jacobi; per timestep the ghost layers are
                 exchanged while the slab interior is swept.

A job has P = world * parts_local parts; production runs one part per GPU.
The partition and exchange schedule are pure host functions of the library
(``spmv_part``, ``stencil_part``, ``spmv_schedule``, ``stencil_schedule``); the
CPU tests run that same schedule over gloo (``run_schedule``) with the oracle
as the per-part compute, and the GPU tests run several parts on one device
through NCCL self send/recv.

Reference: the paper's kernels have no multi-GPU form (reference SPEC.md:101
lists multi-GPU aggregation as a non-goal); SURVEY.md §2.4 / §8(e) define
this decomposition.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import List, Optional, Sequence

from . import (CUDA_CORE, FP64, _check, _dev_ptr, _kc, _KChar, _stream, _u64, _weights, lib,
               stencil_preset)

UNIQUE_ID_BYTES = 128


class _Op(C.Structure):
    _fields_ = [("kind", C.c_int32), ("peer", C.c_int32), ("part", C.c_int32), ("reserved", C.c_int32),
                ("offset", C.c_uint64), ("count", C.c_uint64)]


@dataclass(frozen=True)
class HaloOp:
    """One transfer of a rank's exchange, in posting order: kind 'send' or
    'recv', peer rank, local part index, offset / count in doubles of that
    part's x window or field buffer."""

    kind: str
    peer: int
    part: int
    offset: int
    count: int


# ---------------------------------------------------------------------------
# partitions (rl_dist_block / rl_dist_spmv_part / rl_dist_stencil_part)
# ---------------------------------------------------------------------------
def block_range(n: int, parts: int, part: int):
    """Contiguous block [lo, hi) of n items (sizes differ by <= 1)."""
    lo, hi = _u64(), _u64()
    _check(lib().rl_dist_block(n, parts, part, C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


def scale_chunk(n_global: int, world: int, rank: int):
    return block_range(n_global, world, rank)


@dataclass
class SpmvPartition:
    """Rows [r0, r1) of an n-row matrix with half-bandwidth hb, and its x
    window x_win[i] = x[i + col_base] for global columns [col_base, col_end)."""

    n: int
    hb: int
    parts: int
    part: int

    def __post_init__(self):
        v = [_u64() for _ in range(4)]
        _check(lib().rl_dist_spmv_part(self.n, self.hb, self.parts, self.part, *[C.byref(x) for x in v]))
        self.r0, self.r1, self.col_base, self.col_end = (x.value for x in v)
        self.lo_halo = self.r0 - self.col_base
        self.hi_halo = self.col_end - self.r1

    @property
    def rows(self) -> int:
        return self.r1 - self.r0

    @property
    def window(self) -> int:
        return self.col_end - self.col_base

    def own_slice(self):
        return slice(self.lo_halo, self.lo_halo + self.rows)

    def interior_rows(self):
        """Local rows whose band lies inside the owned x (no halo needed)."""
        lo = min(self.rows, self.hb) if self.lo_halo else 0
        hi = max(lo, self.rows - self.hb) if self.hi_halo else self.rows
        return lo, hi


def _dims_of(preset: str, shape: Sequence[int]):
    """numpy-order global shape -> the C dims {nx, ny, nz}."""
    if stencil_preset(preset)[0] == 2:
        ny, nx = shape
        return (_u64 * 3)(nx, ny, 1)
    nz, ny, nx = shape
    return (_u64 * 3)(nx, ny, nz)


@dataclass
class SlabPartition:
    """Slab of the outer axis (rows in 2D, planes in 3D) of a global grid of
    numpy shape `shape`: owned [o0, o1), buffer [g_lo, g_hi) with `radius`
    ghost layers per side where a neighbour exists."""

    preset: str
    shape: tuple
    parts: int
    part: int

    def __post_init__(self):
        v = [_u64() for _ in range(4)]
        _check(lib().rl_dist_stencil_part(self.preset.encode(), _dims_of(self.preset, self.shape), self.parts,
                                          self.part, *[C.byref(x) for x in v]))
        self.o0, self.o1, self.g_lo, self.g_hi = (x.value for x in v)
        self.radius = stencil_preset(self.preset)[2]

    @property
    def local_outer(self) -> int:
        return self.g_hi - self.g_lo

    @property
    def local_shape(self) -> tuple:
        return (self.local_outer,) + tuple(self.shape[1:])

    def own_local(self):
        return self.o0 - self.g_lo, self.o1 - self.g_lo


# ---------------------------------------------------------------------------
# the exchange schedule (rl_dist_spmv_schedule / rl_dist_stencil_schedule)
# ---------------------------------------------------------------------------
def _ops(fn, *args) -> List[HaloOp]:
    n = _u64()
    _check(fn(*args, None, 0, C.byref(n)))
    arr = (_Op * max(1, n.value))()
    _check(fn(*args, C.cast(arr, C.c_void_p), n.value, C.byref(n)))
    return [HaloOp("send" if o.kind == 0 else "recv", o.peer, o.part, o.offset, o.count) for o in arr[:n.value]]


def spmv_schedule(n: int, hb: int, world: int, parts_local: int, rank: int) -> List[HaloOp]:
    return _ops(lib().rl_dist_spmv_schedule, n, hb, world, parts_local, rank)


def stencil_schedule(preset: str, shape: Sequence[int], world: int, parts_local: int, rank: int) -> List[HaloOp]:
    return _ops(lib().rl_dist_stencil_schedule, preset.encode(), _dims_of(preset, shape), world, parts_local, rank)


def run_schedule(ops: Sequence[HaloOp], buffers: Sequence, rank: int) -> None:
    """Carry out one rank's schedule over torch.distributed (gloo, CPU
    tensors): what the NCCL group of rl_dist_* does on GPUs.  buffers[part] is
    a flat view of that local part's x window / field.  Transfers with a peer
    rank are posted in schedule order (gloo, like NCCL, matches the sends and
    receives of one peer pair in order); transfers to this same rank are
    matched in order and copied (NCCL's self send/recv)."""
    import torch.distributed as dist

    reqs = []
    self_sends = []
    for o in ops:
        if o.peer == rank:
            if o.kind == "send":
                self_sends.append(buffers[o.part][o.offset:o.offset + o.count].clone())
            continue
        view = buffers[o.part][o.offset:o.offset + o.count]
        reqs.append(dist.isend(view, o.peer) if o.kind == "send" else dist.irecv(view, o.peer))
    k = 0
    for o in ops:
        if o.peer == rank and o.kind == "recv":
            buffers[o.part][o.offset:o.offset + o.count].copy_(self_sends[k])
            k += 1
    for r in reqs:
        r.wait()


# ---------------------------------------------------------------------------
# GPU path (rl_dist_*)
# ---------------------------------------------------------------------------
def unique_id() -> bytes:
    buf = (C.c_uint8 * UNIQUE_ID_BYTES)()
    _check(lib().rl_dist_unique_id(C.cast(buf, C.c_void_p)))
    return bytes(buf)


class Comm:
    """NCCL communicator of the library (rl_dist_init on the current device)."""

    def __init__(self, world: int, rank: int, uid: bytes):
        buf = (C.c_uint8 * UNIQUE_ID_BYTES).from_buffer_copy(uid)
        h = C.c_void_p()
        _check(lib().rl_dist_init(world, rank, C.cast(buf, C.c_void_p), C.byref(h)))
        self.h = h
        self.world, self.rank = world, rank

    @classmethod
    def single(cls) -> "Comm":
        """A world-1 communicator (one process, one GPU)."""
        return cls(1, 0, unique_id())

    @classmethod
    def from_env(cls) -> "Comm":
        """World/rank from the torchrun environment; rank 0's unique id is
        broadcast over the initialised torch.distributed group."""
        import torch.distributed as dist

        world = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        if world == 1:
            return cls.single()
        obj = [unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return cls(world, rank, obj[0])

    def info(self):
        w, r, d, v = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        _check(lib().rl_dist_info(self.h, C.byref(w), C.byref(r), C.byref(d), C.byref(v)))
        return {"world": w.value, "rank": r.value, "device": d.value, "nccl_version": v.value}

    def allreduce_max(self, value: float) -> float:
        v = C.c_double(value)
        _check(lib().rl_dist_allreduce_max(self.h, C.byref(v)))
        return v.value

    def allreduce_sum(self, value: int) -> int:
        v = _u64(value)
        _check(lib().rl_dist_allreduce_u64(self.h, C.byref(v)))
        return v.value

    def close(self):
        if self.h:
            _check(lib().rl_dist_destroy(self.h))
            self.h = None


def dist_scale(comm: Comm, a, b, q: float, n_global: int, unit: int = CUDA_CORE, stream=None,
               precision: int = FP64):
    """a = q*b on this rank's chunk scale_chunk(n_global, world, rank)."""
    k = _KChar()
    _check(lib().rl_dist_scale(comm.h, unit, precision, _dev_ptr(a, "f64", "a"), _dev_ptr(b, "f64", "b"),
                               float(q), n_global, _stream(stream), C.byref(k)))
    return _kc(k)


def _ptrs(ts, dtype, what):
    return (C.c_void_p * len(ts))(*[_dev_ptr(t, dtype, what) for t in ts])


class DistSpmv:
    """rl_dist_spmv: parts[i] = (row_ptr, col, val, x_window, y) device tensors
    of local part i (columns global; the owned x at own_slice())."""

    def __init__(self, comm: Comm, n: int, hb: int, parts, unit: int = CUDA_CORE, precision: int = FP64):
        self._keep = parts
        cols = list(zip(*parts))
        h = C.c_void_p()
        _check(lib().rl_dist_spmv_create(comm.h, unit, precision, n, hb, len(parts),
                                         _ptrs(cols[0], "i32", "row_ptr"), _ptrs(cols[1], "i32", "col"),
                                         _ptrs(cols[2], "f64", "val"), _ptrs(cols[3], "f64", "x"),
                                         _ptrs(cols[4], "f64", "y"), C.byref(h)))
        self.h = h

    def execute(self, stream=None):
        k = _KChar()
        _check(lib().rl_dist_spmv_execute(self.h, _stream(stream), C.byref(k)))
        return _kc(k)

    def close(self):
        if self.h:
            _check(lib().rl_dist_spmv_destroy(self.h))
            self.h = None


class DistStencil:
    """rl_dist_stencil: us[i] / vs[i] = local part i's buffers (SlabPartition
    local_shape), global numpy shape `shape`."""

    def __init__(self, comm: Comm, preset: str, shape, us, vs, weights=None, unit: int = CUDA_CORE,
                 precision: int = FP64):
        self._keep = (list(us), list(vs))
        w = _weights(preset, weights)
        self._w = w
        h = C.c_void_p()
        _check(lib().rl_dist_stencil_create(comm.h, unit, precision, preset.encode(), _dims_of(preset, shape),
                                            C.cast(w, C.c_void_p) if w is not None else None, len(us),
                                            _ptrs(us, "f64", "u"), _ptrs(vs, "f64", "v"), C.byref(h)))
        self.h = h

    def run(self, steps: int, stream=None):
        """Returns (KernelCharacterization, result_in_v)."""
        k, inv = _KChar(), C.c_int()
        _check(lib().rl_dist_stencil_run(self.h, steps, _stream(stream), C.byref(inv), C.byref(k)))
        return _kc(k), bool(inv.value)

    def close(self):
        if self.h:
            _check(lib().rl_dist_stencil_destroy(self.h))
            self.h = None


def init_process_group(backend: Optional[str] = None) -> tuple:
    """Rank/world from the torchrun environment (MASTER_ADDR should be 127.0.0.1)."""
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1 and not dist.is_initialized():
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        dist.init_process_group(backend=backend)
    return rank, world
