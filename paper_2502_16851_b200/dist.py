"""Multi-GPU decomposition of the three kernels (one process per GPU).

torch.distributed (NCCL over NVLink/NVSwitch on the GPU box, gloo in the CPU
tests) carries the exchanges; the arithmetic is always the sm_100a C-ABI
kernels, injected as callables so the host logic (partitions, halo indices,
exchange order, interior/edge overlap) is testable on CPU with the oracle in
their place.

* STREAM Scale   contiguous n/P chunks, no communication.
* CSR SpMV       contiguous row blocks, x partitioned identically; each step
                 exchanges the band halo of x (hb doubles per side) with the
                 two neighbours (grouped isend/irecv), runs the interior rows
                 (those whose band stays inside the owned x) while the halo is
                 in flight, then the two edge row blocks.
* Stencils       slabs along the slowest axis (rows in 2D, planes in 3D) with
                 one ghost row/plane per side; per step the ghosts are
                 exchanged while the slab interior is swept, then the two edge
                 rows/planes are swept and the buffers swap.

Reference: the paper's kernels have no multi-GPU form (reference SPEC.md:101
lists multi-GPU aggregation as a non-goal); SURVEY.md §2.4 / §8(e) define
this decomposition.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import torch
import torch.distributed as dist


def block_range(n: int, world: int, rank: int):
    """Contiguous block [lo, hi) of n items for `rank` (sizes differ by <= 1)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


# ---------------------------------------------------------------------------
# STREAM
# ---------------------------------------------------------------------------
def scale_chunk(n_global: int, world: int, rank: int):
    return block_range(n_global, world, rank)


# ---------------------------------------------------------------------------
# SpMV x-halo exchange
# ---------------------------------------------------------------------------
@dataclass
class SpmvPartition:
    """Row block [r0, r1) of an n-row banded matrix (half-bandwidth hb) and the
    layout of the local x window: x_win[i] = x[i + col_base] for global
    columns [col_base, col_base + len)."""

    n: int
    hb: int
    world: int
    rank: int

    def __post_init__(self):
        self.r0, self.r1 = block_range(self.n, self.world, self.rank)
        self.col_base = max(0, self.r0 - self.hb)
        self.col_end = min(self.n, self.r1 + self.hb)
        self.lo_halo = self.r0 - self.col_base      # doubles received from rank-1
        self.hi_halo = self.col_end - self.r1       # doubles received from rank+1
        if self.world > 1 and (self.r1 - self.r0) < self.hb:
            raise ValueError("band half-width exceeds the rows per rank: neighbour-only "
                             "halo exchange needs rows_per_rank >= hb")

    @property
    def rows(self) -> int:
        return self.r1 - self.r0

    @property
    def window(self) -> int:
        return self.col_end - self.col_base

    def interior_rows(self):
        """Local rows whose band lies inside the owned x: no halo needed."""
        lo = self.hb if self.rank > 0 else 0
        hi = self.rows - (self.hb if self.rank < self.world - 1 else 0)
        return (lo, max(lo, hi))

    def own_slice(self):
        return slice(self.lo_halo, self.lo_halo + self.rows)


def spmv_halo_ops(part: SpmvPartition, x_win: torch.Tensor):
    """P2P ops that fill x_win's halos from the neighbours' owned x."""
    ops = []
    own = x_win[part.own_slice()]
    if part.rank > 0:
        ops.append(dist.P2POp(dist.irecv, x_win[: part.lo_halo], part.rank - 1))
        ops.append(dist.P2POp(dist.isend, own[: part.hb], part.rank - 1))
    if part.rank < part.world - 1:
        ops.append(dist.P2POp(dist.irecv, x_win[part.lo_halo + part.rows:], part.rank + 1))
        ops.append(dist.P2POp(dist.isend, own[part.rows - part.hb:], part.rank + 1))
    return ops


def dist_spmv_step(part: SpmvPartition, x_win: torch.Tensor,
                   run_rows: Callable[[int, int], None]) -> None:
    """One distributed y = A x: halo exchange overlapped with the interior rows.

    run_rows(lo, hi) computes local rows [lo, hi) reading x_win with
    col_base = part.col_base (enqueued on the current stream)."""
    ops = spmv_halo_ops(part, x_win)
    reqs = dist.batch_isend_irecv(ops) if ops else []
    i0, i1 = part.interior_rows()
    if i1 > i0:
        run_rows(i0, i1)
    for r in reqs:
        r.wait()
    if i0 > 0:
        run_rows(0, i0)
    if i1 < part.rows:
        run_rows(i1, part.rows)


# ---------------------------------------------------------------------------
# Stencil slabs with ghost rows/planes
# ---------------------------------------------------------------------------
@dataclass
class SlabPartition:
    """Slab [o0, o1) of the outer axis (n_outer rows/planes) with one ghost
    layer per side where a neighbour exists.  Local buffers cover global outer
    indices [g_lo, g_hi)."""

    n_outer: int
    world: int
    rank: int
    radius: int = 1

    def __post_init__(self):
        self.o0, self.o1 = block_range(self.n_outer, self.world, self.rank)
        self.g_lo = max(0, self.o0 - self.radius)
        self.g_hi = min(self.n_outer, self.o1 + self.radius)
        if self.world > 1 and (self.o1 - self.o0) < 2 * self.radius + 1:
            raise ValueError("slab thinner than its halo")

    @property
    def local_outer(self) -> int:
        return self.g_hi - self.g_lo

    def own_local(self):
        return self.o0 - self.g_lo, self.o1 - self.g_lo

    def interior_local(self):
        """Own layers that do not read a ghost layer."""
        a, b = self.own_local()
        lo = a + (self.radius if self.rank > 0 else 0)
        hi = b - (self.radius if self.rank < self.world - 1 else 0)
        return lo, max(lo, hi)


def stencil_halo_ops(part: SlabPartition, field: torch.Tensor):
    r = part.radius
    a, b = part.own_local()
    ops = []
    if part.rank > 0:
        ops.append(dist.P2POp(dist.irecv, field[a - r:a], part.rank - 1))
        ops.append(dist.P2POp(dist.isend, field[a:a + r], part.rank - 1))
    if part.rank < part.world - 1:
        ops.append(dist.P2POp(dist.irecv, field[b:b + r], part.rank + 1))
        ops.append(dist.P2POp(dist.isend, field[b - r:b], part.rank + 1))
    return ops


def dist_stencil_step(part: SlabPartition, src: torch.Tensor, dst: torch.Tensor,
                      sweep: Callable[[torch.Tensor, torch.Tensor, int, int], None]) -> None:
    """One timestep dst = S(src) on this slab.  sweep(src, dst, lo, hi) updates
    local outer indices [lo, hi) (boundary layers are skipped by the kernel)."""
    ops = stencil_halo_ops(part, src)
    reqs = dist.batch_isend_irecv(ops) if ops else []
    i0, i1 = part.interior_local()
    if i1 > i0:
        sweep(src, dst, i0, i1)
    for q in reqs:
        q.wait()
    a, b = part.own_local()
    if i0 > a:
        sweep(src, dst, a, i0)
    if b > i1:
        sweep(src, dst, i1, b)


def dist_stencil(part: SlabPartition, u: torch.Tensor, v: torch.Tensor, steps: int,
                 sweep: Callable[[torch.Tensor, torch.Tensor, int, int], None]) -> torch.Tensor:
    """`steps` double-buffered timesteps; returns the buffer holding the result."""
    for t in range(steps):
        src, dst = (u, v) if t % 2 == 0 else (v, u)
        dist_stencil_step(part, src, dst, sweep)
    return u if steps % 2 == 0 else v


def init_process_group(backend: Optional[str] = None) -> tuple[int, int]:
    """Rank/world from the torchrun environment (MASTER_ADDR should be 127.0.0.1)."""
    import os

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1 and not dist.is_initialized():
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        dist.init_process_group(backend=backend)
    return rank, world
