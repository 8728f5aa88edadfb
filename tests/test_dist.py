"""Multi-process host logic of the sharded paths (CPU, gloo backend).

world_size 2 and 3, one process per rank over 127.0.0.1; the exchange code
is paper_2502_16851_b200.dist -- the same functions bench.py drives over NCCL
on GPUs -- with the CPU oracle standing in for the sm_100a kernels as the
per-rank compute.  Halo layers start as NaN so any row/plane that the
exchange fails to deliver poisons the result."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2502_16851_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _spmv_worker(rank, world, port, n, k, hb, seed, out):
    _init(rank, world, port)
    try:
        part = D.SpmvPartition(n, hb, world, rank)
        rp, col, val = O.gen_band_csr(part.rows, part.r0, n, k, hb, seed)
        xw = np.full(part.window, np.nan)
        xw[part.own_slice()] = O.fill_uniform(part.rows, seed, 4, part.r0, 1)
        x_win = torch.from_numpy(xw)
        y = np.full(part.rows, np.nan)
        order = []

        def run_rows(lo, hi):
            order.append((lo, hi))
            sub_rp = (rp[lo:hi + 1] - rp[lo]).astype(np.int32)
            y[lo:hi] = O.spmv_csr(sub_rp, col[rp[lo]:rp[hi]].copy(), val[rp[lo]:rp[hi]].copy(),
                                  x_win.numpy(), col_base=part.col_base)

        D.dist_spmv_step(part, x_win, run_rows)
        out[rank] = (part.r0, part.r1, y.copy(), order, part.interior_rows())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_dist_spmv_halo_exchange(world):
    n, k, hb, seed = 3000, 16, 400, 7
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_spmv_worker, args=(world, _free_port(), n, k, hb, seed, out), nprocs=world, join=True)
    rp, col, val = O.gen_band_csr(n, 0, n, k, hb, seed)
    ref = O.spmv_csr(rp, col, val, O.fill_uniform(n, seed, 4, 0, 1))
    got = np.empty(n)
    for r in range(world):
        r0, r1, y, order, interior = out[r]
        got[r0:r1] = y
        # interior rows run first (overlapping the exchange), edges after
        assert order[0] == tuple(interior) or interior[0] == interior[1]
    assert not np.isnan(got).any()
    assert O.rel_err(got, ref) < 1e-14


def test_spmv_partition_geometry():
    p = D.SpmvPartition(1 << 22, 65536, 8, 3)
    assert (p.r1 - p.r0) == 1 << 19
    assert p.lo_halo == p.hi_halo == 65536
    assert p.interior_rows() == (65536, (1 << 19) - 65536)
    edge = D.SpmvPartition(1 << 22, 65536, 8, 0)
    assert edge.lo_halo == 0 and edge.col_base == 0 and edge.interior_rows()[0] == 0
    with pytest.raises(ValueError):
        D.SpmvPartition(1000, 600, 4, 1)   # halo wider than a neighbour's rows
    lo, hi = D.scale_chunk(10, 3, 2)
    assert (lo, hi) == (7, 10)
    assert sum(D.block_range(1001, 8, r)[1] - D.block_range(1001, 8, r)[0] for r in range(8)) == 1001


def _stencil_worker(rank, world, port, preset, gshape, steps, seed, out):
    _init(rank, world, port)
    try:
        part = D.SlabPartition(gshape[0], world, rank, 1)
        local = (part.local_outer,) + tuple(gshape[1:])
        u = O.stencil_init(local, 1, seed, outer_begin=part.g_lo, global_shape=gshape)
        a, b = part.own_local()
        u[:a] = np.nan          # ghosts must come from the neighbours
        u[b:] = np.nan
        v = u.copy()
        tu, tv = torch.from_numpy(u), torch.from_numpy(v)

        def sweep(src, dst, lo, hi):
            # the kernel skips global boundary layers; in local coordinates a
            # rank's own first/last layer is a global boundary only at the ends
            glo = max(lo, 1 - part.g_lo)
            ghi = min(hi, gshape[0] - 1 - part.g_lo)
            if glo < ghi:
                O.stencil_sweep(preset, src.numpy(), dst.numpy(), glo, ghi)

        res = D.dist_stencil(part, tu, tv, steps, sweep)
        out[rank] = (part.o0, part.o1, res.numpy()[a:b].copy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("preset,gshape", [("2d5pt", (61, 33)), ("3d7pt", (23, 9, 12)), ("3d27pt", (19, 8, 10))])
def test_dist_stencil_slabs(world, preset, gshape):
    steps, seed = 4, 5
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_stencil_worker, args=(world, _free_port(), preset, gshape, steps, seed, out), nprocs=world,
             join=True)
    ref = O.stencil(preset, O.stencil_init(gshape, 1, seed), steps)
    got = np.empty(gshape)
    for r in range(world):
        o0, o1, block = out[r]
        got[o0:o1] = block
    assert not np.isnan(got).any()
    assert O.rel_err(got, ref) < 1e-14
