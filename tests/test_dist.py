"""Multi-process host logic of the sharded paths (CPU, gloo backend).

The partition and the per-rank exchange schedule come from the library
itself (rl_dist_spmv_part / rl_dist_stencil_part / rl_dist_*_schedule in
csrc/dist.cpp -- exactly what rl_dist_spmv / rl_dist_stencil post as one NCCL
group on GPUs); here they are carried out over gloo by dist.run_schedule,
with the CPU oracle standing in for the sm_100a kernels as the per-part
compute.  world 2 and 3 processes over 127.0.0.1, one or two parts per rank
(two parts per rank exercise the self send/recv transfers the single-GPU
tests use).  Halo layers start as NaN so anything the schedule fails to
deliver poisons the result."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import paper_2502_16851_b200 as P
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


def _spmv_worker(rank, world, port, L, n, k, hb, seed, calls, out):
    _init(rank, world, port)
    try:
        parts = [D.SpmvPartition(n, hb, world * L, rank * L + i) for i in range(L)]
        ops = D.spmv_schedule(n, hb, world, L, rank)
        res = []
        for call in range(calls):
            bufs, mats = [], []
            for p in parts:
                rp, col, val = O.gen_band_csr(p.rows, p.r0, n, k, hb, seed)
                xw = np.full(p.window, np.nan)
                xw[p.own_slice()] = O.fill_uniform(p.rows, seed + call, 4, p.r0, 1)
                bufs.append(torch.from_numpy(xw))
                mats.append((rp, col, val))
            D.run_schedule(ops, bufs, rank)
            ys = []
            for p, xw, (rp, col, val) in zip(parts, bufs, mats):
                i0, i1 = p.interior_rows()
                y = np.full(p.rows, np.nan)
                for lo, hi in ((i0, i1), (0, i0), (i1, p.rows)):   # the plan's interior-then-edges order
                    if hi > lo:
                        sub = (rp[lo:hi + 1] - rp[lo]).astype(np.int32)
                        y[lo:hi] = O.spmv_csr(sub, col[rp[lo]:rp[hi]].copy(), val[rp[lo]:rp[hi]].copy(),
                                              xw.numpy(), col_base=p.col_base)
                ys.append((p.r0, p.r1, y))
            res.append(ys)
        out[rank] = res
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,L", [(2, 1), (2, 2), (3, 1)])
def test_dist_spmv_schedule_over_gloo(world, L):
    n, k, hb, seed, calls = 3000, 16, 300, 7, 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_spmv_worker, args=(world, _free_port(), L, n, k, hb, seed, calls, out), nprocs=world, join=True)
    rp, col, val = O.gen_band_csr(n, 0, n, k, hb, seed)
    for call in range(calls):
        ref = O.spmv_csr(rp, col, val, O.fill_uniform(n, seed + call, 4, 0, 1))
        got = np.full(n, np.nan)
        for r in range(world):
            for r0, r1, y in out[r][call]:
                got[r0:r1] = y
        assert not np.isnan(got).any()
        assert O.rel_err(got, ref) < 1e-14


def test_spmv_partition_geometry():
    p = D.SpmvPartition(1 << 22, 65536, 8, 3)
    assert (p.r1 - p.r0) == 1 << 19
    assert p.lo_halo == p.hi_halo == 65536
    assert p.interior_rows() == (65536, (1 << 19) - 65536)
    edge = D.SpmvPartition(1 << 22, 65536, 8, 0)
    assert edge.lo_halo == 0 and edge.col_base == 0 and edge.interior_rows()[0] == 0
    with pytest.raises(P.RooflensError) as e:
        D.SpmvPartition(1000, 600, 4, 1)   # halo wider than a neighbour's rows
    assert e.value.kind == "ValidationError"
    assert D.scale_chunk(10, 3, 2) == (7, 10)
    assert sum(D.block_range(1001, 8, r)[1] - D.block_range(1001, 8, r)[0] for r in range(8)) == 1001
    with pytest.raises(P.RooflensError):
        D.block_range(10, 0, 0)


def test_schedules_pair_up():
    """Every send has exactly one matching receive (same size, peers swapped)
    and, per ordered rank pair, sends and receives are posted in the same
    order -- the property NCCL's in-order matching needs."""
    cases = [("spmv", dict(n=1 << 16, hb=1000)), ("2d5pt", dict(shape=(64, 40))),
             ("3d27pt", dict(shape=(60, 6, 8))), ("2d49pt", dict(shape=(120, 16)))]
    for kind, kw in cases:
        for world, L in ((1, 3), (2, 1), (2, 3), (4, 2), (8, 1)):
            sched = {r: (D.spmv_schedule(kw["n"], kw["hb"], world, L, r) if kind == "spmv" else
                         D.stencil_schedule(kind, kw["shape"], world, L, r)) for r in range(world)}
            total = sum(len(v) for v in sched.values())
            assert total == 4 * (world * L - 1)
            for a in range(world):
                for b in range(world):
                    sends = [(o.count,) for o in sched[a] if o.kind == "send" and o.peer == b]
                    recvs = [(o.count,) for o in sched[b] if o.kind == "recv" and o.peer == a]
                    assert sends == recvs, (kind, world, L, a, b)


def _stencil_worker(rank, world, port, L, preset, gshape, steps, seed, out):
    _init(rank, world, port)
    try:
        r = P.stencil_preset(preset)[2]
        parts = [D.SlabPartition(preset, gshape, world * L, rank * L + i) for i in range(L)]
        ops = D.stencil_schedule(preset, gshape, world, L, rank)
        us, vs = [], []
        for p in parts:
            u = O.stencil_init(p.local_shape, r, seed, outer_begin=p.g_lo, global_shape=gshape)
            a, b = p.own_local()
            u[:a] = np.nan          # ghosts must come from the neighbours
            u[b:] = np.nan
            us.append(u)
            vs.append(u.copy())
        for t in range(steps):
            src, dst = (us, vs) if t % 2 == 0 else (vs, us)
            D.run_schedule(ops, [torch.from_numpy(s.reshape(-1)) for s in src], rank)
            for p, s, d in zip(parts, src, dst):
                a, b = p.own_local()
                # the kernel skips global boundary layers; in local coordinates a
                # part's own first/last layers are global boundaries only at the ends
                glo, ghi = max(a, r - p.g_lo), min(b, gshape[0] - r - p.g_lo)
                if glo < ghi:
                    O.stencil_sweep(preset, s, d, glo, ghi)
        res = us if steps % 2 == 0 else vs
        out[rank] = [(p.o0, p.o1, f[slice(*p.own_local())].copy()) for p, f in zip(parts, res)]
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,L", [(2, 1), (2, 2), (3, 1)])
@pytest.mark.parametrize("preset,gshape", [("2d5pt", (61, 33)), ("3d7pt", (23, 9, 12)), ("3d27pt", (19, 8, 10)),
                                           ("2d49pt", (45, 20))])
def test_dist_stencil_schedule_over_gloo(world, L, preset, gshape):
    steps, seed = 4, 5
    r = P.stencil_preset(preset)[2]
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_stencil_worker, args=(world, _free_port(), L, preset, gshape, steps, seed, out), nprocs=world,
             join=True)
    ref = O.stencil(preset, O.stencil_init(gshape, r, seed), steps)
    got = np.full(gshape, np.nan)
    for rk in range(world):
        for o0, o1, block in out[rk]:
            got[o0:o1] = block
    assert not np.isnan(got).any()
    assert O.rel_err(got, ref) < 1e-14
