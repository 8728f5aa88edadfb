"""GPU parity of the sharded path (rl_dist_*, csrc/dist.cpp) on one B200.

Only one GPU is reachable here, so the multi-part schedule runs as several
parts on the same device: a world-1 NCCL communicator with parts_local = 2..4,
whose halo transfers are NCCL self send/recv inside the same group the
multi-GPU run posts (the exchange order per peer is the one
tests/test_dist.py checks over gloo between processes).  The per-part
compute is the sm_100a kernels; the halos start NaN-poisoned every call, so a
transfer the schedule misses shows up in the result.  Bar: 1e-12 norm-wise
relative error against the oracle (bit-exact for STREAM).  The first call of
a plan runs eagerly; the later ones replay the captured CUDA graph, and x /
the field change between calls so a replay that read stale inputs fails.
"""
import numpy as np
import pytest

import oracle as O
import paper_2502_16851_b200 as P
from paper_2502_16851_b200 import dist as D

pytestmark = pytest.mark.gpu

UNITS = [P.CUDA_CORE, P.TENSOR_CORE]
TOL = 1e-12


@pytest.fixture(scope="module")
def comm(cuda):
    c = D.Comm.single()
    yield c
    c.close()


def test_comm_info(comm):
    info = comm.info()
    assert info["world"] == 1 and info["rank"] == 0 and info["device"] == 0
    assert info["nccl_version"] >= 22700
    assert comm.allreduce_max(2.5) == 2.5
    assert comm.allreduce_sum(41) == 41


@pytest.mark.parametrize("unit", UNITS)
def test_dist_scale(comm, unit):
    import torch

    n = 1_000_003
    b = torch.empty(n, dtype=torch.float64, device="cuda")
    P.fill_uniform(b, 3, 1, 0, 1)
    a = torch.empty_like(b)
    kc = D.dist_scale(comm, a, b, 3.0, n, unit=unit)
    torch.cuda.synchronize()
    assert O.bit_mismatches(a.cpu().numpy(), O.scale(O.fill_uniform(n, 3, 1, 0, 1), 3.0)) == 0
    assert kc.traffic_bytes == 16 * n


def _spmv_parts(torch, n, k, hb, L, seed):
    parts, tens = [], []
    for i in range(L):
        p = D.SpmvPartition(n, hb, L, i)
        rp = torch.empty(p.rows + 1, dtype=torch.int32, device="cuda")
        col = torch.empty(p.rows * k, dtype=torch.int32, device="cuda")
        val = torch.empty(p.rows * k, dtype=torch.float64, device="cuda")
        P.gen_band_csr(p.rows, p.r0, n, k, hb, seed, rp, col, val)
        x = torch.empty(p.window, dtype=torch.float64, device="cuda")
        y = torch.full((p.rows,), float("nan"), dtype=torch.float64, device="cuda")
        parts.append(p)
        tens.append((rp, col, val, x, y))
    return parts, tens


@pytest.mark.parametrize("L", [1, 2, 3, 4])
@pytest.mark.parametrize("unit", UNITS)
def test_dist_spmv_parts_on_one_gpu(comm, L, unit):
    import torch

    n, k, hb, seed = 120_000, 16, 9000, 11
    parts, tens = _spmv_parts(torch, n, k, hb, L, seed)
    plan = D.DistSpmv(comm, n, hb, tens, unit=unit)
    rp, col, val = O.gen_band_csr(n, 0, n, k, hb, seed)
    try:
        for call in range(4):   # eager, capture + replay, replay, replay
            for p, (_, _, _, x, y) in zip(parts, tens):
                x.fill_(float("nan"))
                P.fill_uniform(x[p.own_slice()], seed + call, 4, p.r0, 1)
                y.fill_(float("nan"))
            kc = plan.execute()
            torch.cuda.synchronize()
            got = np.concatenate([t[4].cpu().numpy() for t in tens])
            ref = O.spmv_csr(rp, col, val, O.fill_uniform(n, seed + call, 4, 0, 1))
            assert not np.isnan(got).any(), call
            assert O.rel_err(got, ref) <= TOL, call
        assert (kc.work_flops, kc.traffic_bytes) == (P.spmv_csr_model(n, n, n * k).work_flops,
                                                    P.spmv_csr_model(n, n, n * k).traffic_bytes)
    finally:
        plan.close()


def test_dist_spmv_rejects_out_of_band(comm):
    import torch

    n, k, hb = 20_000, 8, 3000
    parts, tens = _spmv_parts(torch, n, k, hb, 2, 3)
    with pytest.raises(P.RooflensError) as e:
        D.DistSpmv(comm, n, hb // 2, tens)   # the matrix's band is wider than the declared halo
    assert e.value.kind == "ValidationError"


def _ghost_poisoned(torch, preset, gshape, p, seed):
    r = P.stencil_preset(preset)[2]
    u0 = O.stencil_init(p.local_shape, r, seed, outer_begin=p.g_lo, global_shape=gshape)
    a, b = p.own_local()
    u0[:a] = np.nan
    u0[b:] = np.nan
    return torch.from_numpy(u0).cuda(), torch.from_numpy(u0.copy()).cuda()


CASES = [("2d5pt", (203, 260)), ("3d7pt", (41, 30, 68)), ("3d27pt", (37, 24, 70)), ("2d9pt", (99, 132)),
         ("2d49pt", (120, 132))]


@pytest.mark.parametrize("L", [2, 3])
@pytest.mark.parametrize("unit", UNITS)
@pytest.mark.parametrize("preset,gshape", CASES)
def test_dist_stencil_parts_on_one_gpu(comm, L, unit, preset, gshape):
    import torch

    r = P.stencil_preset(preset)[2]
    parts = [D.SlabPartition(preset, gshape, L, i) for i in range(L)]
    # eager first; then 2-timestep graph replays; 23 = two 10-timestep graphs + a pair + an odd eager step
    for seed, steps in ((5, 3), (6, 4), (7, 23)):
        bufs = [_ghost_poisoned(torch, preset, gshape, p, seed) for p in parts]
        plan = D.DistStencil(comm, preset, gshape, [b[0] for b in bufs], [b[1] for b in bufs], unit=unit)
        try:
            for _ in range(2 if seed > 5 else 1):   # the second run of a plan replays its graph
                bufs2 = [_ghost_poisoned(torch, preset, gshape, p, seed) for p in parts]
                for (u, v), (u2, v2) in zip(bufs, bufs2):
                    u.copy_(u2)
                    v.copy_(v2)
                kc, in_v = plan.run(steps)
                torch.cuda.synchronize()
                got = np.concatenate([(b[1] if in_v else b[0]).cpu().numpy()[slice(*p.own_local())]
                                      for p, b in zip(parts, bufs)])
                ref = O.stencil(preset, O.stencil_init(gshape, r, seed), steps)
                assert not np.isnan(got).any()
                assert O.rel_err(got, ref) <= TOL
                inner = int(np.prod([s - 2 * r for s in gshape]))
                assert kc.traffic_bytes == 16 * inner * steps
        finally:
            plan.close()


@pytest.mark.slow
@pytest.mark.parametrize("unit", UNITS)
def test_dist_spmv_baseline_matrix_two_parts(comm, unit):
    """BASELINE configs[1] (2^22 rows, +-65536 band) split in two parts on one
    GPU against the single-launch kernel on the whole matrix."""
    import torch

    n, k, hb, seed = 1 << 22, 16, 65536, 2025
    parts, tens = _spmv_parts(torch, n, k, hb, 2, seed)
    for p, (_, _, _, x, _) in zip(parts, tens):
        x.fill_(float("nan"))
        P.fill_uniform(x[p.own_slice()], seed, 4, p.r0, 1)
    plan = D.DistSpmv(comm, n, hb, tens, unit=unit)
    for _ in range(3):
        plan.execute()
    torch.cuda.synchronize()
    got = torch.cat([t[4] for t in tens])
    rp = torch.empty(n + 1, dtype=torch.int32, device="cuda")
    col = torch.empty(n * k, dtype=torch.int32, device="cuda")
    val = torch.empty(n * k, dtype=torch.float64, device="cuda")
    P.gen_band_csr(n, 0, n, k, hb, seed, rp, col, val)
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    P.fill_uniform(x, seed, 4, 0, 1)
    ref = torch.empty(n, dtype=torch.float64, device="cuda")
    P.spmv_csr(rp, col, val, x, ref, unit=unit)
    torch.cuda.synchronize()
    assert float(torch.linalg.norm(got - ref) / torch.linalg.norm(ref)) <= TOL
    plan.close()
