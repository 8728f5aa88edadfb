"""Maximum-size edge cases: element counts past 2^31 (64-bit indexing in every
kernel's address arithmetic).  The arrays are 17 GB each (B200 has 180 GB);
results are checked on the device against an independent torch computation
(STREAM, bit-exact) or, for the stencils, by running the oracle on the
sub-volume that determines the last rows / planes of the grid."""
import numpy as np
import pytest

import oracle as O
import paper_2502_16851_b200 as P

pytestmark = pytest.mark.gpu

UNITS = [P.CUDA_CORE, P.TENSOR_CORE]
TOL = 1e-12


@pytest.mark.parametrize("unit", UNITS)
def test_scale_past_2_31(cuda, unit):
    import torch

    n = (1 << 31) + 1027
    b = torch.empty(n, dtype=torch.float64, device="cuda")
    P.fill_uniform(b, 7, 1, 0, 1)
    a = torch.empty_like(b)
    P.scale(a, b, -2.5, unit=unit)
    ref = b * -2.5
    torch.cuda.synchronize()
    assert torch.equal(a, ref)
    del a, b, ref
    torch.cuda.empty_cache()


def _check_tail_rows(u0_tail, out_tail, preset, w=None):
    """out_tail[1:-1] must equal one oracle sweep of u0_tail (rows 1..-2)."""
    ref = O.stencil(preset, u0_tail, 1, w)
    assert O.rel_err(out_tail[1:-1], ref[1:-1]) <= TOL


@pytest.mark.parametrize("unit", UNITS)
def test_2d5pt_past_2_31_points(cuda, unit):
    import torch

    ny, nx = 46342, 46342  # 2.148e9 points
    u = torch.empty((ny, nx), dtype=torch.float64, device="cuda")
    P.stencil_init(u, 1, 11)
    v = u.clone()
    P.stencil("2d5pt", u, v, 1, unit=unit)
    torch.cuda.synchronize()
    k = 5  # the last k rows (the last one is the Dirichlet ring)
    u_tail = u[ny - k - 1:].cpu().numpy()
    v_tail = v[ny - k - 1:].cpu().numpy()
    # the tail sub-grid's first row and columns 0 / nx-1 act as its ring
    _check_tail_rows(u_tail, v_tail, "2d5pt")
    del u, v
    torch.cuda.empty_cache()


@pytest.mark.parametrize("unit", UNITS)
def test_3d7pt_past_2_31_points(cuda, unit):
    import torch

    n = 1292  # 2.157e9 points
    u = torch.empty((n, n, n), dtype=torch.float64, device="cuda")
    P.stencil_init(u, 1, 13)
    v = u.clone()
    P.stencil("3d7pt", u, v, 1, unit=unit)
    torch.cuda.synchronize()
    k = 3
    u_tail = u[n - k - 1:].cpu().numpy()
    v_tail = v[n - k - 1:].cpu().numpy()
    ref = O.stencil("3d7pt", u_tail, 1)
    assert O.rel_err(v_tail[1:-1, 1:-1, 1:-1], ref[1:-1, 1:-1, 1:-1]) <= TOL
    assert np.array_equal(v_tail[-1], u_tail[-1])  # the last plane is the Dirichlet ring
    del u, v
    torch.cuda.empty_cache()


@pytest.mark.parametrize("unit", UNITS)
def test_spmv_large_rows(cuda, unit):
    """2^29 rows, 3 nonzeros per row (1.6e9 nonzeros, ~30 GB): rows sampled
    across the whole range (and the last ones) against a host recomputation."""
    import torch

    m, k, hb = 1 << 29, 3, 1000
    rp = torch.empty(m + 1, dtype=torch.int32, device="cuda")
    col = torch.empty(m * k, dtype=torch.int32, device="cuda")
    val = torch.empty(m * k, dtype=torch.float64, device="cuda")
    x = torch.empty(m, dtype=torch.float64, device="cuda")
    y = torch.full((m,), float("nan"), dtype=torch.float64, device="cuda")
    P.gen_band_csr(m, 0, m, k, hb, 3, rp, col, val)
    P.fill_uniform(x, 3, 4, 0, 1)
    P.spmv_csr(rp, col, val, x, y, unit=unit)
    torch.cuda.synchronize()
    rows = np.concatenate([np.random.default_rng(0).integers(0, m, 2000), np.arange(m - 64, m)])
    r = torch.from_numpy(rows).cuda()
    starts = rp[r].long()
    idx = starts[:, None] + torch.arange(k, device="cuda")[None, :]  # k nonzeros per row
    ref = (val[idx] * x[col[idx].long()]).sum(dim=1)
    got = y[r]
    assert float(torch.linalg.norm(got - ref) / torch.linalg.norm(ref)) <= TOL
    assert int(rp[-1]) == m * k
    del rp, col, val, x, y
    torch.cuda.empty_cache()


@pytest.mark.parametrize("unit", UNITS)
def test_spmv_plan_colsort_large(cuda, unit):
    """2^24 rows, 8 nonzeros per row, +-65536 band through the column-sorted
    plan: blocks capped at 8192 rows (2048 blocks, ~7 waves), rows sampled
    across the whole range against a host recomputation."""
    import torch

    m, k, hb = 1 << 24, 8, 65536
    rp = torch.empty(m + 1, dtype=torch.int32, device="cuda")
    col = torch.empty(m * k, dtype=torch.int32, device="cuda")
    val = torch.empty(m * k, dtype=torch.float64, device="cuda")
    x = torch.empty(m, dtype=torch.float64, device="cuda")
    P.gen_band_csr(m, 0, m, k, hb, 5, rp, col, val)
    P.fill_uniform(x, 5, 4, 0, 1)
    plan = P.SpmvPlan(rp.cpu(), col.cpu(), val.cpu(), m, unit=unit)
    try:
        assert plan.layout() == "colsort"
        y = torch.full((m,), float("nan"), dtype=torch.float64, device="cuda")
        plan.execute(x, y)
        torch.cuda.synchronize()
        assert not torch.isnan(y).any()
        rows = np.concatenate([np.random.default_rng(1).integers(0, m, 4000), np.arange(m - 64, m)])
        r = torch.from_numpy(rows).cuda()
        idx = rp[r].long()[:, None] + torch.arange(k, device="cuda")[None, :]
        ref = (val[idx] * x[col[idx].long()]).sum(dim=1)
        assert float(torch.linalg.norm(y[r] - ref) / torch.linalg.norm(ref)) <= TOL
    finally:
        plan.close()
    del rp, col, val, x
    torch.cuda.empty_cache()
