"""The kernels against committed golden vectors (tests/golden/kernels.npz,
made by tests/golden/make_kernel_golden.py from numpy and math.fsum, not from
this repo's oracle): STREAM bit-exact, SpMV (raw CSR kernels and the plan)
and the stencils within 1e-12 norm-wise, both units."""
import os

import numpy as np
import pytest

import oracle as O
import paper_2502_16851_b200 as P

pytestmark = pytest.mark.gpu
UNITS = [P.CUDA_CORE, P.TENSOR_CORE]
G = np.load(os.path.join(os.path.dirname(__file__), "golden", "kernels.npz"))


@pytest.mark.parametrize("unit", UNITS)
def test_golden_scale(cuda, unit):
    import torch

    b = torch.from_numpy(G["scale_b"]).cuda()
    a = torch.full_like(b, float("nan"))
    P.scale(a, b, float(G["scale_q"]), unit=unit)
    torch.cuda.synchronize()
    assert O.bit_mismatches(a.cpu().numpy(), G["scale_a"]) == 0


@pytest.mark.parametrize("unit", UNITS)
@pytest.mark.parametrize("path", ["csr", "plan"])
def test_golden_spmv(cuda, unit, path):
    import torch

    rp, col, val, x, y = (G[k] for k in ("spmv_rp", "spmv_col", "spmv_val", "spmv_x", "spmv_y"))
    m = rp.size - 1
    if path == "csr":
        d = [torch.from_numpy(t).cuda() for t in (rp, col, val, x)]
        dy = torch.full((m,), float("nan"), dtype=torch.float64, device="cuda")
        P.spmv_csr(d[0], d[1], d[2], d[3], dy, unit=unit)
        torch.cuda.synchronize()
        got = dy.cpu().numpy()
    else:
        plan = P.SpmvPlan(rp, col, val, x.size, unit=unit)
        try:
            got = np.full(m, np.nan)
            plan.execute_host(x, got)
        finally:
            plan.close()
    assert O.rel_err(got, y) <= 1e-12


@pytest.mark.parametrize("unit", UNITS)
@pytest.mark.parametrize("preset,key,steps", [("2d5pt", "s2d", 3), ("3d7pt", "s3d7", 2), ("3d27pt", "s3d27", 2)])
def test_golden_stencil(cuda, unit, preset, key, steps):
    import torch

    u0 = G[f"{key}_u0"]
    u = torch.from_numpy(u0.copy()).cuda()
    v = torch.from_numpy(u0.copy()).cuda()
    P.stencil(preset, u, v, steps, unit=unit)
    torch.cuda.synchronize()
    got = (u if steps % 2 == 0 else v).cpu().numpy()
    assert O.rel_err(got, G[f"{key}_v"]) <= 1e-12
