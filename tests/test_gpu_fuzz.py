"""Seeded randomised parity sweep: every executing kernel x unit over random
small shapes, random CSR structures (empty rows, long rows, unsorted-free
random columns), random stencil weights and odd/even extents, each compared
with the CPU oracle at the north-star tolerance (STREAM bit-exact, the rest
1e-12 norm-wise).  Complements the hand-picked edge cases in the per-kernel
test files."""
import numpy as np
import pytest

import oracle as O
import paper_2502_16851_b200 as P

pytestmark = pytest.mark.gpu

UNITS = [P.CUDA_CORE, P.TENSOR_CORE]
TOL = 1e-12
CASES = 40


def _rng(i):
    return np.random.default_rng(1000 + i)


@pytest.mark.parametrize("case", range(CASES))
@pytest.mark.parametrize("unit", UNITS)
def test_fuzz_scale(cuda, case, unit):
    import torch

    rng = _rng(case)
    n = int(rng.integers(1, 200000))
    off = int(rng.integers(0, 4))  # misaligned views
    b_full = torch.from_numpy(rng.uniform(-1e3, 1e3, n + off)).cuda()
    b = b_full[off:]
    a = torch.full_like(b, float("nan"))
    q = float(rng.uniform(-4, 4))
    P.scale(a, b, q, unit=unit)
    torch.cuda.synchronize()
    assert O.bit_mismatches(a.cpu().numpy(), O.scale(b.cpu().numpy(), q)) == 0


@pytest.mark.parametrize("case", range(CASES))
@pytest.mark.parametrize("unit", UNITS)
def test_fuzz_spmv_plan(cuda, case, unit):
    """Random CSR structures through rl_spmv_plan (the K17 column-sorted
    layout whenever every row has <= 1024 nonzeros, else CSR): empty rows,
    a long row, local and scattered columns, rectangular shapes, both the
    device and the host entry points."""
    import torch

    rng = _rng(500 + case)
    m, n = int(rng.integers(1, 40000)), int(rng.integers(1, 40000))
    lens = rng.integers(0, 48, m)
    lens[rng.random(m) < 0.15] = 0
    if m > 3 and case % 3 == 0:
        lens[int(rng.integers(0, m))] = min(n, int(rng.integers(200, 1500)))  # sometimes past 1024
    lens = np.minimum(lens, n)
    if lens.sum() == 0:
        lens[0] = 1
    local = case % 2 == 0  # banded columns, else scattered over all of x
    cols = []
    for i, l in enumerate(lens):
        if local:
            c0 = min(max(0, i * n // max(m, 1) - 500), max(0, n - 1000))
            span = min(n - c0, 1000)
            cols.append(np.sort(rng.choice(span, min(l, span), replace=False)) + c0)
        else:
            cols.append(np.sort(rng.choice(n, l, replace=False)))
    lens = np.array([c.size for c in cols])
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    col = np.concatenate(cols).astype(np.int32)
    val = rng.uniform(-1, 1, rp[-1])
    x = rng.uniform(-1, 1, n)
    ref = O.spmv_csr(rp, col, val, x)
    plan = P.SpmvPlan(rp, col, val, n, unit=unit)
    try:
        assert plan.layout() == ("colsort" if lens.max() <= 1024 else "csr")
        dy = torch.full((m,), float("nan"), dtype=torch.float64, device="cuda")
        plan.execute(torch.from_numpy(x).cuda(), dy)
        torch.cuda.synchronize()
        assert O.rel_err(dy.cpu().numpy(), ref) <= TOL
        hy = np.full(m, np.nan)
        plan.execute_host(x, hy)
        assert O.rel_err(hy, ref) <= TOL
    finally:
        plan.close()


@pytest.mark.parametrize("case", range(CASES))
@pytest.mark.parametrize("unit", UNITS)
def test_fuzz_spmv(cuda, case, unit):
    import torch

    rng = _rng(case)
    m, n = int(rng.integers(1, 5000)), int(rng.integers(1, 5000))
    lens = rng.integers(0, 40, m)
    lens[rng.random(m) < 0.2] = 0
    if m > 3:
        lens[int(rng.integers(0, m))] = min(n, int(rng.integers(100, 2000)))  # one long row
    lens = np.minimum(lens, n)
    if lens.sum() == 0:
        lens[0] = 1
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    col = np.concatenate([np.sort(rng.choice(n, l, replace=False)) for l in lens]).astype(np.int32)
    val = rng.uniform(-1, 1, rp[-1])
    x = rng.uniform(-1, 1, n)
    d = [torch.from_numpy(t).cuda() for t in (rp, col, val, x)]
    y = torch.full((m,), float("nan"), dtype=torch.float64, device="cuda")
    P.spmv_csr(d[0], d[1], d[2], d[3], y, unit=unit)
    torch.cuda.synchronize()
    assert O.rel_err(y.cpu().numpy(), O.spmv_csr(rp, col, val, x)) <= TOL


@pytest.mark.parametrize("case", range(CASES))
@pytest.mark.parametrize("unit", UNITS)
def test_fuzz_gemv(cuda, case, unit):
    import torch

    rng = _rng(case)
    m, n = int(rng.integers(1, 700)), int(rng.integers(1, 3000))
    A = rng.uniform(-1, 1, (m, n))
    x = rng.uniform(-1, 1, n)
    y = torch.full((m,), float("nan"), dtype=torch.float64, device="cuda")
    P.gemv(torch.from_numpy(A).cuda(), torch.from_numpy(x).cuda(), y, unit=unit)
    torch.cuda.synchronize()
    assert O.rel_err(y.cpu().numpy(), O.gemv(A, x)) <= TOL


PRESETS = ["2d5pt", "2d9pt", "2d13pt", "2d49pt", "3d7pt", "3d27pt"]


@pytest.mark.parametrize("case", range(CASES))
@pytest.mark.parametrize("unit", UNITS)
def test_fuzz_stencil(cuda, case, unit):
    import torch

    rng = _rng(case)
    preset = PRESETS[case % len(PRESETS)]
    dim, npts, r = P.stencil_preset(preset)
    if dim == 2:
        shape = (int(rng.integers(2 * r + 1, 300)), int(rng.integers(2 * r + 1, 300)))
    else:
        shape = tuple(int(rng.integers(3, 40)) for _ in range(3))
    if unit == P.TENSOR_CORE and preset in ("2d9pt", "2d13pt", "2d49pt") and shape[-1] % 2:
        shape = shape[:-1] + (shape[-1] + 1,)  # the TC kernels of these presets need 16-byte rows
    w = rng.uniform(-0.3, 0.4, npts) if rng.random() < 0.5 else None
    steps = int(rng.integers(1, 4))
    u0 = O.stencil_init(shape, r, int(rng.integers(1, 1 << 30)))
    u = torch.from_numpy(u0.copy()).cuda()
    v = torch.from_numpy(u0.copy()).cuda()
    P.stencil(preset, u, v, steps, weights=w, unit=unit)
    torch.cuda.synchronize()
    out = (u if steps % 2 == 0 else v).cpu().numpy()
    assert O.rel_err(out, O.stencil(preset, u0, steps, w)) <= TOL, (preset, shape, steps)
