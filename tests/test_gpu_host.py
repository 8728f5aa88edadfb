"""GPU parity of the end-to-end entry points on host buffers (rl_*_host,
rl_spmv_plan_*): pinned or pageable host arrays in, host arrays out."""
import numpy as np
import pytest

import oracle as O
import paper_2502_16851_b200 as P

pytestmark = pytest.mark.gpu
UNITS = [P.CUDA_CORE, P.TENSOR_CORE]


@pytest.mark.parametrize("unit", UNITS)
@pytest.mark.parametrize("n", [1, 1000, (4 << 20) + 77])
def test_scale_host(cuda, unit, n):
    b = O.fill_uniform(n, 3, 1, 0, 1)
    a = np.full(n, np.nan)
    kc = P.scale_host(a, b, 3.0, unit=unit)
    assert O.bit_mismatches(a, O.scale(b, 3.0)) == 0
    assert kc.traffic_bytes == 16 * n


@pytest.mark.parametrize("unit", UNITS)
def test_spmv_host_and_plan(cuda, unit):
    import torch

    m, k, hb = 300000, 16, 65536
    rp, col, val = O.gen_band_csr(m, 0, m, k, hb, 8)
    x = O.fill_uniform(m, 8, 4, 0, 1)
    ref = O.spmv_csr(rp, col, val, x)
    y = np.full(m, np.nan)
    kc = P.spmv_csr_host(rp, col, val, x, y, unit=unit)
    assert O.rel_err(y, ref) <= 1e-12
    assert kc == P.spmv_csr_model(m, m, m * k)
    # plan: matrix resident, x/y per call; pinned host buffers
    t = lambda a: torch.from_numpy(a).pin_memory()
    plan = P.SpmvPlan(t(rp), t(col), t(val), m, unit=unit)
    xp, yp = t(x), torch.full((m,), float("nan"), dtype=torch.float64).pin_memory()
    for _ in range(3):
        kc2 = plan.execute_host(xp, yp)
    assert O.rel_err(yp.numpy(), ref) <= 1e-12 and kc2 == kc
    # device execute on the same plan
    dx, dy = torch.from_numpy(x).cuda(), torch.empty(m, dtype=torch.float64, device="cuda")
    plan.execute(dx, dy)
    torch.cuda.synchronize()
    assert O.rel_err(dy.cpu().numpy(), ref) <= 1e-12
    plan.close()


def test_spmv_plan_validates_indices(cuda):
    rp = np.array([0, 2], np.int32)
    with pytest.raises(P.RooflensError) as e:
        P.SpmvPlan(rp, np.array([0, 5], np.int32), np.ones(2), 3)
    assert e.value.kind == "IndexOutOfRange"
    with pytest.raises(P.RooflensError) as e:
        P.SpmvPlan(np.array([0, 3], np.int32), np.array([0, 1], np.int32), np.ones(2), 3)
    assert e.value.kind == "ValidationError"


@pytest.mark.parametrize("unit", UNITS)
@pytest.mark.parametrize("preset,shape,steps", [("2d5pt", (130, 260), 3), ("3d7pt", (20, 24, 68), 2),
                                                ("3d27pt", (18, 20, 66), 3)])
def test_stencil_host(cuda, unit, preset, shape, steps):
    u0 = O.stencil_init(shape, 1, 6)
    u, v = u0.copy(), u0.copy()
    kc = P.stencil_host(preset, u, v, steps, unit=unit)
    out = u if steps % 2 == 0 else v
    assert O.rel_err(out, O.stencil(preset, u0, steps)) <= 1e-12
    assert kc.traffic_bytes == 16 * int(np.prod([s - 2 for s in shape])) * steps


def _plan_check(torch, rp, col, val, ncols, unit, expect_layout):
    """expect_layout: the plan's layout name ("csr", "colsort")."""
    x = np.random.default_rng(5).uniform(-1, 1, ncols)
    ref = O.spmv_csr(rp, col, val, x)
    plan = P.SpmvPlan(rp, col, val, ncols, unit=unit)
    assert plan.layout() == expect_layout
    y = np.full(rp.size - 1, np.nan)
    plan.execute_host(x, y)
    assert O.rel_err(y, ref) <= 1e-12
    dx = torch.from_numpy(x).cuda()
    dy = torch.full((rp.size - 1,), float("nan"), dtype=torch.float64, device="cuda")
    plan.execute(dx, dy)
    torch.cuda.synchronize()
    assert O.rel_err(dy.cpu().numpy(), ref) <= 1e-12
    # a second execution: bit-identical on CSR and on the CUDA-core column-sorted
    # layout (integer grid, flagged rows summed again in a fixed order); the tensor-core
    # one adds into shared-memory rows with FP64 atomics, last bits may move
    dy2 = torch.full_like(dy, float("nan"))
    plan.execute(dx, dy2)
    torch.cuda.synchronize()
    if expect_layout == "csr" or unit == P.CUDA_CORE:
        assert torch.equal(dy, dy2)
    else:
        assert O.rel_err(dy2.cpu().numpy(), dy.cpu().numpy()) <= 1e-15
    plan.close()


def test_plan_default_layout(cuda):
    """Plans take the column-sorted row-block layout (K17) when every row has
    <= 1024 nonzeros (both units); spmv_plan_colsort = 0 keeps the CSR."""
    import torch

    rp, col, val = O.gen_band_csr(10000, 0, 10000, 8, 500, 3)
    _plan_check(torch, rp, col, val, 10000, P.CUDA_CORE, "colsort")
    _plan_check(torch, rp, col, val, 10000, P.TENSOR_CORE, "colsort")
    try:
        P.tuning_set("spmv_plan_colsort", 0)
        _plan_check(torch, rp, col, val, 10000, P.CUDA_CORE, "csr")
    finally:
        P.tuning_set("spmv_plan_colsort", 1)


@pytest.mark.parametrize("unit", UNITS)
@pytest.mark.parametrize("m,n,k,hb", [(1024 * 5 + 3, 1024 * 5 + 3, 16, 65536), (100000, 100000, 16, 65536),
                                      (50000, 60000, 7, 300), (20000, 20000, 64, 20000),
                                      (30000, 30000, 5, 200000)])
def test_colsort_plan_banded(cuda, unit, m, n, k, hb):
    """Column-sorted row blocks: banded matrices, rectangular, and bands
    wider than the block count."""
    import torch

    rp, col, val = O.gen_band_csr(m, 0, n, k, hb, 37)
    prev = P.tuning_set("spmv_plan_colsort", 1)
    try:
        _plan_check(torch, rp, col, val, n, unit, "colsort")
    finally:
        P.tuning_set("spmv_plan_colsort", prev)


def test_colsort_plan_ragged_and_fallbacks(cuda):
    """Empty rows, ragged lengths and a full 1024-nonzero row stay on the
    column-sorted layout; a 1025-nonzero row keeps the CSR (long-row path)."""
    import torch

    rng = np.random.default_rng(12)
    m, n = 20000, 400000
    lens = rng.integers(0, 30, m)
    lens[::7] = 0
    lens[100] = 1024

    def build(lens, spread):
        rows = []
        for i, l in enumerate(lens):
            c0 = min(i * (n // m), n - spread)
            rows.append(np.sort(rng.choice(spread, l, replace=False)) + c0)
        rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
        return rp, np.concatenate(rows).astype(np.int32), rng.uniform(-1, 1, rp[-1])

    rp, col, val = build(lens, 5000)
    _plan_check(torch, rp, col, val, n, P.CUDA_CORE, "colsort")
    lens2 = lens.copy()
    lens2[200] = 1025
    rp, col, val = build(lens2, 5000)
    _plan_check(torch, rp, col, val, n, P.CUDA_CORE, "csr")
    rp, col, val = build(lens, 300000)  # rows spanning up to 300000 columns
    _plan_check(torch, rp, col, val, n, P.CUDA_CORE, "colsort")


@pytest.mark.parametrize("unit", UNITS)
def test_plan_ragged_dense_and_empty(cuda, unit):
    """Empty rows, very dense rows, a rectangular matrix and an odd column
    count through the default (CSR) plan layout."""
    import torch

    rng = np.random.default_rng(11)
    m, n = 20000, 30000
    lens = rng.integers(0, 30, m)
    lens[::5] = 0
    lens[7] = 9000        # one very dense row
    lens[8000:8010] = 3000
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    col = np.concatenate([np.sort(rng.choice(n, l, replace=False)) for l in lens]).astype(np.int32)
    val = rng.uniform(-1, 1, rp[-1])
    _plan_check(torch, rp, col, val, n, unit, "csr")
    _plan_check(torch, rp, col, val, n + 1, unit, "csr")


@pytest.mark.parametrize("colsort", [0, 1])
def test_plan_graph_replay_pinned(cuda, colsort):
    """Pinned x/y: execute_host runs as a captured CUDA graph.  New x
    contents are picked up on replay, a new (x, y) pair re-captures, and the
    launch counter advances per replay."""
    import torch

    P.tuning_set("spmv_plan_colsort", colsort)
    try:
        m = n = 70000
        rp, col, val = O.gen_band_csr(m, 0, n, 12, 9000, 17)
        plan = P.SpmvPlan(rp, col, val, n)
        rng = np.random.default_rng(1)
        xs = [torch.from_numpy(rng.uniform(-1, 1, n)).pin_memory() for _ in range(2)]
        ys = [torch.full((m,), float("nan"), dtype=torch.float64).pin_memory() for _ in range(2)]
        for it in range(3):
            for j in range(2):
                xs[j].copy_(torch.from_numpy(rng.uniform(-1, 1, n)))
                before = P.kernel_launches()
                plan.execute_host(xs[j], ys[j])
                assert P.kernel_launches() > before
                ref = O.spmv_csr(rp, col, val, xs[j].numpy())
                assert O.rel_err(ys[j].numpy(), ref) <= 1e-12
        plan.close()
    finally:
        P.tuning_set("spmv_plan_colsort", 1)


def test_plan_with_long_rows_pinned(cuda):
    """A skewed matrix through the plan: the long-row kernel runs inside the
    captured graph (its workspace is reserved at plan creation)."""
    import torch

    rng = np.random.default_rng(8)
    m = n = 30000
    lens = np.minimum(rng.zipf(1.6, m), 2500)
    lens[[5, 7000, 29000]] = 12000
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    col = np.concatenate([np.sort(rng.choice(n, l, replace=False)) for l in lens]).astype(np.int32)
    val = rng.uniform(-1, 1, rp[-1])
    plan = P.SpmvPlan(rp, col, val, n)
    hx = torch.from_numpy(rng.uniform(-1, 1, n)).pin_memory()
    hy = torch.empty(m, dtype=torch.float64).pin_memory()
    for _ in range(3):
        plan.execute_host(hx, hy)
        assert O.rel_err(hy.numpy(), O.spmv_csr(rp, col, val, hx.numpy())) <= 1e-12
    dy = torch.empty(m, dtype=torch.float64, device="cuda")
    plan.execute(hx.cuda(), dy)
    torch.cuda.synchronize()
    assert O.rel_err(dy.cpu().numpy(), O.spmv_csr(rp, col, val, hx.numpy())) <= 1e-12
    plan.close()


def test_plan_short_rows(cuda):
    """A short-row CSR (mean < 4 nonzeros, a few long rows): the plan picks the
    lane-per-row kernel from its host profile; pinned and pageable paths."""
    import torch

    rng = np.random.default_rng(21)
    m, n = 50000, 20000
    lens = rng.integers(0, 5, m)
    lens[rng.choice(m, 12, replace=False)] = 2500
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    col = np.concatenate([np.sort(rng.choice(n, l, replace=False)) for l in lens]).astype(np.int32)
    val = rng.uniform(-1, 1, rp[-1])
    _plan_check(torch, rp, col, val, n, P.CUDA_CORE, "csr")


def test_plan_graph_leading_empty_rows(cuda):
    """The first row chunks have no nonzeros (their x prefix is empty): the
    captured graph still contains their kernels and y copies, so replays with
    a poisoned y rewrite every row (capture fork event)."""
    import torch

    rng = np.random.default_rng(3)
    m = n = 64000
    lens = rng.integers(1, 20, m)
    lens[: m // 4] = 0
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    col = np.concatenate([np.sort(rng.choice(n, l, replace=False)) for l in lens]).astype(np.int32)
    val = rng.uniform(-1, 1, rp[-1])
    plan = P.SpmvPlan(rp, col, val, n)
    hx = torch.from_numpy(rng.uniform(-1, 1, n)).pin_memory()
    hy = torch.empty(m, dtype=torch.float64).pin_memory()
    for _ in range(3):
        hy.fill_(float("nan"))
        hx.copy_(torch.from_numpy(rng.uniform(-1, 1, n)))
        plan.execute_host(hx, hy)
        y = hy.numpy()
        assert not np.isnan(y).any()
        assert (y[: m // 4] == 0).all()
        assert O.rel_err(y, O.spmv_csr(rp, col, val, hx.numpy())) <= 1e-12
    plan.close()
