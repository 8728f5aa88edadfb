"""GPU parity: CSR SpMV (K3 CUDA core, K4 tensor core) vs the CPU oracle.

Bar (BASELINE.json north_star): 1e-12 norm-wise relative error (summation
order and DMMA accumulation order differ from the oracle's row-order sum).
"""
import numpy as np
import pytest

import oracle as O
import paper_2502_16851_b200 as P

pytestmark = pytest.mark.gpu

UNITS = [P.CUDA_CORE, P.TENSOR_CORE]
TOL = 1e-12


def _to_dev(torch, *arrs):
    return [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in arrs]


def _run(torch, rp, col, val, x, unit):
    d_rp, d_col, d_val, d_x = _to_dev(torch, rp, col, val, x)
    d_y = torch.full((rp.size - 1,), float("nan"), dtype=torch.float64, device="cuda")
    kc = P.spmv_csr(d_rp, d_col, d_val, d_x, d_y, unit=unit)
    torch.cuda.synchronize()
    return d_y.cpu().numpy(), kc


def _ragged(rng, m, n, max_len, empty_frac=0.1):
    lens = rng.integers(0, max_len + 1, size=m)
    lens[rng.random(m) < empty_frac] = 0
    lens = np.minimum(lens, n)
    rp = np.zeros(m + 1, np.int64)
    rp[1:] = np.cumsum(lens)
    col = np.concatenate([np.sort(rng.choice(n, size=l, replace=False)) for l in lens]
                         ) if rp[-1] else np.zeros(0, np.int64)
    val = rng.uniform(-1, 1, size=rp[-1])
    return rp.astype(np.int32), col.astype(np.int32), val


@pytest.mark.parametrize("m,n,k,hb", [(64, 64, 16, 65536), (1000, 1000, 16, 100), (4099, 4099, 16, 65536),
                                      (20000, 20000, 16, 65536), (333, 333, 5, 7), (257, 257, 33, 40)])
@pytest.mark.parametrize("unit", UNITS)
def test_spmv_banded(cuda, m, n, k, hb, unit):
    import torch

    rp, col, val = O.gen_band_csr(m, 0, n, k, hb, 99)
    x = O.fill_uniform(n, 99, 4, 0, 1)
    y, kc = _run(torch, rp, col, val, x, unit)
    ref = O.spmv_csr(rp, col, val, x)
    assert O.rel_err(y, ref) <= TOL
    nnz = m * k
    assert kc.work_flops == 2 * nnz
    assert kc.traffic_bytes == (nnz + m + n) * 8 + (nnz + m + 1) * 4


@pytest.mark.parametrize("max_len", [3, 16, 40, 130])
@pytest.mark.parametrize("unit", UNITS)
def test_spmv_ragged_and_empty_rows(cuda, max_len, unit):
    import torch

    rng = np.random.default_rng(max_len)
    rp, col, val = _ragged(rng, 3001, 2500, max_len)
    x = rng.uniform(-1, 1, 2500)
    y, _ = _run(torch, rp, col, val, x, unit)
    ref = O.spmv_csr(rp, col, val, x)
    assert O.rel_err(y, ref) <= TOL
    assert np.all(y[np.diff(rp) == 0] == 0.0)  # empty rows give exactly 0


@pytest.mark.parametrize("unit", UNITS)
def test_spmv_single_row_and_column(cuda, unit):
    import torch

    rp = np.array([0, 1], np.int32)
    y, _ = _run(torch, rp, np.array([0], np.int32), np.array([2.5]), np.array([-4.0]), unit)
    assert y[0] == -10.0
    # one dense row of 1000
    n = 1000
    rp = np.array([0, n], np.int32)
    col = np.arange(n, dtype=np.int32)
    val = np.linspace(-1, 1, n)
    x = np.cos(np.arange(n))
    y, _ = _run(torch, rp, col, val, x, unit)
    assert O.rel_err(y, O.spmv_csr(rp, col, val, x)) <= TOL


@pytest.mark.parametrize("unit", UNITS)
def test_spmv_rows_with_col_base(cuda, unit):
    """Row-range form used by the row-partitioned path: x is a window."""
    import torch

    m, n, k, hb = 5000, 5000, 16, 300
    rp, col, val = O.gen_band_csr(m, 0, n, k, hb, 3)
    x = O.fill_uniform(n, 3, 4, 0, 1)
    ref = O.spmv_csr(rp, col, val, x)
    r0, r1 = 1200, 3700
    lo, hi = r0 - hb, r1 + hb
    d_rp, d_col, d_val = _to_dev(torch, rp, col, val)
    d_xw = torch.from_numpy(x[lo:hi].copy()).cuda()
    d_y = torch.zeros(m, dtype=torch.float64, device="cuda")
    P.spmv_csr_rows(r0, r1, d_rp, d_col, d_val, d_xw, d_y, col_base=lo, unit=unit)
    torch.cuda.synchronize()
    y = d_y.cpu().numpy()
    assert O.rel_err(y[r0:r1], ref[r0:r1]) <= TOL
    assert np.all(y[:r0] == 0) and np.all(y[r1:] == 0)


def test_spmv_generator_matches_oracle(cuda):
    import torch

    m, n, k, hb = 70000, 70000, 16, 65536
    d_rp = torch.empty(m + 1, dtype=torch.int32, device="cuda")
    d_col = torch.empty(m * k, dtype=torch.int32, device="cuda")
    d_val = torch.empty(m * k, dtype=torch.float64, device="cuda")
    P.gen_band_csr(m, 0, n, k, hb, 42, d_rp, d_col, d_val)
    torch.cuda.synchronize()
    rp, col, val = O.gen_band_csr(m, 0, n, k, hb, 42)
    assert np.array_equal(d_rp.cpu().numpy(), rp)
    assert np.array_equal(d_col.cpu().numpy(), col)
    assert O.bit_mismatches(d_val.cpu().numpy(), val) == 0


@pytest.mark.slow
@pytest.mark.parametrize("unit", UNITS)
def test_spmv_full_config(cuda, unit):
    """BASELINE configs[1]: n = 2^22, 16 nnz/row in a +-65536 band."""
    import torch

    n, k, hb, seed = 1 << 22, 16, 65536, 2025
    d_rp = torch.empty(n + 1, dtype=torch.int32, device="cuda")
    d_col = torch.empty(n * k, dtype=torch.int32, device="cuda")
    d_val = torch.empty(n * k, dtype=torch.float64, device="cuda")
    d_x = torch.empty(n, dtype=torch.float64, device="cuda")
    d_y = torch.empty(n, dtype=torch.float64, device="cuda")
    P.gen_band_csr(n, 0, n, k, hb, seed, d_rp, d_col, d_val)
    P.fill_uniform(d_x, seed, 4, 0, 1)
    kc = P.spmv_csr(d_rp, d_col, d_val, d_x, d_y, unit=unit)
    torch.cuda.synchronize()
    assert kc.traffic_bytes == 889192452 and kc.work_flops == 134217728
    rp, col, val = O.gen_band_csr(n, 0, n, k, hb, seed)
    x = O.fill_uniform(n, seed, 4, 0, 1)
    assert np.array_equal(d_col.cpu().numpy(), col)
    ref = O.spmv_csr(rp, col, val, x)
    assert O.rel_err(d_y.cpu().numpy(), ref) <= TOL


def test_spmv_errors(cuda):
    import torch

    z = torch.zeros(4, dtype=torch.float64, device="cuda")
    rp = torch.zeros(5, dtype=torch.int32, device="cuda")
    with pytest.raises(P.RooflensError) as e:  # nnz = 0: the model rejects it
        P.spmv_csr(rp, rp[:0], z[:0], z, z)
    assert e.value.kind == "ValidationError"


def _skewed_csr(m, n, seed, huge=(3, 20000)):
    """Power-law row lengths plus a few huge rows (many pieces each)."""
    rng = np.random.default_rng(seed)
    lens = np.minimum(rng.zipf(1.6, m), 3000).astype(np.int64)
    for r in rng.choice(m, huge[0], replace=False):
        lens[r] = huge[1]
    lens = np.minimum(lens, n)
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    col = np.concatenate([np.sort(rng.choice(n, l, replace=False)) for l in lens]).astype(np.int32)
    return rp, col, rng.uniform(-1, 1, rp[-1])


@pytest.mark.parametrize("unit", UNITS)
def test_spmv_long_rows_diverted(cuda, unit):
    """Rows past spmv_long_min go to the load-balanced second kernel (rows cut
    into spmv_long_piece-nonzero pieces, equal runs of pieces per warp);
    results equal the oracle."""
    import torch

    m, n = 20000, 30000
    rp, col, val = _skewed_csr(m, n, 3)
    assert np.diff(rp).max() > 8192 and (np.diff(rp) > 64).sum() > 50
    x = np.random.default_rng(4).uniform(-1, 1, n)
    d = [torch.from_numpy(t).cuda() for t in (rp, col, val, x)]
    y = torch.full((m,), float("nan"), dtype=torch.float64, device="cuda")
    for _ in range(3):  # the counters reset themselves between calls
        P.spmv_csr(d[0], d[1], d[2], d[3], y, unit=unit)
        torch.cuda.synchronize()
        assert O.rel_err(y.cpu().numpy(), O.spmv_csr(rp, col, val, x)) <= TOL


@pytest.mark.parametrize("unit", UNITS)
@pytest.mark.parametrize("piece", [64, 100, 777, 2048, 1 << 20])
@pytest.mark.parametrize("group", [8, 16, 32])
def test_spmv_long_row_pieces(cuda, unit, piece, group):
    """Any piece size (not a multiple of 4, or larger than every row) gives
    the oracle's result, bit-identical from call to call (split rows are
    summed in piece order by whichever warp finishes last)."""
    import torch

    m, n = 6000, 30000
    rp, col, val = _skewed_csr(m, n, 8, huge=(5, 25000))
    x = np.random.default_rng(9).uniform(-1, 1, n)
    d = [torch.from_numpy(t).cuda() for t in (rp, col, val, x)]
    y = torch.full((m,), float("nan"), dtype=torch.float64, device="cuda")
    P.tuning_set("spmv_long_piece", piece)
    P.tuning_set("spmv_long_group", group)
    try:
        outs = []
        for _ in range(3):
            P.spmv_csr(d[0], d[1], d[2], d[3], y, unit=unit)
            torch.cuda.synchronize()
            outs.append(y.cpu().numpy().copy())
    finally:
        P.tuning_set("spmv_long_piece", 512)
        P.tuning_set("spmv_long_group", 8)
    assert O.rel_err(outs[0], O.spmv_csr(rp, col, val, x)) <= TOL
    assert O.bit_mismatches(outs[0], outs[1]) == 0 and O.bit_mismatches(outs[0], outs[2]) == 0


@pytest.mark.parametrize("unit", UNITS)
def test_spmv_long_row_piece_capacity(cuda, unit):
    """More split pieces than the workspace holds (65536 at this size): the
    rows past capacity are computed whole by one warp, still exact."""
    import torch

    m, n = 3000, 8000
    rng = np.random.default_rng(12)
    lens = rng.integers(2000, 4000, m)
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    col = np.concatenate([np.sort(rng.choice(n, l, replace=False)) for l in lens]).astype(np.int32)
    val = rng.uniform(-1, 1, rp[-1])
    assert rp[-1] // 64 > 65536
    x = rng.uniform(-1, 1, n)
    d = [torch.from_numpy(t).cuda() for t in (rp, col, val, x)]
    y = torch.full((m,), float("nan"), dtype=torch.float64, device="cuda")
    P.tuning_set("spmv_long_piece", 64)
    try:
        P.spmv_csr(d[0], d[1], d[2], d[3], y, unit=unit)
        torch.cuda.synchronize()
    finally:
        P.tuning_set("spmv_long_piece", 512)
    assert O.rel_err(y.cpu().numpy(), O.spmv_csr(rp, col, val, x)) <= TOL


@pytest.mark.parametrize("unit", UNITS)
@pytest.mark.parametrize("long_rows", [False, True])
@pytest.mark.parametrize("m", [1, 31, 33, 5000, 70001])
def test_spmv_short_rows(cuda, unit, long_rows, m):
    """Rows of 0-5 nonzeros (power-law graphs' many tiny rows), with and
    without diverted long rows; empty rows give 0."""
    import torch

    n = 4000
    rng = np.random.default_rng(m + 7 * long_rows)
    lens = rng.integers(0, 6, m)
    if long_rows and m > 40:
        lens[rng.choice(m, 20, replace=False)] = rng.integers(65, 3000, 20)
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    if rp[-1] == 0:
        lens[0] = 1
        rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    col = np.concatenate([np.sort(rng.choice(n, l, replace=False)) for l in lens]).astype(np.int32)
    val = rng.uniform(-1, 1, rp[-1])
    x = rng.uniform(-1, 1, n)
    d = [torch.from_numpy(t).cuda() for t in (rp, col, val, x)]
    y = torch.full((m,), float("nan"), dtype=torch.float64, device="cuda")
    for _ in range(2):
        P.spmv_csr(d[0], d[1], d[2], d[3], y, unit=unit)
        torch.cuda.synchronize()
        got = y.cpu().numpy()
        assert O.rel_err(got, O.spmv_csr(rp, col, val, x)) <= TOL
        assert np.all(got[lens == 0] == 0.0)


@pytest.mark.parametrize("unit", UNITS)
def test_spmv_profile_cache_stale_is_still_correct(cuda, unit):
    """The long-row profile is cached per buffer triple: rewriting the same
    buffers with a different structure must still give exact results."""
    import torch

    m, n = 4000, 4000
    rp1, col1, val1 = O.gen_band_csr(m, 0, n, 8, 100, 1)           # short rows only
    rp2, col2, val2 = _skewed_csr(m, n, 5, huge=(2, 3500))          # long rows
    nnz = max(rp1[-1], rp2[-1])
    drp = torch.empty(m + 1, dtype=torch.int32, device="cuda")
    dcol = torch.empty(nnz, dtype=torch.int32, device="cuda")
    dval = torch.empty(nnz, dtype=torch.float64, device="cuda")
    x = np.random.default_rng(6).uniform(-1, 1, n)
    dx = torch.from_numpy(x).cuda()
    y = torch.empty(m, dtype=torch.float64, device="cuda")
    for rp, col, val in ((rp1, col1, val1), (rp2, col2, val2), (rp1, col1, val1)):
        drp.copy_(torch.from_numpy(rp))
        dcol[:rp[-1]].copy_(torch.from_numpy(col))
        dval[:rp[-1]].copy_(torch.from_numpy(val))
        P.spmv_csr(drp, dcol, dval, dx, y, unit=unit)
        torch.cuda.synchronize()
        assert O.rel_err(y.cpu().numpy(), O.spmv_csr(rp, col, val, x)) <= TOL


@pytest.mark.parametrize("unit", UNITS)
@pytest.mark.parametrize("val_off,col_off", [(1, 0), (0, 1), (1, 3), (2, 2), (3, 1)])
@pytest.mark.parametrize("max_len", [16, 300])   # 300: rows go through the long-row kernel too
def test_spmv_offset_views(cuda, unit, val_off, col_off, max_len):
    """val / col as views at an element offset inside larger buffers: the
    256-bit val and 128-bit col vector loads need 32- / 16-byte aligned bases,
    so such views must take the element loads (a vector load would raise
    cudaErrorMisalignedAddress and poison the context)."""
    import torch

    rng = np.random.default_rng(100 + val_off * 7 + col_off)
    m, n = 3001, 4000
    rp, col, val = _ragged(rng, m, n, max_len, empty_frac=0.05)
    x = rng.uniform(-1, 1, n)
    nnz = int(rp[-1])
    vbuf = torch.empty(nnz + 8, dtype=torch.float64, device="cuda")
    cbuf = torch.empty(nnz + 8, dtype=torch.int32, device="cuda")
    vbuf[val_off:val_off + nnz] = torch.from_numpy(val).cuda()
    cbuf[col_off:col_off + nnz] = torch.from_numpy(col).cuda()
    d_rp, d_x = _to_dev(torch, rp, x)
    y = torch.full((m,), float("nan"), dtype=torch.float64, device="cuda")
    P.spmv_csr(d_rp, cbuf[col_off:col_off + nnz], vbuf[val_off:val_off + nnz], d_x, y, unit=unit)
    torch.cuda.synchronize()
    assert O.rel_err(y.cpu().numpy(), O.spmv_csr(rp, col, val, x)) <= TOL


def _plan_case(case):
    rng = np.random.default_rng({"band": 1, "ragged": 2, "empty_block": 3, "long_rows": 4, "narrow": 5,
                                 "rect": 6, "scattered": 7, "tiny": 8, "hot_row": 9}[case])
    if case == "band":
        m = n = 300_000
        rp, col, val = O.gen_band_csr(m, 0, n, 16, 20000, 9)
    elif case == "narrow":
        m = n = 70_001
        rp, col, val = O.gen_band_csr(m, 0, n, 5, 4, 4)
    elif case == "tiny":
        m = n = 37
        rp, col, val = O.gen_band_csr(m, 0, n, 3, 5, 4)
    elif case == "rect":
        m, n = 90_001, 250_000
        rp, col, val = O.gen_band_csr(m, 0, n, 12, 60000, 5)
    elif case == "scattered":  # every row reaches across all of x
        m = n = 100_000
        rp = np.arange(m + 1, dtype=np.int32) * 8
        col = np.concatenate([np.sort(rng.choice(n, 8, replace=False)) for _ in range(m)]).astype(np.int32)
        val = rng.uniform(-1, 1, col.size)
    else:
        m = n = 200_000
        hbw = 6000
        lens = rng.integers(0, 40, size=m)
        if case == "empty_block":
            lens[50_000:90_000] = 0
        if case == "long_rows":
            lens[rng.choice(m, 20, replace=False)] = 1000
        if case == "hot_row":  # past kColsortMaxRowLen: the plan keeps CSR
            lens[777] = 1025
        cols = []
        for i, l in enumerate(lens):
            lo, hi = max(0, i - hbw), min(n, i + hbw + 1)
            cols.append(np.sort(rng.choice(np.arange(lo, hi), size=min(l, hi - lo), replace=False)))
        rp = np.zeros(m + 1, np.int64)
        rp[1:] = np.cumsum([c.size for c in cols])
        col = np.concatenate(cols).astype(np.int32)
        rp = rp.astype(np.int32)
        val = rng.uniform(-1, 1, size=col.size)
    return m, n, rp, col, val


@pytest.mark.parametrize("unit", UNITS)
@pytest.mark.parametrize("case", ["band", "ragged", "empty_block", "long_rows", "narrow", "rect", "scattered",
                                  "tiny", "hot_row"])
def test_spmv_plan_colsort_layout(cuda, unit, case):
    """K17 (spmv_colsort.cu): column-sorted row blocks with y in shared
    memory, the plans' default layout when eligible (rows of <= 1024
    nonzeros).  Both units, through rl_spmv_plan_execute (device x, y) and
    execute_host, on repeated calls with new x, NaN-poisoned y."""
    import torch

    m, n, rp, col, val = _plan_case(case)
    prev = P.tuning_set("spmv_plan_colsort", 1)
    try:
        plan = P.SpmvPlan(rp, col, val, n, unit=unit)
    finally:
        P.tuning_set("spmv_plan_colsort", prev)
    try:
        assert plan.layout() == ("csr" if case == "hot_row" else "colsort"), plan.layout()
        for call in range(3):
            x = O.fill_uniform(n, 40 + call, 4, 0, 1)
            ref = O.spmv_csr(rp, col, val, x)
            dx = torch.from_numpy(x).cuda()
            dy = torch.full((m,), float("nan"), dtype=torch.float64, device="cuda")
            plan.execute(dx, dy)
            torch.cuda.synchronize()
            assert O.rel_err(dy.cpu().numpy(), ref) <= TOL, call
            if case == "empty_block":
                assert (dy[50_000:90_000] == 0).all()
            hx = torch.from_numpy(x).pin_memory()
            hy = torch.full((m,), float("nan"), dtype=torch.float64).pin_memory()
            plan.execute_host(hx, hy)
            assert O.rel_err(hy.numpy(), ref) <= TOL, call
    finally:
        plan.close()


def test_spmv_plan_colsort_opt_out(cuda):
    """tuning key spmv_plan_colsort = 0 keeps the caller's CSR."""
    m, n, rp, col, val = _plan_case("band")
    prev = P.tuning_set("spmv_plan_colsort", 0)
    try:
        plan = P.SpmvPlan(rp, col, val, n)
    finally:
        P.tuning_set("spmv_plan_colsort", prev)
    assert plan.layout() == "csr"
    plan.close()


@pytest.mark.parametrize("unit", UNITS)
def test_spmv_plan_colsort_baseline(cuda, unit):
    """The BASELINE matrix (2^22 rows, 16 nnz/row, +-65536 band) through the
    K17 plan built from the device generator's CSR: 1e-12 vs the oracle, and
    the layout moves no more bytes than the CSR it replaces."""
    import torch

    m, k, hb = 1 << 22, 16, 65536
    rp, col, val = O.gen_band_csr(m, 0, m, k, hb, 2025)
    x = O.fill_uniform(m, 2025, 4, 0, 1)
    prev = P.tuning_set("spmv_plan_colsort", 1)
    try:
        plan = P.SpmvPlan(rp, col, val, m, unit=unit)
    finally:
        P.tuning_set("spmv_plan_colsort", prev)
    try:
        layout, nbytes = plan.info()
        assert layout == "colsort" and nbytes <= (m + 1) * 4 + m * k * 12
        dx = torch.from_numpy(x).cuda()
        dy = torch.full((m,), float("nan"), dtype=torch.float64, device="cuda")
        plan.execute(dx, dy)
        torch.cuda.synchronize()
        assert O.rel_err(dy.cpu().numpy(), O.spmv_csr(rp, col, val, x)) <= TOL
    finally:
        plan.close()


def _fsum_rows(rp, col, val, x):
    """Correctly rounded exact row sums of the FP64-rounded products (math.fsum)."""
    import math

    prod = val * x[col]
    return np.array([math.fsum(prod[rp[i]:rp[i + 1]]) for i in range(rp.size - 1)])


@pytest.mark.parametrize("unit", UNITS)
@pytest.mark.parametrize("m,k,hb", [(20000, 16, 65536), (7001, 7, 300), (3000, 64, 1000)])
def test_colsort_within_fp64_summation_bound(cuda, unit, m, k, hb):
    """K17 rows against the exact sum (math.fsum): within the recursive
    summation bound (L - 1) u sum|p| or within 2^-46 of the row's magnitude
    (fixed-point rows), on both units and on every call."""
    import torch

    rng = np.random.default_rng(m + k)
    rp, col, val = O.gen_band_csr(m, 0, m, k, hb, 5)
    x = rng.uniform(-1.0, 1.0, m)
    want = _fsum_rows(rp, col, val, x)
    absum = np.array([np.abs(val[rp[i]:rp[i + 1]] * x[col[rp[i]:rp[i + 1]]]).sum() for i in range(m)])
    lens = np.diff(rp)
    prev = P.tuning_set("spmv_plan_colsort", 1)
    try:
        plan = P.SpmvPlan(rp, col, val, m, unit=unit)
    finally:
        P.tuning_set("spmv_plan_colsort", prev)
    try:
        assert plan.layout() == "colsort"
        dx = torch.from_numpy(x).cuda()
        for _ in range(2):
            dy = torch.full((m,), float("nan"), dtype=torch.float64, device="cuda")
            plan.execute(dx, dy)
            torch.cuda.synchronize()
            err = np.abs(dy.cpu().numpy() - want)
            # FP64 rows (atomics or the row kernel): the recursive-summation bound;
            # fixed-point rows: within 2^-46 of their own magnitude
            assert np.all(err <= np.maximum(np.maximum(lens - 1, 1) * 2.0 ** -53 * absum * 1.0001,
                                            2.0 ** -46 * np.abs(want)))
    finally:
        plan.close()


@pytest.mark.parametrize("unit", UNITS)
def test_colsort_scales_and_ranges(cuda, unit):
    """Per-block scales: rows of very different magnitude in different blocks
    (1e-200 .. 1e200), x spanning 1e-150 .. 1e150 across segments (blocks
    whose x window spans more than 2^24 take the FP64 path), zeros and
    subnormals: each row within 1e-13 of its largest product or of the exact
    sum."""
    import torch

    rng = np.random.default_rng(31)
    m = n = 50000
    rp, col, val = O.gen_band_csr(m, 0, n, 12, 3000, 9)
    row_scale = 10.0 ** np.repeat(rng.integers(-200, 200, m // 500 + 1), 500)[:m]
    val = val * np.repeat(row_scale, np.diff(rp))
    x = O.fill_uniform(n, 3, 4, 0, 1) * 10.0 ** np.repeat(rng.integers(-150, 150, n // 4096 + 1), 4096)[:n]
    x[::97] = 0.0
    x[5::1001] = 5e-324  # subnormal
    want = _fsum_rows(rp, col, val, x)
    prev = P.tuning_set("spmv_plan_colsort", 1)
    try:
        plan = P.SpmvPlan(rp, col, val, n, unit=unit)
    finally:
        P.tuning_set("spmv_plan_colsort", prev)
    try:
        dx = torch.from_numpy(x).cuda()
        dy = torch.empty(m, dtype=torch.float64, device="cuda")
        plan.execute(dx, dy)
        torch.cuda.synchronize()
        y = dy.cpu().numpy()
        scale = np.maximum(np.abs(want), np.array([np.abs(val[rp[i]:rp[i + 1]] * x[col[rp[i]:rp[i + 1]]]).max(initial=0)
                                                   for i in range(m)]))
        ok = scale > 0
        assert np.all(np.abs(y - want)[ok] <= 1e-13 * scale[ok])
        assert np.all(y[~ok] == 0)
    finally:
        plan.close()


@pytest.mark.parametrize("unit", UNITS)
def test_colsort_nonfinite(cuda, unit):
    """Inf/NaN in x or in the values: the affected blocks add in FP64 (IEEE
    semantics) -- the non-finite pattern of y matches the CPU sum's, the
    finite rows stay within 1e-12."""
    import torch

    m = n = 30000
    rp, col, val = O.gen_band_csr(m, 0, n, 10, 2000, 4)
    val = val.copy()
    val[rp[20000] + 3] = np.inf
    x = O.fill_uniform(n, 8, 4, 0, 1)
    x[1234] = np.nan
    x[25000] = -np.inf
    with np.errstate(invalid="ignore"):
        want = np.array([np.sum(val[rp[i]:rp[i + 1]] * x[col[rp[i]:rp[i + 1]]]) for i in range(m)])
    prev = P.tuning_set("spmv_plan_colsort", 1)
    try:
        plan = P.SpmvPlan(rp, col, val, n, unit=unit)
    finally:
        P.tuning_set("spmv_plan_colsort", prev)
    try:
        dy = torch.empty(m, dtype=torch.float64, device="cuda")
        plan.execute(torch.from_numpy(x).cuda(), dy)
        torch.cuda.synchronize()
        y = dy.cpu().numpy()
        assert np.array_equal(np.isnan(y), np.isnan(want))
        assert np.array_equal(np.isposinf(y), np.isposinf(want)) and np.array_equal(np.isneginf(y), np.isneginf(want))
        f = np.isfinite(want)
        assert O.rel_err(y[f], want[f]) <= TOL
    finally:
        plan.close()


@pytest.mark.parametrize("unit", UNITS)
@pytest.mark.parametrize("fixed", [1, 2, 0])
def test_colsort_small_rows_spikes_and_determinism(cuda, unit, fixed):
    """Rows whose sum cancels or whose products all lie far below the block's
    largest (an x spike of 1e12 in every block's window) leave the 64-bit grid
    for the FP64 row kernel: every row within the FP64 recursive-summation
    bound of the exact sum.  Fixed-point results are bit-identical call to
    call (spmv_colsort_fixed: 1 the CUDA-core unit, 2 both); x = 0 gives exact
    zeros."""
    import torch

    rng = np.random.default_rng(77)
    m = n = 60000
    rp, col, val = O.gen_band_csr(m, 0, n, 12, 4000, 6)
    val = val.copy()
    # cancelling rows: second half of each row the negated first half, same x
    for i in range(0, m, 97):
        a, b = rp[i], rp[i + 1]
        h = (b - a) // 2
        val[a + h:a + 2 * h] = -val[a:a + h]
    x = rng.uniform(-1, 1, n)
    x[::5000] = 1e12  # spikes
    want = _fsum_rows(rp, col, val, x)
    absum = np.array([np.abs(val[rp[i]:rp[i + 1]] * x[col[rp[i]:rp[i + 1]]]).sum() for i in range(m)])
    lens = np.diff(rp)
    prev = P.tuning_set("spmv_colsort_fixed", fixed)
    try:
        plan = P.SpmvPlan(rp, col, val, n, unit=unit)
    finally:
        P.tuning_set("spmv_colsort_fixed", prev)
    try:
        dx = torch.from_numpy(x).cuda()
        outs = []
        for _ in range(3):
            dy = torch.full((m,), float("nan"), dtype=torch.float64, device="cuda")
            plan.execute(dx, dy)
            torch.cuda.synchronize()
            outs.append(dy.clone())
        got = outs[-1].cpu().numpy()
        err = np.abs(got - want)
        assert np.all(err <= np.maximum(np.maximum(lens - 1, 1) * 2.0 ** -53 * absum * 1.0001,
                                        2.0 ** -46 * np.abs(want)))
        if fixed == 2 or (fixed == 1 and unit == P.CUDA_CORE):
            assert torch.equal(outs[0], outs[1]) and torch.equal(outs[1], outs[2])
        dz = torch.zeros(n, dtype=torch.float64, device="cuda")
        dy = torch.full((m,), float("nan"), dtype=torch.float64, device="cuda")
        plan.execute(dz, dy)
        torch.cuda.synchronize()
        assert (dy == 0).all()
    finally:
        plan.close()


@pytest.mark.parametrize("unit", UNITS)
def test_colsort_cta_shapes_bit_identical(cuda, unit):
    """K17 on the 64-bit grid: every CTA shape (plain and software-pipelined
    loops, 384-1024 threads) and both thread-unit widths (one entry, or two
    paired entries per thread) add the same integer products, so the results
    are bit-identical; the tensor core's two quadrant DMMA give each product
    RN(val * x), so its grid rows equal the CUDA core's (rows the FP64 row
    kernels re-sum differ within the FP64 summation bound)."""
    import torch

    m = n = 150000
    rp, col, val = O.gen_band_csr(m, 0, n, 16, 20000, 9)
    x = O.fill_uniform(n, 9, 4, 0, 1)
    want = O.spmv_csr(rp, col, val, x)
    key = "spmv_colsort_tc_shape" if unit == P.TENSOR_CORE else "spmv_colsort_cc_shape"
    prev = [P.tuning_set("spmv_colsort_fixed", 2), P.tuning_set("spmv_plan_colsort", 1),
            P.tuning_set("spmv_colsort_vec", 4)]
    plans = {}
    try:
        for vec in (1, 2, 4):
            P.tuning_set("spmv_colsort_vec", vec)
            for u in UNITS:
                plans[(u, vec)] = P.SpmvPlan(rp, col, val, n, unit=u)
        P.tuning_set("spmv_colsort_vec", prev[2])
        dx = torch.from_numpy(x).cuda()
        outs = {}
        for vec in (1, 2, 4):
            for sh in (0, 7, 8, 10, 11, 13, 16):
                old = P.tuning_set(key, sh)
                try:
                    dy = torch.full((m,), float("nan"), dtype=torch.float64, device="cuda")
                    plans[(unit, vec)].execute(dx, dy)
                    torch.cuda.synchronize()
                    outs[(vec, sh)] = dy.cpu().numpy()
                finally:
                    P.tuning_set(key, old)
        ref = outs[(1, 0)]
        assert O.rel_err(ref, want) <= TOL
        for sh, y in outs.items():
            assert np.array_equal(y, ref), sh
        other = [u for u in UNITS if u != unit][0]
        dy = torch.full((m,), float("nan"), dtype=torch.float64, device="cuda")
        plans[(other, 4)].execute(dx, dy)
        torch.cuda.synchronize()
        yo = dy.cpu().numpy()
        same = yo == ref
        assert same.mean() > 0.99
        absum = np.array(
            [np.abs(val[rp[i]:rp[i + 1]] * x[col[rp[i]:rp[i + 1]]]).sum() for i in np.flatnonzero(~same)])
        assert np.all(np.abs(yo - ref)[~same] <= 2 * 16 * 2.0 ** -53 * absum)
    finally:
        for p in plans.values():
            p.close()
        P.tuning_set("spmv_colsort_fixed", prev[0])
        P.tuning_set("spmv_plan_colsort", prev[1])
        P.tuning_set("spmv_colsort_vec", prev[2])


@pytest.mark.parametrize("unit", UNITS)
@pytest.mark.parametrize("blocks", [0, 2400])
def test_colsort_fused_flagged_rows_match_row_kernel(cuda, unit, blocks):
    """Flagged rows re-summed inside the main kernel (spmv_colsort_fuse = 1:
    at the CTA's end for its first 4 blocks, at the block's end past that --
    2400 blocks on 296 CTAs exercise both) give the same bits as the separate
    FP64 row kernel (fuse = 0): the same rows, the same fixed summation order
    per unit.  Rows cancel (half of each row negates the other half) so that
    many rows are flagged."""
    import torch

    m = n = 300000
    rp, col, val = O.gen_band_csr(m, 0, n, 16, 30000, 12)
    val = val.copy()
    for i in range(0, m, 3):
        a, b = rp[i], rp[i + 1]
        h = (b - a) // 2
        val[a + h:a + 2 * h] = -val[a:a + h]
    x = O.fill_uniform(n, 12, 4, 0, 1)
    want = O.spmv_csr(rp, col, val, x)
    prev = [P.tuning_set("spmv_colsort_fixed", 2), P.tuning_set("spmv_plan_colsort", 1),
            P.tuning_set("spmv_plan_colsort_blocks", blocks)]
    try:
        plan = P.SpmvPlan(rp, col, val, n, unit=unit)
    finally:
        P.tuning_set("spmv_plan_colsort_blocks", prev[2])
    try:
        assert plan.layout() == "colsort"
        dx = torch.from_numpy(x).cuda()
        outs = []
        for fuse in (1, 0, 1):
            old = P.tuning_set("spmv_colsort_fuse", fuse)
            try:
                dy = torch.full((m,), float("nan"), dtype=torch.float64, device="cuda")
                plan.execute(dx, dy)
                torch.cuda.synchronize()
                outs.append(dy.cpu().numpy())
            finally:
                P.tuning_set("spmv_colsort_fuse", old)
        assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])
        assert O.rel_err(outs[0], want) <= TOL
    finally:
        plan.close()
        P.tuning_set("spmv_colsort_fixed", prev[0])
        P.tuning_set("spmv_plan_colsort", prev[1])


@pytest.mark.parametrize("unit", UNITS)
@pytest.mark.parametrize("colsort", [1, 0])
def test_plan_execute_host_async_stream(cuda, unit, colsort):
    """rl_spmv_plan_execute_host_async: a stream of independent vectors whose
    calls overlap on the device slots gives, per call, the bits of a
    synchronous execute_host on the same x (three device slots, seven calls); a synchronous call after async
    ones waits for them; wait() with nothing in flight returns."""
    import torch

    m = n = 200000
    rp, col, val = O.gen_band_csr(m, 0, n, 16, 30000, 21)
    prev = P.tuning_set("spmv_plan_colsort", colsort)
    try:
        plan = P.SpmvPlan(rp, col, val, n, unit=unit)
    finally:
        P.tuning_set("spmv_plan_colsort", prev)
    try:
        assert plan.layout() == ("colsort" if colsort else "csr")
        plan.wait()
        xs = [torch.from_numpy(O.fill_uniform(n, 30 + r, 4, 0, 1)).pin_memory() for r in range(3)]
        ys = [torch.full((m,), float("nan"), dtype=torch.float64).pin_memory() for _ in range(7)]
        for k in range(7):
            plan.execute_host_async(xs[k % 3], ys[k])
        plan.wait()
        for k in range(7):
            want = torch.empty(m, dtype=torch.float64).pin_memory()
            plan.execute_host(xs[k % 3], want)
            assert torch.equal(ys[k], want), k
            assert O.rel_err(ys[k].numpy(), O.spmv_csr(rp, col, val, xs[k % 3].numpy())) <= TOL
        y_sync = torch.empty(m, dtype=torch.float64).pin_memory()
        plan.execute_host_async(xs[0], ys[0])
        plan.execute_host(xs[1], y_sync)  # waits for the async call first
        assert torch.equal(ys[0], ys[3]) and torch.equal(y_sync, ys[1])
    finally:
        plan.close()
