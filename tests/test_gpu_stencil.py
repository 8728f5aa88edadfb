"""GPU parity: Jacobi stencils (K5-K10) vs the CPU oracle.

Bar (BASELINE.json north_star): 1e-12 norm-wise relative error.  The
Dirichlet ring must be untouched (bit-exact), which also checks that no
kernel writes outside the interior.
"""
import functools

import numpy as np
import pytest

import oracle as O
import paper_2502_16851_b200 as P

pytestmark = pytest.mark.gpu

UNITS = [P.CUDA_CORE, P.TENSOR_CORE]
TOL = 1e-12


def _run(torch, preset, u0, steps, unit, weights=None):
    u = torch.from_numpy(u0.copy()).cuda()
    v = torch.from_numpy(u0.copy()).cuda()
    kc = P.stencil(preset, u, v, steps, weights=weights, unit=unit)
    torch.cuda.synchronize()
    out = (u if steps % 2 == 0 else v).cpu().numpy()
    return out, kc


def _ring_mask(shape, r):
    m = np.zeros(shape, bool)
    if len(shape) == 2:
        m[:r, :] = m[-r:, :] = m[:, :r] = m[:, -r:] = True
    else:
        m[:r] = m[-r:] = True
        m[:, :r] = m[:, -r:] = True
        m[:, :, :r] = m[:, :, -r:] = True
    return m


SHAPES_2D = [(3, 3), (5, 7), (17, 33), (64, 128), (130, 258), (257, 129), (301, 515), (1030, 1026)]
SHAPES_3D = [(3, 3, 3), (5, 6, 7), (10, 17, 33), (34, 20, 130), (20, 70, 256), (40, 40, 64)]


@pytest.mark.parametrize("shape", SHAPES_2D)
@pytest.mark.parametrize("unit", UNITS)
@pytest.mark.parametrize("steps", [1, 4])
def test_2d5pt(cuda, shape, unit, steps):
    import torch

    u0 = O.stencil_init(shape, 1, 7)
    out, kc = _run(torch, "2d5pt", u0, steps, unit)
    ref = O.stencil("2d5pt", u0, steps)
    assert O.rel_err(out, ref) <= TOL
    ring = _ring_mask(shape, 1)
    assert O.bit_mismatches(out[ring], u0[ring]) == 0
    pts = (shape[0] - 2) * (shape[1] - 2)
    assert (kc.work_flops, kc.traffic_bytes) == (10 * pts * steps, 16 * pts * steps)


@pytest.mark.parametrize("preset", ["3d7pt", "3d27pt"])
@pytest.mark.parametrize("shape", SHAPES_3D)
@pytest.mark.parametrize("unit", UNITS)
@pytest.mark.parametrize("steps", [1, 3])
def test_3d(cuda, preset, shape, unit, steps):
    import torch

    u0 = O.stencil_init(shape, 1, 13)
    out, kc = _run(torch, preset, u0, steps, unit)
    ref = O.stencil(preset, u0, steps)
    assert O.rel_err(out, ref) <= TOL
    ring = _ring_mask(shape, 1)
    assert O.bit_mismatches(out[ring], u0[ring]) == 0
    pts = (shape[0] - 2) * (shape[1] - 2) * (shape[2] - 2)
    npts = 7 if preset == "3d7pt" else 27
    assert kc.traffic_bytes == 16 * pts * steps and kc.work_flops == 2 * npts * pts * steps


@pytest.mark.parametrize("unit", UNITS)
def test_3d27pt_general_weights(cuda, unit):
    """Weights without the |dx|+|dy|+|dz| structure take the general path."""
    import torch

    rng = np.random.default_rng(5)
    w = rng.uniform(0, 1, 27)
    w /= w.sum()
    shape = (18, 21, 70)
    u0 = O.stencil_init(shape, 1, 3)
    out, _ = _run(torch, "3d27pt", u0, 2, unit, weights=w)
    assert O.rel_err(out, O.stencil("3d27pt", u0, 2, w)) <= TOL


@pytest.mark.parametrize("unit", UNITS)
@pytest.mark.parametrize("preset", ["2d5pt", "3d7pt"])
def test_custom_weights(cuda, unit, preset):
    import torch

    npts = 5 if preset == "2d5pt" else 7
    w = np.linspace(0.05, 0.3, npts)
    shape = (66, 130) if preset == "2d5pt" else (12, 19, 68)
    u0 = O.stencil_init(shape, 1, 8)
    out, _ = _run(torch, preset, u0, 3, unit, weights=w)
    assert O.rel_err(out, O.stencil(preset, u0, 3, w)) <= TOL


@pytest.mark.parametrize("preset,shape", [("2d9pt", (40, 77)), ("2d13pt", (41, 71)), ("2d49pt", (33, 45))])
def test_other_presets_odd_nx(cuda, preset, shape):
    """Odd nx: the CUDA core runs the generic kernel; the tensor-core
    kernels need 16-byte rows and refuse."""
    import torch

    r = P.stencil_preset(preset)[2]
    u0 = O.stencil_init(shape, r, 21)
    out, _ = _run(torch, preset, u0, 2, P.CUDA_CORE)
    assert O.rel_err(out, O.stencil(preset, u0, 2)) <= TOL
    with pytest.raises(P.RooflensError) as e:
        _run(torch, preset, u0, 1, P.TENSOR_CORE)
    assert e.value.kind == "ValidationError"


SHAPES_R = [(7, 8), (9, 10), (40, 70), (33, 64), (130, 200), (301, 258), (520, 1030)]


@pytest.mark.parametrize("unit", UNITS)
@pytest.mark.parametrize("preset", ["2d9pt", "2d13pt", "2d49pt"])
@pytest.mark.parametrize("shape", SHAPES_R)
def test_other_presets_tma(cuda, unit, preset, shape):
    """2d9pt / 2d13pt / 2d49pt through the TMA kernels (even nx), both units:
    parity with the oracle and an untouched radius-R Dirichlet ring."""
    import torch

    r = P.stencil_preset(preset)[2]
    u0 = O.stencil_init(shape, r, 5)
    steps = 3
    out, kc = _run(torch, preset, u0, steps, unit)
    ref = O.stencil(preset, u0, steps)
    assert O.rel_err(out, ref) <= TOL
    ring = _ring_mask(shape, r)
    assert np.array_equal(out[ring], u0[ring])
    npts = int(np.prod([s - 2 * r for s in shape])) if min(shape) > 2 * r else 0
    assert kc.traffic_bytes == 16 * npts * steps


@pytest.mark.parametrize("unit", UNITS)
@pytest.mark.parametrize("preset", ["2d9pt", "2d13pt", "2d49pt"])
def test_other_presets_custom_weights_and_range(cuda, unit, preset):
    """Non-symmetric weights (every tap distinct) and a partial row sweep."""
    import torch

    npts, r = P.stencil_preset(preset)[1], P.stencil_preset(preset)[2]
    w = np.random.default_rng(2).uniform(-0.2, 0.3, npts)
    shape = (150, 196)
    u0 = O.stencil_init(shape, r, 9)
    out, _ = _run(torch, preset, u0, 2, unit, weights=w)
    assert O.rel_err(out, O.stencil(preset, u0, 2, w)) <= TOL
    ref1 = O.stencil(preset, u0, 1, w)
    u = torch.from_numpy(u0).cuda()
    v = torch.zeros_like(u)
    P.stencil_sweep(preset, u, v, 37, 111, weights=w, unit=unit)
    torch.cuda.synchronize()
    got = v.cpu().numpy()
    assert O.rel_err(got[37:111, r:-r], ref1[37:111, r:-r]) <= TOL
    assert not got[:37].any() and not got[111:].any()


@pytest.mark.parametrize("unit", UNITS)
def test_sweep_partial_range(cuda, unit):
    """rl_stencil_sweep over a plane range writes exactly those planes."""
    import torch

    shape = (30, 24, 64)
    u0 = O.stencil_init(shape, 1, 4)
    ref = O.stencil("3d7pt", u0, 1)
    u = torch.from_numpy(u0).cuda()
    v = torch.zeros_like(u)
    P.stencil_sweep("3d7pt", u, v, 7, 19, unit=unit)
    torch.cuda.synchronize()
    out = v.cpu().numpy()
    assert O.rel_err(out[7:19], ref[7:19]) <= TOL
    assert np.all(out[:7] == 0) and np.all(out[19:] == 0)


def test_stencil_generator_matches_oracle(cuda):
    import torch

    for shape in [(130, 67), (9, 33, 65)]:
        u = torch.empty(shape, dtype=torch.float64, device="cuda")
        P.stencil_init(u, 1, 77)
        torch.cuda.synchronize()
        assert O.bit_mismatches(u.cpu().numpy(), O.stencil_init(shape, 1, 77)) == 0


@functools.lru_cache(maxsize=3)
def _full_run_oracle(preset):
    """The oracle over a whole BASELINE run: 100 timesteps of 16384^2 (2D) or
    50 of 512^3 (3D) -- a few seconds on the box's cores."""
    shape, steps = ((16384, 16384), 100) if preset == "2d5pt" else ((512, 512, 512), 50)
    return shape, steps, O.stencil(preset, O.stencil_init(shape, 1, 2025), steps)


@pytest.mark.slow
@pytest.mark.parametrize("preset", ["2d5pt", "3d7pt", "3d27pt"])
@pytest.mark.parametrize("variant", ["cc", "tc", "tc_pure"])
def test_full_baseline_run(cuda, preset, variant):
    """BASELINE configs[2..4] end to end: the full grid AND the full timestep
    count (100 for 2D, 50 for 3D) against the oracle at 1e-12, ring untouched;
    tc_pure is the full banded DMMA form (no DFMA taps)."""
    import torch

    shape, steps, ref = _full_run_oracle(preset)
    unit = P.CUDA_CORE if variant == "cc" else P.TENSOR_CORE
    keys = {"stencil_tc2d_hybrid": 0, "stencil_tc3d_hybrid": 0} if variant == "tc_pure" else {}
    prev = {k: P.tuning_set(k, v) for k, v in keys.items()}
    try:
        u = torch.empty(shape, dtype=torch.float64, device="cuda")
        P.stencil_init(u, 1, 2025)
        v = u.clone()
        P.stencil(preset, u, v, steps, unit=unit)
        torch.cuda.synchronize()
    finally:
        for k, val in prev.items():
            P.tuning_set(k, val)
    out = (u if steps % 2 == 0 else v).cpu().numpy()
    del u, v
    assert O.rel_err(out, ref) <= TOL
    ring = _ring_mask(shape, 1)
    assert not out[ring].any()


@pytest.mark.parametrize("shape", [(64, 128), (130, 258), (301, 516), (1030, 1026)])
@pytest.mark.parametrize("steps", [1, 2, 5, 8])
def test_2d5pt_temporal_depth2(cuda, shape, steps):
    """Temporal blocking (t = 2) equals `steps` single timesteps."""
    import torch

    u0 = O.stencil_init(shape, 1, 19)
    u = torch.from_numpy(u0.copy()).cuda()
    v = torch.from_numpy(u0.copy()).cuda()
    kc, out = P.stencil_temporal("2d5pt", u, v, steps, 2)
    torch.cuda.synchronize()
    ref = O.stencil("2d5pt", u0, steps)
    got = out.cpu().numpy()
    assert O.rel_err(got, ref) <= TOL
    ring = _ring_mask(shape, 1)
    assert O.bit_mismatches(got[ring], u0[ring]) == 0
    pts = (shape[0] - 2) * (shape[1] - 2)
    fused, rem = steps // 2, steps % 2
    assert kc.traffic_bytes == 16 * pts * (fused + rem)
    assert kc.work_flops == pts * (fused * 20 + rem * 10)


@pytest.mark.parametrize("t", [2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("shape", [(20, 24), (65, 130), (301, 517), (513, 1026)])
def test_2d5pt_temporal_depth_t(cuda, t, shape):
    """Temporal depth t (register kernel, stencil_tb.cu) equals t * k single
    timesteps, with custom weights, odd and even nx (odd depths only run the
    scalar-load path), and an untouched Dirichlet ring."""
    import torch

    if t % 2 == 0 and shape[1] % 2:
        pytest.skip("even depths need 16-byte rows")
    u0 = O.stencil_init(shape, 1, 23)
    w = np.array([0.4, 0.2, 0.1, 0.17, 0.13])
    steps = 2 * t + 1
    u = torch.from_numpy(u0.copy()).cuda()
    v = torch.from_numpy(u0.copy()).cuda()
    kc, out = P.stencil_temporal("2d5pt", u, v, steps, t, weights=w)
    torch.cuda.synchronize()
    ref = O.stencil("2d5pt", u0, steps, w)
    got = out.cpu().numpy()
    assert O.rel_err(got, ref) <= TOL
    ring = _ring_mask(shape, 1)
    assert O.bit_mismatches(got[ring], u0[ring]) == 0
    pts = (shape[0] - 2) * (shape[1] - 2)
    assert kc.traffic_bytes == 16 * pts * 3  # 2 fused sweeps + 1 single step


@pytest.mark.parametrize("t", [2, 3, 4])
@pytest.mark.parametrize("shape", [(9, 10, 11), (20, 24, 68), (33, 40, 70), (64, 50, 97), (37, 130, 126),
                                   (70, 29, 200)])
def test_3d7pt_temporal_depth_t(cuda, t, shape):
    """3d7pt temporal depth t equals single timesteps; custom weights; the
    Dirichlet shell stays bit-exact.  Even nx: the register-blocked TMA kernel
    (stencil_tb3r.cu); odd nx: the z-column kernel (stencil_tb3.cu)."""
    import torch

    u0 = O.stencil_init(shape, 1, 29)
    w = np.array([0.3, 0.12, 0.08, 0.11, 0.14, 0.1, 0.15])
    steps = 2 * t + 1
    u = torch.from_numpy(u0.copy()).cuda()
    v = torch.from_numpy(u0.copy()).cuda()
    kc, out = P.stencil_temporal("3d7pt", u, v, steps, t, weights=w)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    assert O.rel_err(got, O.stencil("3d7pt", u0, steps, w)) <= TOL
    ring = _ring_mask(shape, 1)
    assert O.bit_mismatches(got[ring], u0[ring]) == 0
    assert kc.traffic_bytes == 16 * int(np.prod([s - 2 for s in shape])) * 3


@pytest.mark.parametrize("t", [2, 3, 4])
@pytest.mark.parametrize("shape", [(9, 10, 11), (20, 24, 68), (37, 130, 126), (70, 29, 200)])
@pytest.mark.parametrize("weights", ["default", "general"])
def test_3d27pt_temporal_depth_t(cuda, t, shape, weights):
    """3d27pt temporal depth t (stencil_tb3.cu, three partial-sum planes per
    level, weights from the parameter bank): equals single timesteps for the
    BASELINE class weights and for 27 unrelated weights; Dirichlet shell
    bit-exact; stencil_model(t) bytes."""
    import torch

    u0 = O.stencil_init(shape, 1, 31)
    w = None if weights == "default" else np.random.default_rng(t).uniform(0.0, 1.0 / 27, 27)
    steps = 2 * t + 1
    u = torch.from_numpy(u0.copy()).cuda()
    v = torch.from_numpy(u0.copy()).cuda()
    kc, out = P.stencil_temporal("3d27pt", u, v, steps, t, weights=w)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    assert O.rel_err(got, O.stencil("3d27pt", u0, steps, w)) <= TOL
    ring = _ring_mask(shape, 1)
    assert O.bit_mismatches(got[ring], u0[ring]) == 0
    pts = int(np.prod([s - 2 for s in shape]))
    assert kc.traffic_bytes == 16 * pts * 3 and kc.work_flops == pts * 54 * (2 * t + 1)


@pytest.mark.parametrize("t", [2, 3, 4])
@pytest.mark.parametrize("shape", [(20, 24), (65, 130), (130, 66), (301, 516), (1030, 1026)])
def test_2d5pt_temporal_tensor_core(cuda, t, shape):
    """2d5pt temporal depth t on the tensor core (stencil_tbtc.cu: overlapped
    64 x 64 tiles, each level the x-band-on-DMMA form) equals single
    timesteps with custom weights; tiles straddling the grid edge; Dirichlet
    ring bit-exact; stencil_model(t) bytes."""
    import torch

    u0 = O.stencil_init(shape, 1, 37)
    w = np.array([0.4, 0.2, 0.1, 0.17, 0.13])
    steps = 2 * t + 1
    u = torch.from_numpy(u0.copy()).cuda()
    v = torch.from_numpy(u0.copy()).cuda()
    kc, out = P.stencil_temporal("2d5pt", u, v, steps, t, weights=w, unit=P.TENSOR_CORE)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    assert O.rel_err(got, O.stencil("2d5pt", u0, steps, w)) <= TOL
    ring = _ring_mask(shape, 1)
    assert O.bit_mismatches(got[ring], u0[ring]) == 0
    pts = (shape[0] - 2) * (shape[1] - 2)
    assert kc.traffic_bytes == 16 * pts * 3


def test_temporal_depth_restrictions(cuda):
    import torch

    u = torch.zeros((20, 24, 64), dtype=torch.float64, device="cuda")
    with pytest.raises(P.RooflensError) as e:
        P.stencil_temporal("3d27pt", u, u.clone(), 10, 5)
    assert e.value.kind == "ValidationError"
    with pytest.raises(P.RooflensError) as e:
        P.stencil_temporal("3d7pt", u, u.clone(), 4, 2, unit=P.TENSOR_CORE)
    assert e.value.kind == "ValidationError"
    with pytest.raises(P.RooflensError) as e:
        P.stencil_temporal("3d7pt", u, u.clone(), 10, 5)
    assert e.value.kind == "ValidationError"
    with pytest.raises(P.RooflensError) as e:
        P.stencil_temporal("2d5pt", u[0], u[1].clone(), 4, 0)
    assert e.value.kind == "InvalidCount"
    with pytest.raises(P.RooflensError) as e:
        P.stencil_temporal("2d5pt", u[0], u[1].clone(), 18, 9)
    assert e.value.kind == "InvalidRange"
    with pytest.raises(P.RooflensError) as e:
        P.stencil_temporal("2d5pt", u[0], u[1].clone(), 10, 5, unit=P.TENSOR_CORE)
    assert e.value.kind == "ValidationError"
    with pytest.raises(P.RooflensError) as e:  # odd nx: no 16-byte rows for the box
        P.stencil_temporal("2d5pt", u[0, :, :63].contiguous(), u[1, :, :63].contiguous(), 4, 2,
                           unit=P.TENSOR_CORE)
    assert e.value.kind == "ValidationError"


@pytest.mark.parametrize("knobs", [
    {"stencil_tc3d_hybrid": 0, "stencil_tc3d_mode": 0},
    {"stencil_tc3d_hybrid": 0, "stencil_tc3d_mode": 3},
    {"stencil_tc3d_hybrid": 1},
    {"stencil_tc3d_hybrid": 1, "stencil_tch_tpw": 4, "stencil_tch_ctas_per_sm": 8},
    {"stencil_tc3d_hybrid": 1, "stencil_tch_tpw": 1, "stencil_tch_k8": 1},
    {"stencil_tc3d_hybrid": 1, "stencil_tch_tpw": 2, "stencil_tch_k8": 1, "stencil3d_balance": 0},
])
@pytest.mark.parametrize("preset", ["3d7pt", "3d27pt"])
@pytest.mark.parametrize("shape", [(10, 17, 66), (34, 20, 130), (40, 40, 64), (12, 70, 200)])
def test_3d_tensor_core_formulations(cuda, knobs, preset, shape):
    """Every 3D tensor-core formulation (full banded with 3 planes resident or
    one plane with partial sums; the x-band kernel st3d_tma_tch with its
    tiles-per-warp / K-window / row-balance knobs) matches the oracle, for
    class and general 27pt weights."""
    import torch

    prev = {k: P.tuning_set(k, v) for k, v in knobs.items()}
    try:
        u0 = O.stencil_init(shape, 1, 23)
        out, _ = _run(torch, preset, u0, 3, P.TENSOR_CORE)
        assert O.rel_err(out, O.stencil(preset, u0, 3)) <= TOL
        if preset == "3d27pt":
            w = np.random.default_rng(7).uniform(0, 1, 27)
            w /= w.sum()
            out, _ = _run(torch, preset, u0, 2, P.TENSOR_CORE, weights=w)
            assert O.rel_err(out, O.stencil(preset, u0, 2, w)) <= TOL
    finally:
        for k, v in prev.items():
            P.tuning_set(k, v)


@pytest.mark.parametrize("hybrid", [0, 1])
@pytest.mark.parametrize("shape", [(70, 132), (130, 260), (33, 1030)])
def test_2d_tensor_core_formulations(cuda, hybrid, shape):
    """2d5pt tensor core: the x-band kernel (st2d_tma_tch) and the full banded
    kernel match the oracle."""
    import torch

    prev = P.tuning_set("stencil_tc2d_hybrid", hybrid)
    try:
        u0 = O.stencil_init(shape, 1, 29)
        out, _ = _run(torch, "2d5pt", u0, 3, P.TENSOR_CORE)
        assert O.rel_err(out, O.stencil("2d5pt", u0, 3)) <= TOL
    finally:
        P.tuning_set("stencil_tc2d_hybrid", prev)


@pytest.mark.parametrize("balance", [0, 1])
@pytest.mark.parametrize("preset", ["3d7pt", "3d27pt"])
def test_3d_row_balanced_tiles(cuda, balance, preset):
    """Row-balanced tiles (rows cut into nty tiles of 13-14 rows at 512 rows;
    here 200 rows -> tiles of <= 16) match the oracle on both units."""
    import torch

    prev = P.tuning_set("stencil3d_balance", balance)
    try:
        u0 = O.stencil_init((6, 200, 256), 1, 31)
        for unit in (P.CUDA_CORE, P.TENSOR_CORE):
            out, _ = _run(torch, preset, u0, 2, unit)
            assert O.rel_err(out, O.stencil(preset, u0, 2)) <= TOL
    finally:
        P.tuning_set("stencil3d_balance", prev)


@pytest.mark.parametrize("shape_knob", [0, 1, 2])
@pytest.mark.parametrize("t", [2, 3, 4])
@pytest.mark.parametrize("chunks", [1, 3, 7])
def test_3d7pt_temporal_z_chunks(cuda, t, chunks, shape_knob):
    """The register-blocked 3D kernel split into z chunks (each chunk
    re-loads its 2t-plane cone) gives the same result as single steps."""
    import torch

    shape = (45, 66, 134)
    u0 = O.stencil_init(shape, 1, 31)
    u = torch.from_numpy(u0.copy()).cuda()
    v = torch.from_numpy(u0.copy()).cuda()
    P.tuning_set("stencil_tb3_chunks", chunks)
    P.tuning_set("stencil_tb3_shape", shape_knob)
    try:
        _, out = P.stencil_temporal("3d7pt", u, v, 2 * t, t)
        torch.cuda.synchronize()
    finally:
        P.tuning_set("stencil_tb3_chunks", 0)
        P.tuning_set("stencil_tb3_shape", 0)
    got = out.cpu().numpy()
    assert O.rel_err(got, O.stencil("3d7pt", u0, 2 * t)) <= TOL
    ring = _ring_mask(shape, 1)
    assert O.bit_mismatches(got[ring], u0[ring]) == 0


@pytest.mark.parametrize("tma_from", [2, 0])
@pytest.mark.parametrize("t", [2, 3, 4, 5, 8])
@pytest.mark.parametrize("shape", [(70, 134), (131, 258), (45, 64)])
def test_2d5pt_temporal_tma_ring(cuda, tma_from, t, shape):
    """2d5pt temporal depth t with the rows streamed through the per-warp TMA
    ring (odd t reads the unaligned column pair) or the register queue."""
    import torch

    u0 = O.stencil_init(shape, 1, 41)
    u = torch.from_numpy(u0.copy()).cuda()
    v = torch.from_numpy(u0.copy()).cuda()
    P.tuning_set("stencil_tb_tma", tma_from)
    try:
        _, out = P.stencil_temporal("2d5pt", u, v, 2 * t + 1, t)
        torch.cuda.synchronize()
    finally:
        P.tuning_set("stencil_tb_tma", 4)
    got = out.cpu().numpy()
    assert O.rel_err(got, O.stencil("2d5pt", u0, 2 * t + 1)) <= TOL
    ring = _ring_mask(shape, 1)
    assert O.bit_mismatches(got[ring], u0[ring]) == 0
