"""Out-of-bounds write detection (compute-sanitizer is unavailable on this
pool): every output lives inside a larger device buffer whose margins hold a
sentinel; after the kernel the margins must be bit-identical.  Shapes are
chosen to end mid-vector / mid-tile so any overrun of a vectorised or tiled
store lands in a margin."""
import numpy as np
import pytest

import oracle as O
import paper_2502_16851_b200 as P

pytestmark = pytest.mark.gpu

UNITS = [P.CUDA_CORE, P.TENSOR_CORE]
MARGIN = 4096  # doubles on each side
SENTINEL = 1234.5678


def _guarded(torch, n):
    buf = torch.full((n + 2 * MARGIN,), SENTINEL, dtype=torch.float64, device="cuda")
    return buf, buf[MARGIN:MARGIN + n]


def _margins_intact(buf):
    b = buf.cpu().numpy()
    return np.all(b[:MARGIN] == SENTINEL) and np.all(b[-MARGIN:] == SENTINEL)


@pytest.mark.parametrize("unit", UNITS)
@pytest.mark.parametrize("n", [1, 3, 255, 257, 100003])
def test_guard_scale(cuda, unit, n):
    import torch

    b = torch.from_numpy(np.random.default_rng(n).uniform(-1, 1, n)).cuda()
    buf, a = _guarded(torch, n)
    P.scale(a, b, 2.0, unit=unit)
    torch.cuda.synchronize()
    assert _margins_intact(buf)
    assert O.bit_mismatches(a.cpu().numpy(), O.scale(b.cpu().numpy(), 2.0)) == 0


@pytest.mark.parametrize("unit", UNITS)
@pytest.mark.parametrize("m", [1, 7, 1001, 8195])
def test_guard_spmv_and_gemv(cuda, unit, m):
    import torch

    n = m + 5
    rp, col, val = O.gen_band_csr(m, 0, n, 3, 4, 9)
    x = np.random.default_rng(m).uniform(-1, 1, n)
    d = [torch.from_numpy(t).cuda() for t in (rp, col, val, x)]
    buf, y = _guarded(torch, m)
    P.spmv_csr(d[0], d[1], d[2], d[3], y, unit=unit)
    torch.cuda.synchronize()
    assert _margins_intact(buf)
    assert O.rel_err(y.cpu().numpy(), O.spmv_csr(rp, col, val, x)) <= 1e-12
    A = np.random.default_rng(m + 1).uniform(-1, 1, (m, 37))
    xg = np.random.default_rng(m + 2).uniform(-1, 1, 37)
    buf2, yg = _guarded(torch, m)
    P.gemv(torch.from_numpy(A).cuda(), torch.from_numpy(xg).cuda(), yg, unit=unit)
    torch.cuda.synchronize()
    assert _margins_intact(buf2)
    assert O.rel_err(yg.cpu().numpy(), O.gemv(A, xg)) <= 1e-12


@pytest.mark.parametrize("unit", UNITS)
@pytest.mark.parametrize("preset,shape", [
    ("2d5pt", (66, 130)), ("2d5pt", (17, 36)), ("2d9pt", (40, 70)), ("2d13pt", (41, 72)),
    ("2d49pt", (35, 74)), ("3d7pt", (11, 18, 66)), ("3d27pt", (10, 17, 34)),
])
def test_guard_stencils(cuda, unit, preset, shape):
    """u and v are views into guarded buffers (16-byte aligned, so the TMA
    paths run); the margins past both ends of v must survive."""
    import torch

    r = P.stencil_preset(preset)[2]
    u0 = O.stencil_init(shape, r, 3)
    n = u0.size
    bu, u = _guarded(torch, n)
    bv, v = _guarded(torch, n)
    u.copy_(torch.from_numpy(u0.ravel()))
    v.copy_(u)
    uu, vv = u.view(shape), v.view(shape)
    P.stencil(preset, uu, vv, 1, unit=unit)
    torch.cuda.synchronize()
    assert _margins_intact(bv) and _margins_intact(bu)
    assert O.rel_err(vv.cpu().numpy(), O.stencil(preset, u0, 1)) <= 1e-12


@pytest.mark.parametrize("t", [2, 5])
def test_guard_temporal(cuda, t):
    import torch

    shape = (70, 134)
    u0 = O.stencil_init(shape, 1, 4)
    n = u0.size
    bu, u = _guarded(torch, n)
    bv, v = _guarded(torch, n)
    u.copy_(torch.from_numpy(u0.ravel()))
    v.copy_(u)
    _, out = P.stencil_temporal("2d5pt", u.view(shape), v.view(shape), t, t)
    torch.cuda.synchronize()
    assert _margins_intact(bv) and _margins_intact(bu)
    assert O.rel_err(out.cpu().numpy(), O.stencil("2d5pt", u0, t)) <= 1e-12
