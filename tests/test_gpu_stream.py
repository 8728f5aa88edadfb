"""GPU parity: STREAM Scale (K1 CUDA core, K2 tensor core) vs the CPU oracle.

Bar (BASELINE.json north_star): bit-exact.  Inputs are generated on the
device by the C-ABI generator and checked bit-for-bit against the oracle's
own generator first, so the parity comparison is over identical inputs.
"""
import numpy as np
import pytest

import oracle as O
import paper_2502_16851_b200 as P

pytestmark = pytest.mark.gpu

UNITS = [P.CUDA_CORE, P.TENSOR_CORE]


def _dev_uniform(torch, n, seed, sid, kind):
    t = torch.empty(n, dtype=torch.float64, device="cuda")
    P.fill_uniform(t, seed, sid, 0, kind)
    return t


@pytest.mark.parametrize("n", [1, 3, 4, 31, 255, 256, 257, 1000, 4099, 65536 + 17, 1 << 20])
@pytest.mark.parametrize("unit", UNITS)
def test_scale_bit_exact_sizes(cuda, n, unit):
    import torch

    b = _dev_uniform(torch, n, 11, 1, 1)
    bh = O.fill_uniform(n, 11, 1, 0, 1)
    assert O.bit_mismatches(b.cpu().numpy(), bh) == 0, "device generator != oracle generator"
    a = torch.full_like(b, float("nan"))
    kc = P.scale(a, b, 3.0, unit=unit)
    torch.cuda.synchronize()
    ref = O.scale(bh, 3.0)
    assert O.bit_mismatches(a.cpu().numpy(), ref) == 0
    assert (kc.work_flops, kc.traffic_bytes) == (n, 16 * n)


@pytest.mark.parametrize("offset", [1, 2, 3, 5])
@pytest.mark.parametrize("unit", UNITS)
def test_scale_unaligned_views(cuda, offset, unit):
    import torch

    n = 10007
    base_b = _dev_uniform(torch, n + 8, 5, 1, 1)
    base_a = torch.zeros(n + 8, dtype=torch.float64, device="cuda")
    b = base_b[offset:offset + n]
    a = base_a[(offset + 1) % 4: (offset + 1) % 4 + n]
    P.scale(a, b, -2.5, unit=unit)
    torch.cuda.synchronize()
    ref = O.scale(np.ascontiguousarray(b.cpu().numpy()), -2.5)
    assert O.bit_mismatches(a.cpu().numpy(), ref) == 0
    # nothing outside the destination view was written
    lo = (offset + 1) % 4
    assert torch.all(base_a[:lo] == 0) and torch.all(base_a[lo + n:] == 0)


@pytest.mark.parametrize("unit", UNITS)
def test_scale_special_values(cuda, unit):
    """Finite specials are exact on both units; CC also matches q*b for
    -0/inf/nan.  The TC form A = B(qI) maps -0 to +0 and spreads non-finite
    inputs within a 4-element fragment row (documented limitation)."""
    import torch

    vals = np.array([0.0, 1.0, -1.0, 5e-324, 2.2250738585072014e-308, 1.7976931348623157e308 / 4,
                     -3.5, 1e-300, 123456.789] * 40, np.float64)
    b = torch.from_numpy(vals).cuda()
    a = torch.empty_like(b)
    P.scale(a, b, 3.0, unit=unit)
    torch.cuda.synchronize()
    assert O.bit_mismatches(a.cpu().numpy(), O.scale(vals, 3.0)) == 0
    if unit == P.CUDA_CORE:
        sp = np.array([-0.0, np.inf, -np.inf, np.nan] * 64, np.float64)
        b = torch.from_numpy(sp).cuda()
        a = torch.empty_like(b)
        P.scale(a, b, 3.0, unit=unit)
        torch.cuda.synchronize()
        assert O.bit_mismatches(a.cpu().numpy(), O.scale(sp, 3.0)) == 0


@pytest.mark.slow
@pytest.mark.parametrize("unit", UNITS)
def test_scale_full_config_bit_exact(cuda, unit):
    """BASELINE configs[0]: n = 2^27, q = 3, b ~ U[-1,1)."""
    import torch

    n = 1 << 27
    b = _dev_uniform(torch, n, 2025, 1, 1)
    a = torch.empty_like(b)
    kc = P.scale(a, b, 3.0, unit=unit)
    torch.cuda.synchronize()
    bh = O.fill_uniform(n, 2025, 1, 0, 1)
    assert O.bit_mismatches(b.cpu().numpy(), bh) == 0
    assert O.bit_mismatches(a.cpu().numpy(), O.scale(bh, 3.0)) == 0
    assert kc.traffic_bytes == 2147483648 and kc.work_flops == 134217728


def test_scale_errors(cuda):
    import torch

    b = torch.zeros(8, dtype=torch.float64, device="cuda")
    with pytest.raises(P.RooflensError) as e:
        P.scale(b.clone(), b, 1.0, precision=P.FP32)
    assert e.value.kind == "ValidationError"
    with pytest.raises(P.RooflensError) as e:
        P.scale(b[:0], b[:0], 1.0)
    assert e.value.kind == "InvalidCount"
