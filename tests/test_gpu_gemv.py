"""GPU parity: dense GEMV (next row #4) vs the CPU oracle, both units."""
import numpy as np
import pytest

import oracle as O
import paper_2502_16851_b200 as P




@pytest.mark.gpu
@pytest.mark.parametrize("unit", [P.CUDA_CORE, P.TENSOR_CORE])
@pytest.mark.parametrize("m,n", [(1, 1), (7, 13), (64, 128), (1000, 1003), (300, 4096), (4097, 512)])
def test_gemv(cuda, unit, m, n):
    import torch

    rng = np.random.default_rng(m * 7 + n)
    A = rng.uniform(-1, 1, (m, n))
    x = rng.uniform(-1, 1, n)
    dA, dx = torch.from_numpy(A).cuda(), torch.from_numpy(x).cuda()
    dy = torch.full((m,), float("nan"), dtype=torch.float64, device="cuda")
    kc = P.gemv(dA, dx, dy, unit=unit)
    torch.cuda.synchronize()
    assert O.rel_err(dy.cpu().numpy(), O.gemv(A, x)) <= 1e-12
    assert kc == P.gemv_model(m, n)


def test_gemv_oracle_vs_numpy():
    rng = np.random.default_rng(0)
    A, x = rng.uniform(-1, 1, (300, 257)), rng.uniform(-1, 1, 257)
    assert O.rel_err(O.gemv(A, x), A @ x) < 1e-14
