"""Every kernel variant once at small, edge-case sizes (for compute-sanitizer).

  compute-sanitizer --tool memcheck python tools/sanitize_smoke.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2502_16851_b200 as P  # noqa: E402


def main():
    for unit in (P.CUDA_CORE, P.TENSOR_CORE):
        for n in (1, 255, 257, 4099):
            b = torch.empty(n, dtype=torch.float64, device="cuda")
            P.fill_uniform(b, 1, 1, 0, 1)
            a = torch.empty_like(b)
            P.scale(a, b, 3.0, unit=unit)
        base = torch.zeros(1000, dtype=torch.float64, device="cuda")
        P.scale(base[3:503], base[1:501], 2.0, unit=unit)
        for m, k, hb in ((100, 16, 30), (1000, 7, 200), (3000, 16, 65536)):
            rp, col, val = O.gen_band_csr(m, 0, m, k, hb, 2)
            x = O.fill_uniform(m, 2, 4, 0, 1)
            d = [torch.from_numpy(t).cuda() for t in (rp, col, val, x)]
            y = torch.empty(m, dtype=torch.float64, device="cuda")
            P.spmv_csr(d[0], d[1], d[2], d[3], y, unit=unit)
        rng = np.random.default_rng(1)
        lens = rng.integers(0, 40, 257)
        rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
        col = np.concatenate([np.sort(rng.choice(300, l, replace=False)) for l in lens]).astype(np.int32)
        val = rng.uniform(-1, 1, rp[-1])
        d = [torch.from_numpy(t).cuda() for t in (rp, col, val, rng.uniform(-1, 1, 300))]
        y = torch.empty(257, dtype=torch.float64, device="cuda")
        P.spmv_csr(d[0], d[1], d[2], d[3], y, unit=unit)
        for preset, shapes in (("2d5pt", [(3, 3), (17, 33), (70, 130), (33, 258)]),
                               ("3d7pt", [(3, 3, 3), (9, 17, 33), (12, 20, 130)]),
                               ("3d27pt", [(5, 6, 7), (10, 17, 66), (9, 33, 128)])):
            for shape in shapes:
                u = torch.empty(shape, dtype=torch.float64, device="cuda")
                P.stencil_init(u, 1, 3)
                v = u.clone()
                P.stencil(preset, u, v, 2, unit=unit)
        w = np.random.default_rng(2).uniform(0, 1, 27)
        u = torch.empty((10, 17, 66), dtype=torch.float64, device="cuda")
        P.stencil_init(u, 1, 3)
        P.stencil("3d27pt", u, u.clone(), 1, weights=w / w.sum(), unit=unit)
    for preset, shape in (("2d9pt", (20, 30)), ("2d13pt", (20, 30)), ("2d49pt", (20, 30))):
        u = torch.empty(shape, dtype=torch.float64, device="cuda")
        P.stencil_init(u, P.stencil_preset(preset)[2], 3)
        P.stencil(preset, u, u.clone(), 1)
    torch.cuda.synchronize()
    print("sanitize smoke ok")


if __name__ == "__main__":
    main()
