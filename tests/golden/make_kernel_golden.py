"""Generate tests/golden/kernels.npz: small golden input/output vectors for the
executing kernels, computed WITHOUT this repo's oracle (oracle/oracle.c) --
numpy for STREAM and the stencils (the equations of PAPER.md:147-151 and
211-215 written as array expressions), math.fsum for the SpMV row sums
(correctly rounded).  The reference ships no kernel and no
golden vectors, so these pin both the oracle
(tests/test_oracle.py) and the GPU kernels (tests/test_gpu_golden.py) to an
independent restatement.

    python tests/golden/make_kernel_golden.py
"""
import math
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def stencil_numpy(u0, offsets, weights, steps):
    """Jacobi sweeps on the interior (radius-1 box), Dirichlet ring kept."""
    u = u0.copy()
    nd = u.ndim
    inner = tuple(slice(1, s - 1) for s in u.shape)
    for _ in range(steps):
        v = u.copy()
        acc = np.zeros_like(u[inner])
        for off, w in zip(offsets, weights):
            sl = tuple(slice(1 + o, s - 1 + o) for o, s in zip(off, u.shape))
            acc = acc + w * u[sl]
        v[inner] = acc
        u = v
    return u


def main():
    rng = np.random.default_rng(20251020)
    out = {}
    # STREAM Scale: one rounding per element
    b = rng.uniform(-1, 1, 4099)
    out["scale_b"], out["scale_q"] = b, np.array(3.0)
    out["scale_a"] = 3.0 * b
    # SpMV: ragged rows (empty, long), sorted unique columns; fsum row sums
    m, n = 700, 900
    lens = rng.integers(0, 40, m)
    lens[::11] = 0
    lens[5] = 600
    rows = [np.sort(rng.choice(n, l, replace=False)) for l in lens]
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    col = np.concatenate(rows).astype(np.int32)
    val = rng.uniform(-1, 1, rp[-1])
    x = rng.uniform(-1, 1, n)
    prod = val * x[col]
    y = np.array([math.fsum(prod[rp[i]:rp[i + 1]]) for i in range(m)])
    out.update(spmv_rp=rp, spmv_col=col, spmv_val=val, spmv_x=x, spmv_y=y)
    # 2d5pt, BASELINE weights, 3 steps; offsets in canonical order (c, y-, y+, x-, x+)
    u2 = np.zeros((40, 52))
    u2[1:-1, 1:-1] = rng.uniform(0, 1, (38, 50))
    off2 = [(0, 0), (-1, 0), (1, 0), (0, -1), (0, 1)]
    w2 = [0.5, 0.125, 0.125, 0.125, 0.125]
    out["s2d_u0"], out["s2d_v"] = u2, stencil_numpy(u2, off2, w2, 3)
    # 3d7pt (c, z-, z+, y-, y+, x-, x+), 2 steps
    u3 = np.zeros((12, 14, 20))
    u3[1:-1, 1:-1, 1:-1] = rng.uniform(0, 1, (10, 12, 18))
    off7 = [(0, 0, 0), (-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0), (0, 0, -1), (0, 0, 1)]
    w7 = [0.4, 0.1, 0.1, 0.1, 0.1, 0.1, 0.1]
    out["s3d7_u0"], out["s3d7_v"] = u3, stencil_numpy(u3, off7, w7, 2)
    # 3d27pt: w = 1/(1 + |dx| + |dy| + |dz|) normalised (raw sum 10), canonical (dz, dy, dx) order, 2 steps
    off27 = [(dz, dy, dx) for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]
    w27 = [1.0 / (1 + abs(a) + abs(b) + abs(c)) / 10.0 for a, b, c in off27]
    out["s3d27_u0"], out["s3d27_v"] = u3, stencil_numpy(u3, off27, w27, 2)
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **out)
    print("wrote", os.path.join(HERE, "kernels.npz"), sorted(out))


if __name__ == "__main__":
    main()
