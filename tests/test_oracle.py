"""Pin the CPU oracle (CPU tests).

The reference ships no executing kernel and no result fixtures, so the
oracle's arithmetic is checked against independent restatements of the
paper's equations (numpy / scipy.sparse / a pure-Python splitmix64) and
hand-computed known answers; its inputs are checked against BASELINE.json's
stated distributions."""
import numpy as np
import pytest
import scipy.sparse as sp

import oracle as O

M64 = (1 << 64) - 1


def _fmix(z):
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def _mix(key, idx):
    return _fmix((key + (idx + 1) * 0x9E3779B97F4A7C15) & M64)


def _key(seed, stream):
    return _mix(_fmix(seed ^ 0x243F6A8885A308D3), stream)


def test_rng_matches_python_restatement():
    for seed in (0, 1, 2025, (1 << 63) + 5):
        for stream in (1, 2, 3, 4, 5):
            k = _key(seed, stream)
            assert O.orc().orc_key(seed, stream) == k
            got = O.fill_uniform(50, seed, stream, 17, 1)
            want = [2.0 * ((_mix(k, 17 + i) >> 11) * 2.0 ** -53) - 1.0 for i in range(50)]
            assert got.tolist() == want


def test_uniform_ranges():
    u = O.fill_uniform(1 << 20, 3, 1, 0, 0)
    assert u.min() >= 0.0 and u.max() < 1.0 and abs(u.mean() - 0.5) < 2e-3
    s = O.fill_uniform(1 << 20, 3, 1, 0, 1)
    assert s.min() >= -1.0 and s.max() < 1.0 and abs(s.mean()) < 4e-3


def test_scale_bit_exact_vs_numpy():
    b = O.fill_uniform(100003, 9, 1, 0, 1)
    for q in (3.0, -0.5, 1e300, 7.123456789):
        assert O.bit_mismatches(O.scale(b, q), q * b) == 0


@pytest.mark.parametrize("m,n,k,hb", [(1000, 1000, 16, 65536), (5000, 5000, 16, 100), (300, 300, 7, 6),
                                      (64, 64, 16, 15)])
def test_band_csr_generator_properties(m, n, k, hb):
    rp, col, val = O.gen_band_csr(m, 0, n, k, hb, 5)
    assert np.array_equal(rp, np.arange(m + 1) * k)
    c = col.reshape(m, k).astype(np.int64)
    rows = np.arange(m)[:, None]
    assert np.all(np.diff(c, axis=1) > 0)                           # sorted, distinct
    assert np.all(c >= np.maximum(0, rows - hb)) and np.all(c <= np.minimum(n - 1, rows + hb))
    assert val.min() >= -1 and val.max() < 1


def test_band_csr_partition_consistency():
    """Rows [r0, r1) generated alone equal the same rows of the whole matrix."""
    rp, col, val = O.gen_band_csr(4000, 0, 4000, 16, 500, 11)
    rp2, col2, val2 = O.gen_band_csr(1000, 1500, 4000, 16, 500, 11)
    assert np.array_equal(col2, col[1500 * 16:2500 * 16])
    assert np.array_equal(val2, val[1500 * 16:2500 * 16])


def test_spmv_vs_scipy():
    rp, col, val = O.gen_band_csr(20000, 0, 20000, 16, 65536, 1)
    x = O.fill_uniform(20000, 1, 4, 0, 1)
    y = O.spmv_csr(rp, col, val, x)
    ref = sp.csr_matrix((val, col, rp), shape=(20000, 20000)) @ x
    assert O.rel_err(y, ref) < 1e-14


def test_spmv_ragged_and_col_base():
    rng = np.random.default_rng(0)
    lens = rng.integers(0, 30, 500)
    lens[::7] = 0
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    col = np.concatenate([np.sort(rng.choice(800, l, replace=False)) for l in lens]).astype(np.int32)
    val = rng.uniform(-1, 1, rp[-1])
    x = rng.uniform(-1, 1, 800)
    ref = sp.csr_matrix((val, col, rp), shape=(500, 800)) @ x
    assert O.rel_err(O.spmv_csr(rp, col, val, x), ref) < 1e-14
    # col_base: the window x_win holds global columns [100, 900)
    xg = rng.uniform(-1, 1, 900)
    cs = (col + 100).astype(np.int32)
    ref2 = sp.csr_matrix((val, cs, rp), shape=(500, 900)) @ xg
    assert O.rel_err(O.spmv_csr(rp, cs, val, xg[100:].copy(), col_base=100), ref2) < 1e-14


def test_spmv_known_answer():
    # [[2, 0, 1], [0, 0, 0], [0, 3, 4]] @ [1, 2, 3] = [5, 0, 18]
    rp = np.array([0, 2, 2, 4], np.int32)
    col = np.array([0, 2, 1, 2], np.int32)
    val = np.array([2.0, 1.0, 3.0, 4.0])
    assert O.spmv_csr(rp, col, val, np.array([1.0, 2.0, 3.0])).tolist() == [5.0, 0.0, 18.0]


def _np_offsets(preset):
    buf = np.zeros(64 * 3, np.int32)
    n = O.orc().orc_preset_offsets(preset.encode(), buf.ctypes.data)
    return buf[: 3 * n].reshape(n, 3)


def _np_stencil(preset, u, steps, w=None):
    """Independent numpy restatement of Eq. 11."""
    off = _np_offsets(preset)
    w = O.default_weights(preset) if w is None else np.asarray(w)
    r = int(np.abs(off).max())
    a, b = u.copy(), u.copy()
    for _ in range(steps):
        inner = tuple(slice(r, s - r) for s in a.shape)
        acc = np.zeros_like(a[inner])
        for (dz, dy, dx), ww in zip(off, w):
            sh = (dz, dy, dx) if a.ndim == 3 else (dy, dx)
            src = tuple(slice(r + d, s - r + d) for d, s in zip(sh, a.shape))
            acc = acc + ww * a[src]
        b[inner] = acc
        a, b = b, a
    return a


@pytest.mark.parametrize("preset,shape", [("2d5pt", (37, 53)), ("2d9pt", (30, 31)), ("2d13pt", (40, 41)),
                                          ("2d49pt", (25, 30)), ("3d7pt", (9, 12, 17)), ("3d27pt", (10, 11, 13))])
def test_stencil_vs_numpy(preset, shape):
    r = 3 if preset in ("2d13pt", "2d49pt") else 1
    u0 = O.stencil_init(shape, r, 4)
    for steps in (1, 2, 5):
        got = O.stencil(preset, u0, steps)
        want = _np_stencil(preset, u0, steps)
        assert O.rel_err(got, want) < 1e-14


def test_stencil_known_answer_2d5pt():
    """Single interior point: v = 0.5*u + 0.125*(N+S+E+W)."""
    u = np.zeros((3, 3))
    u[1, 1] = 8.0
    out = O.stencil("2d5pt", u, 1)
    assert out[1, 1] == 4.0 and out.sum() == 4.0
    u = np.arange(25, dtype=np.float64).reshape(5, 5)
    u[0, :] = u[-1, :] = u[:, 0] = u[:, -1] = 0.0
    out = O.stencil("2d5pt", u, 1)
    # interior (2,2) = 0.5*12 + 0.125*(7+17+11+13) = 12
    assert out[2, 2] == 12.0
    assert np.all(out[0] == 0) and np.all(out[:, -1] == 0)


def test_stencil_init_and_slabs():
    g = O.stencil_init((20, 9, 11), 1, 3)
    assert np.all(g[0] == 0) and np.all(g[-1] == 0) and np.all(g[:, 0] == 0) and np.all(g[:, :, -1] == 0)
    inner = g[1:-1, 1:-1, 1:-1]
    assert inner.min() >= 0 and inner.max() < 1
    slab = O.stencil_init((6, 9, 11), 1, 3, outer_begin=7, global_shape=(20, 9, 11))
    assert O.bit_mismatches(slab, g[7:13]) == 0
    g2 = O.stencil_init((30, 17), 1, 3)
    s2 = O.stencil_init((5, 17), 1, 3, outer_begin=25, global_shape=(30, 17))
    assert O.bit_mismatches(s2, g2[25:30]) == 0


def test_default_weights_rule():
    w = O.default_weights("3d27pt")
    manh = np.abs(_np_offsets("3d27pt")).sum(axis=1)
    assert np.allclose(w, (1.0 / (1 + manh)) / 10.0, rtol=0, atol=0)
    assert O.default_weights("2d5pt").tolist() == [0.5, 0.125, 0.125, 0.125, 0.125]
    assert O.default_weights("3d7pt").tolist() == [0.4] + [0.1] * 6


def test_oracle_against_committed_golden_vectors():
    """oracle/oracle.c against tests/golden/kernels.npz (numpy / math.fsum
    restatements, independent of the oracle): STREAM bit-exact, SpMV and the
    stencils within 1e-14."""
    import os

    G = np.load(os.path.join(os.path.dirname(__file__), "golden", "kernels.npz"))
    assert O.bit_mismatches(O.scale(G["scale_b"], float(G["scale_q"])), G["scale_a"]) == 0
    y = O.spmv_csr(G["spmv_rp"], G["spmv_col"], G["spmv_val"], G["spmv_x"])
    assert O.rel_err(y, G["spmv_y"]) <= 1e-14
    for preset, key, steps in (("2d5pt", "s2d", 3), ("3d7pt", "s3d7", 2), ("3d27pt", "s3d27", 2)):
        assert O.rel_err(O.stencil(preset, G[f"{key}_u0"], steps), G[f"{key}_v"]) <= 1e-14, preset
