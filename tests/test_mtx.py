"""Matrix Market ingestion.

CPU: rl_mtx_stats against the reference's own parse_stats_file (oracle/_ref)
on valid files and every error kind; rl_mtx_read_csr against scipy.io.mmread;
rl_matrix_analysis_of against the reference's stats_to_report.
GPU: SpMV on a CSR loaded from a .mtx file."""
import ctypes as C
import os

import numpy as np
import pytest
import scipy.io
import scipy.sparse as sp

import oracle as O
import paper_2502_16851_b200 as P

GOOD = {
    "general_real": "%%MatrixMarket matrix coordinate real general\n% comment\n4 5 6\n1 1 2.5\n2 3 -1\n4 5 3e-2\n3 1 7\n4 4 1\n1 5 -2\n",
    "symmetric": "%%MatrixMarket matrix coordinate real symmetric\n3 3 4\n1 1 4\n2 1 1\n3 2 -2\n3 3 5\n",
    "skew": "%%MatrixMarket matrix coordinate real skew-symmetric\n3 3 2\n2 1 1.5\n3 1 -0.5\n",
    "pattern": "%%MatrixMarket matrix coordinate pattern general\n3 3 3\n1 2\n2 3\n3 1\n",
    "integer_crlf": "%%MatrixMarket matrix coordinate integer general\r\n2 2 2\r\n1 1 3\r\n2 2 -4\r\n",
    "blank_lines": "%%MatrixMarket matrix coordinate real general\n\n% c\n2 2 1\n\n2 1 9\n\n",
}
BAD = {
    "bad_banner": ("%%MatrixMarkt matrix coordinate real general\n1 1 1\n1 1 1\n", "BadBanner"),
    "bad_object": ("%%MatrixMarket vector coordinate real general\n1 1 1\n1 1 1\n", "BadBanner"),
    "array": ("%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n", "UnsupportedFormat"),
    "truncated": ("%%MatrixMarket matrix coordinate real general\n3 3 3\n1 1 1\n2 2 2\n", "TruncatedFile"),
    "no_size": ("%%MatrixMarket matrix coordinate real general\n% only comments\n", "TruncatedFile"),
    "bad_index": ("%%MatrixMarket matrix coordinate real general\n3 3 1\n4 1 1\n", "IndexOutOfRange"),
    "zero_index": ("%%MatrixMarket matrix coordinate real general\n3 3 1\n0 1 1\n", "IndexOutOfRange"),
    "bad_value": ("%%MatrixMarket matrix coordinate real general\n3 3 1\n1 1 abc\n", "MalformedEntry"),
    "tokens": ("%%MatrixMarket matrix coordinate real general\n3 3 1\n1 1\n", "MalformedEntry"),
    "extra": ("%%MatrixMarket matrix coordinate real general\n3 3 1\n1 1 1\n2 2 2\n", "MalformedEntry"),
    "skew_diag": ("%%MatrixMarket matrix coordinate real skew-symmetric\n3 3 1\n2 2 1\n", "MalformedEntry"),
    "size_line": ("%%MatrixMarket matrix coordinate real general\n3 3\n", "MalformedEntry"),
    "empty_matrix": ("%%MatrixMarket matrix coordinate real general\n3 3 0\n", "ValidationError"),
    "empty_file": ("", "BadBanner"),
}


@pytest.fixture
def mtx(tmp_path):
    def write(name, text):
        p = tmp_path / f"{name}.mtx"
        p.write_bytes(text.encode())
        return str(p)
    return write


def _ref_stats(path):
    r, c, n = C.c_uint64(), C.c_uint64(), C.c_uint64()
    rc = O.ref().ref_parse_stats_file(path.encode(), C.byref(r), C.byref(c), C.byref(n))
    return rc, (r.value, c.value, n.value)


ref_only = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref absent")


@ref_only
@pytest.mark.parametrize("name", sorted(GOOD))
def test_stats_match_reference(mtx, name):
    path = mtx(name, GOOD[name])
    rc, want = _ref_stats(path)
    assert rc == 0
    assert P.mtx_stats(path) == want


@ref_only
@pytest.mark.parametrize("name", sorted(BAD))
def test_errors_match_reference(mtx, name):
    text, kind = BAD[name]
    path = mtx(name, text)
    rc, _ = _ref_stats(path)
    with pytest.raises(P.RooflensError) as e:
        P.mtx_stats(path)
    assert e.value.kind == kind and e.value.code == rc


def test_missing_file_is_io_error(tmp_path):
    with pytest.raises(P.RooflensError) as e:
        P.mtx_stats(str(tmp_path / "nope.mtx"))
    assert e.value.kind == "IoError"


@pytest.mark.parametrize("name", sorted(GOOD))
def test_csr_matches_scipy(mtx, name):
    path = mtx(name, GOOD[name])
    rp, col, val, ncols = P.mtx_read_csr(path)
    got = sp.csr_matrix((val, col, rp), shape=(rp.size - 1, ncols)).toarray()
    want = scipy.io.mmread(path)
    want = want.toarray() if sp.issparse(want) else np.asarray(want)
    assert np.array_equal(got, want.astype(np.float64))
    assert all(np.all(np.diff(col[rp[i]:rp[i + 1]]) >= 0) for i in range(rp.size - 1))
    assert rp[-1] == P.mtx_stats(path)[2]


@ref_only
def test_matrix_analysis_matches_reference():
    spec = P.HardwareSpec("B200", 6.5431e12, 126e6, 36.43e12, 37.15e12)
    for rows, cols, nnz in ((1 << 22, 1 << 22, 1 << 26), (5558326, 5558326, 59524291), (1000, 1000, 5000)):
        got = P.matrix_analysis(rows, cols, nnz, spec)
        w, q, csr = C.c_uint64(), C.c_uint64(), C.c_uint64()
        bd, kw, fits = C.c_int(), C.c_int(), C.c_int()
        kc, wc = C.c_double(), C.c_double()
        rc = O.ref().ref_stats_to_report(rows, cols, nnz, spec.memory_bandwidth, spec.l2_cache_bytes,
                                         spec.peak_cuda_core, spec.peak_tensor_core, C.byref(w), C.byref(q),
                                         C.byref(bd), C.byref(kc), C.byref(kw), C.byref(wc), C.byref(csr),
                                         C.byref(fits))
        assert rc == 0
        assert (got["work_flops"], got["traffic_bytes"], got["boundedness"], got["kernel_ceiling"],
                got["kernel_ceiling_warnings"], got["workload_ceiling"], got["csr_bytes"], got["fits_in_l2"]) == \
            (w.value, q.value, bd.value, kc.value, kw.value, wc.value, csr.value, fits.value)


@pytest.mark.gpu
@pytest.mark.parametrize("unit", [P.CUDA_CORE, P.TENSOR_CORE])
def test_spmv_from_mtx_file(cuda, tmp_path, unit):
    import torch

    A = sp.random(3000, 2500, density=0.004, format="coo", random_state=np.random.default_rng(3))
    S = sp.random(2000, 2000, density=0.002, format="coo", random_state=np.random.default_rng(4))
    S = sp.tril(S + S.T).tocoo()
    for name, M, sym in (("gen", A, "general"), ("sym", S, "symmetric")):
        path = str(tmp_path / f"{name}.mtx")
        scipy.io.mmwrite(path, M, symmetry=sym)
        rp, col, val, ncols = P.mtx_read_csr(path)
        x = np.random.default_rng(1).uniform(-1, 1, ncols)
        ref = O.spmv_csr(rp, col, val, x)
        full = scipy.io.mmread(path).tocsr() @ x
        assert O.rel_err(ref, full) < 1e-14
        d = [torch.from_numpy(np.ascontiguousarray(t)).cuda() for t in (rp, col, val, x)]
        y = torch.empty(rp.size - 1, dtype=torch.float64, device="cuda")
        P.spmv_csr(d[0], d[1], d[2], d[3], y, unit=unit)
        torch.cuda.synchronize()
        assert O.rel_err(y.cpu().numpy(), ref) <= 1e-12
