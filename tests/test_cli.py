"""CLI / analysis report (reference SPEC.md:447-531 examples)."""
import csv
import io
import json

import numpy as np

import pytest

import paper_2502_16851_b200 as P
from paper_2502_16851_b200 import cli


def run(*argv):
    out = io.StringIO()
    rc = cli.main(list(argv), out=out)
    return rc, out.getvalue()


def test_hardware_list_and_show():
    rc, txt = run("hardware", "list")
    assert rc == 0 and "A100-80GB" in txt and "GH200" in txt
    rc, txt = run("hardware", "show", "A100-80GB")
    assert rc == 0
    rows = dict(line.split(None, 1) for line in txt.strip().splitlines())
    assert float(rows["fp64_balance_cuda_core"]) == 5.0
    assert abs(float(rows["fp64_alpha"]) - 2.01) < 0.01
    assert run("hardware", "show", "nosuch")[0] == 2


def test_analyze_gemv_workload_ceiling():
    """"Speedup_A100(GEMV) < 1.05"."""
    rc, txt = run("analyze", "--hw", "A100-80GB", "--kernel", "gemv", "--m", "100000", "--n", "100000",
                  "--format", "json")
    rep = json.loads(txt)
    wc = [b["value"] for b in rep["bounds"] if b["kind"] == "workload ceiling"][0]
    assert rc == 0 and 1.0499 <= wc <= 1.0500


def test_analyze_temporal_depth_with_balance_override():
    """t > 15.98 on GH200 with B = 9.99."""
    rc, txt = run("analyze", "--hw", "GH200", "--kernel", "stencil", "--shape", "2d5pt",
                  "--balance-override", "9.99", "--format", "json")
    rep = json.loads(txt)
    assert rc == 0 and rep["min_temporal_depth"] == 16 and rep["balance_overridden"]


def test_analyze_scale_verdict():
    rc, txt = run("analyze", "--hw", "A100-80GB", "--kernel", "scale", "--n", "1", "--format", "json")
    rep = json.loads(txt)
    tc = [b["value"] for b in rep["bounds"] if b["kind"] == "tensor-core ceiling"][0]
    assert rc == 0 and rep["boundedness"] == "memory-bound"
    assert abs(tc - 4 / 3) < 1e-12 or tc == P.tensor_core_ceiling(19.5 / 9.7)


def test_formats_agree_and_are_deterministic():
    args = ("analyze", "--hw", "A100-80GB", "--kernel", "spmv-csr", "--m", "4194304", "--nnz", "67108864")
    j = json.loads(run(*args, "--format", "json")[1])
    rows = dict(csv.reader(io.StringIO(run(*args, "--format", "csv")[1])))
    assert float(rows["intensity"]) == j["kernel"]["intensity"]
    assert int(rows["traffic_bytes"]) == 889192452
    assert run(*args, "--format", "csv") == run(*args, "--format", "csv")
    assert run(*args) == run(*args)


def test_matrix_table_sorted_and_partial_failure(tmp_path):
    a = tmp_path / "a.mtx"
    a.write_text("%%MatrixMarket matrix coordinate real general\n3 3 4\n1 1 1\n2 2 1\n3 3 1\n1 3 1\n")
    b = tmp_path / "b.mtx"
    b.write_text("%%MatrixMarket matrix coordinate real symmetric\n3 3 2\n1 1 1\n2 1 1\n")
    bad = tmp_path / "bad.mtx"
    bad.write_text("%%MatrixMarkt matrix coordinate real general\n")
    rc, txt = run("matrix", "--hw", "A100-80GB", str(a), str(b))
    lines = txt.strip().splitlines()
    assert rc == 0 and lines[1].startswith("b.mtx,") and lines[2].startswith("a.mtx,")
    rc, txt = run("matrix", "--hw", "A100-80GB", str(a), str(bad))
    assert rc == 2 and "error bad.mtx" in txt and "a.mtx," in txt


def test_roofline_csv_matches_attainable(tmp_path):
    out = tmp_path / "r.csv"
    rc, _ = run("roofline", "--hw", "A100-80GB", "--out", str(out), "--points", "16")
    assert rc == 0
    spec = P.builtin_spec("A100-80GB")
    rows = list(csv.DictReader(open(out)))
    assert any(float(r["intensity"]) == 5.0 for r in rows)  # ridge inserted
    for r in rows:
        unit = P.CUDA_CORE if r["ceiling_name"].endswith("CudaCore") else P.TENSOR_CORE
        assert float(r["attainable"]) == P.attainable(spec, float(r["intensity"]), unit)
    svg = tmp_path / "r.svg"
    assert run("roofline", "--hw", "A100-80GB", "--out", str(svg))[0] == 0
    assert svg.read_text().startswith("<svg")


@pytest.mark.gpu
def test_measure_runs_kernel(cuda):
    rc, txt = run("measure", "--kernel", "scale", "--n", str(1 << 24), "--reps", "3", "--format", "json")
    rep = json.loads(txt)
    assert rc == 0 and rep["measured"]["gbs"] > 100


@pytest.mark.gpu
@pytest.mark.parametrize("argv", [
    ("--kernel", "gemv", "--m", "2048", "--n", "8192"),
    ("--kernel", "2d49pt", "--unit", "tc"),
    ("--kernel", "2d5pt", "--t", "5"),
])
def test_measure_next_rows(cuda, argv):
    rc, txt = run("measure", *argv, "--reps", "2", "--format", "json")
    rep = json.loads(txt)
    assert rc == 0 and rep["measured"]["gbs"] > 100 and rep["kernel"]["traffic_bytes"] > 0


@pytest.mark.gpu
def test_measure_mtx_file(cuda, tmp_path):
    import scipy.io
    import scipy.sparse as sp

    path = tmp_path / "a.mtx"
    scipy.io.mmwrite(str(path), sp.random(3000, 3000, density=0.01, format="coo",
                                          random_state=np.random.default_rng(0)))
    rc, txt = run("measure", "--kernel", "spmv-csr", "--mtx", str(path), "--reps", "2", "--format", "json")
    rep = json.loads(txt)
    assert rc == 0 and rep["kernel"]["name"] == "spmv-csr:a.mtx"
    assert run("measure", "--kernel", "scale", "--mtx", str(path))[0] == 1


def test_precision_flag(tmp_path):
    """Analysis runs at any precision the spec has peaks for (MissingPeak ->
    exit 2 otherwise); the kernels (measure) are FP64 only."""
    assert run("--precision", "fp64", "hardware", "list")[0] == 0
    assert run("--precision", "fp32", "measure", "--kernel", "scale")[0] == 2
    doc = tmp_path / "s.json"
    doc.write_text(json.dumps({"name": "X", "memory_bandwidth_tbps": 2.0, "l2_cache_mb": 40,
                               "peaks": {"fp64": {"cuda_core_tflops": 10.0},
                                         "fp32": {"cuda_core_tflops": 20.0, "tensor_core_tflops": 160.0}}}))
    rc, txt = run("--precision", "fp32", "analyze", "--hw", str(doc), "--kernel", "scale", "--n", "1000",
                  "--format", "json")
    rep = json.loads(txt)
    assert rc == 0 and rep["precision"] == "FP32" and rep["alpha"] == 8.0
    assert rep["kernel"]["traffic_bytes"] == 8000 and rep["balance"] == 10.0
    assert run("--precision", "fp16", "analyze", "--hw", str(doc), "--kernel", "scale", "--n", "8")[0] == 2


def test_measured_b200_spec_document():
    """The measured B200 is a reference-schema spec document
    (profiles/B200-measured.json, written from bench.py's `hardware_spec`),
    read through load_spec_file and round-tripping serialize_spec."""
    spec = cli.measured_b200()
    assert spec == P.load_spec_file(cli.SPEC_DOC)
    assert P.serialize_spec(spec) == open(cli.SPEC_DOC).read()
    assert 5.0 < P.machine_balance(spec) < 6.5 and 0.9 < P.tensor_alpha(spec) < 1.2
    rc, txt = run("analyze", "--hw", "B200-measured", "--kernel", "spmv-csr", "--m", "4194304", "--nnz",
                  "67108864", "--format", "json")
    assert rc == 0 and json.loads(txt)["machine"]["name"] == "B200-measured"
