"""Accounting parity (CPU): the product's W/Q models, presets, bounds, roofline
and spec loading against the REFERENCE library.

Two sources, same assertions:
  * tests/golden/accounting.json -- fixtures produced by running the reference
    library (tests/golden/make_golden.py); available everywhere;
  * oracle/_ref -- the reference library itself, queried live (this container;
    skipped where the prebuilt shim is absent).
Integers must match exactly; doubles bit-exactly (the product evaluates the
same formulas in the same order, e.g. tensor_core_ceiling's 1+(a-1)/(1+a)
form, reference bounds.cpp:87-97).
"""
import ctypes as C
import json
import os
import random

import pytest

import oracle as O
import paper_2502_16851_b200 as P

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "accounting.json")))


def _call(fn, args, doc=None):
    """Run the product's equivalent of a golden case -> dict like the fixture."""
    try:
        if fn == "scale_model":
            k = P.scale_model(args[0], args[1])
            return {"work": k.work_flops, "traffic": k.traffic_bytes}
        if fn == "gemv_model":
            k = P.gemv_model(*args)
            return {"work": k.work_flops, "traffic": k.traffic_bytes}
        if fn == "spmv_generic_model":
            k = P.spmv_generic_model(*args)
            return {"work": k.work_flops, "traffic": k.traffic_bytes}
        if fn == "spmv_csr_model":
            k = P.spmv_csr_model(*args)
            return {"work": k.work_flops, "traffic": k.traffic_bytes}
        if fn == "stencil_model":
            k = P.stencil_model(args[0], args[1], args[2])
            return {"work": k.work_flops, "traffic": k.traffic_bytes,
                    "points": P.stencil_preset(args[0])[1]}
        if fn == "kernel_speedup_ceiling":
            v, nw = P.kernel_speedup_ceiling(*args)
            return {"value": v, "warnings": nw}
        if fn == "tensor_core_ceiling":
            return {"value": P.tensor_core_ceiling(*args)}
        if fn == "workload_ceiling":
            return {"value": P.workload_ceiling(*args)}
        if fn == "min_temporal_depth":
            return {"value": P.min_temporal_depth(*args)}
        if fn == "tc_scale_trick_throughput":
            return {"value": P.tc_scale_trick_throughput(*args)}
        if fn == "unoverlapped_speedup":
            return {"value": P.unoverlapped_speedup(*args)}
        if fn in ("machine_balance", "attainable", "tensor_alpha"):
            bw, pcc, ptc = args[:3]
            spec = P.HardwareSpec("probe", bw, 0.0, pcc, ptc)
            if fn == "machine_balance":
                return {"value": P.machine_balance(spec, args[3])}
            if fn == "attainable":
                return {"value": P.attainable(spec, args[4], args[3])}
            return {"value": P.tensor_alpha(spec)}
        if fn == "classify":
            return {"value": P.classify(*args)}
        if fn == "load_spec":
            s = P.load_spec(doc)
            return {"bw": s.memory_bandwidth, "l2": s.l2_cache_bytes, "p_cc": s.peak_cuda_core,
                    "p_tc": s.peak_tensor_core}
        if fn == "spec_eval":
            s = P.load_spec(doc)
            _, what, unit, prec, i = args
            if what == "machine_balance":
                return {"value": P.machine_balance(s, unit, prec)}
            if what == "tensor_alpha":
                return {"value": P.tensor_alpha(s, prec)}
            if what == "attainable":
                return {"value": P.attainable(s, i, unit, prec)}
            return {"value": P.ridge_point(s, unit, prec)}
        if fn == "serialize_spec":
            return {"text": P.serialize_spec(P.load_spec(doc))}
        if fn == "builtin_spec":
            s = P.builtin_spec(args[0])
            return {"bw": s.memory_bandwidth, "l2": s.l2_cache_bytes, "p_cc": s.peak_cuda_core,
                    "p_tc": s.peak_tensor_core}
    except P.RooflensError as e:
        return {"error": e.kind}
    raise AssertionError(f"unhandled case {fn}")


@pytest.mark.parametrize("case", GOLDEN["cases"], ids=lambda c: f"{c['fn']}{c['args']}")
def test_golden_against_reference_fixture(case):
    want = {k: v for k, v in case.items() if k not in ("fn", "args", "doc")}
    got = _call(case["fn"], case["args"], case.get("doc"))
    assert got == want


def test_error_message_format_matches_reference():
    """rooflens::Error prefixes the kind (reference error.hpp:38-40)."""
    with pytest.raises(P.RooflensError) as e:
        P.spmv_csr_model(10, 10, 101)
    assert str(e.value).startswith("ValidationError: ")
    with pytest.raises(P.RooflensError) as e:
        P.stencil_model("9d999pt")
    assert e.value.kind == "ValidationError" and "unknown stencil preset" in str(e.value)


ref_only = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref (reference build) absent")


@ref_only
def test_random_models_match_live_reference():
    """Randomised sweep against the live reference library."""
    R = O.ref()
    rng = random.Random(1234)
    for _ in range(3000):
        m, n = rng.randint(1, 1 << 40), rng.randint(1, 1 << 40)
        nnz = rng.randint(0, min(m * n, 1 << 50))
        ib = rng.choice([0, 1, 2, 3, 4, 8, 16])
        prec = rng.randint(0, 2)
        w, q = C.c_uint64(), C.c_uint64()
        rc = R.ref_spmv_csr_model(m, n, nnz, ib, prec, C.byref(w), C.byref(q))
        try:
            k = P.spmv_csr_model(m, n, nnz, ib, prec)
        except P.RooflensError as e:
            assert rc == e.code, (m, n, nnz, ib, R.ref_last_error())
        else:
            assert rc == 0 and (k.work_flops, k.traffic_bytes) == (w.value, q.value)
        sn = rng.choice([0, 1, rng.randint(1, 1 << 63)])
        rc = R.ref_scale_model(sn, prec, C.byref(w), C.byref(q))
        try:
            k = P.scale_model(sn, prec)
        except P.RooflensError as e:
            assert rc == e.code
        else:
            assert rc == 0 and (k.work_flops, k.traffic_bytes) == (w.value, q.value)


@ref_only
def test_random_bounds_match_live_reference():
    R = O.ref()
    rng = random.Random(99)
    for _ in range(3000):
        a = rng.choice([rng.uniform(0.5, 4.0), 1.0, 2.0])
        b = rng.uniform(0.01, 20.0)
        i = rng.choice([rng.uniform(1e-3, 30.0), 0.0])
        o, nw = C.c_double(), C.c_int()
        rc = R.ref_kernel_speedup_ceiling(a, b, i, C.byref(o), C.byref(nw))
        try:
            v, w = P.kernel_speedup_ceiling(a, b, i)
        except P.RooflensError as e:
            assert rc == e.code
        else:
            assert rc == 0 and v == o.value and w == nw.value
        t = C.c_uint64()
        rc = R.ref_min_temporal_depth(b, i, C.byref(t))
        try:
            v = P.min_temporal_depth(b, i)
        except P.RooflensError as e:
            assert rc == e.code
        else:
            assert rc == 0 and v == t.value


def test_stencil_presets_and_default_weights():
    expect = {"2d5pt": (2, 5, 1), "2d9pt": (2, 9, 1), "2d13pt": (2, 13, 3), "2d49pt": (2, 49, 3),
              "3d7pt": (3, 7, 1), "3d27pt": (3, 27, 1)}
    for name, info in expect.items():
        assert P.stencil_preset(name) == info
        w = P.stencil_default_weights(name)
        assert len(w) == info[1]
        assert w == list(O.default_weights(name))  # oracle restates BASELINE.json's rule
        assert abs(sum(w) - 1.0) < 1e-15
    w27 = P.stencil_default_weights("3d27pt")
    assert w27[13] == (1.0 / 1.0) / 10.0 and w27[0] == (1.0 / 4.0) / 10.0  # raw/S, S = 10


def test_baseline_known_answers():
    """SURVEY.md §4 known-answer pins, computed by the reference library."""
    assert P.scale_model(1 << 27) == P.KernelCharacterization(134217728, 2147483648)
    assert P.spmv_csr_model(1 << 22, 1 << 22, 1 << 26) == P.KernelCharacterization(134217728, 889192452)
    assert P.stencil_model("2d5pt") == P.KernelCharacterization(10, 16)
    assert P.stencil_model("3d7pt") == P.KernelCharacterization(14, 16)
    assert P.stencil_model("3d27pt") == P.KernelCharacterization(54, 16)
    assert P.tensor_core_ceiling(2.0) == 4.0 / 3.0


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref absent")
@pytest.mark.parametrize("unit", [P.CUDA_CORE, P.TENSOR_CORE])
@pytest.mark.parametrize("lims", [(1e-3, 1e3, 2), (0.01, 100.0, 7), (1.0, 2.0, 33), (1e-2, 1e4, 128)])
def test_sample_curve_matches_reference(unit, lims):
    """ridge_point / sample_curve (roofline.cpp:36-79): identical samples,
    the ridge inserted in order, bit-exact doubles."""
    import ctypes as C

    import numpy as np

    spec = P.HardwareSpec("B200", 6.5431e12, 126e6, 36.43e12, 37.15e12)
    i_min, i_max, n = lims
    got = P.sample_curve(spec, i_min, i_max, n, unit=unit)
    xs = np.empty(n + 1)
    ys = np.empty(n + 1)
    cnt = C.c_uint64()
    rc = O.ref().ref_sample_curve(spec.memory_bandwidth, spec.peak_cuda_core, spec.peak_tensor_core, unit,
                                  i_min, i_max, n, xs.ctypes.data, ys.ctypes.data, n + 1, C.byref(cnt))
    assert rc == 0
    want = list(zip(xs[:cnt.value].tolist(), ys[:cnt.value].tolist()))
    assert got == want
    assert P.ridge_point(spec, unit) == P.machine_balance(spec, unit)


def test_sample_curve_errors():
    spec = P.HardwareSpec("B200", 6.5431e12, 126e6, 36.43e12, 37.15e12)
    for args in ((0.0, 1.0, 4), (2.0, 1.0, 4), (1.0, 2.0, 1)):
        with pytest.raises(P.RooflensError) as e:
            P.sample_curve(spec, *args)
        assert e.value.kind == "InvalidRange"


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref absent")
def test_mem_cmp_ratio_and_overlapped_total_match_reference():
    import ctypes as C

    rng = random.Random(7)
    for _ in range(200):
        b, i = rng.choice([0.0, 1.0, rng.uniform(0.1, 50)]), rng.choice([0.0, -1.0, rng.uniform(1e-3, 100)])
        out = C.c_double()
        rc = O.ref().ref_mem_cmp_ratio(b, i, C.byref(out))
        if rc == 0:
            assert P.mem_cmp_ratio(b, i) == out.value
        else:
            with pytest.raises(P.RooflensError) as e:
                P.mem_cmp_ratio(b, i)
            assert e.value.code == rc
        t = [rng.choice([0.0, -1.0, rng.uniform(0, 10)]) for _ in range(3)]
        rc = O.ref().ref_overlapped_total(*t, C.byref(out))
        if rc == 0:
            assert P.overlapped_total(*t) == out.value
        else:
            with pytest.raises(P.RooflensError) as e:
                P.overlapped_total(*t)
            assert e.value.code == rc


def test_load_spec_file_and_round_trip(tmp_path):
    """load_spec_file (hardware.cpp:239-247): IoError for a missing file; a
    serialized spec loads back to the same table (hardware.cpp:249-264)."""
    with pytest.raises(P.RooflensError) as e:
        P.load_spec_file(tmp_path / "absent.json")
    assert e.value.kind == "IoError" and "cannot open spec file" in str(e.value)
    spec = P.HardwareSpec("B200", 6.5431e12, 126e6, 36.43e12, 37.15e12, fp32=(72.1e12, 0.0))
    f = tmp_path / "b200.json"
    f.write_text(P.serialize_spec(spec))
    assert P.load_spec_file(f) == spec
    assert P.machine_balance(spec, P.CUDA_CORE, 1) == 72.1e12 / 6.5431e12
    with pytest.raises(P.RooflensError) as e:
        P.tensor_alpha(spec, 1)
    assert e.value.kind == "MissingPeak"


@ref_only
def test_random_peak_tables_match_live_reference():
    """Every (unit, precision) evaluation and serialize_spec on random peak
    tables (entries absent, zero, negative or positive) against the reference."""
    R = O.ref()
    rng = random.Random(77)
    for _ in range(400):
        peaks = {}
        for pk in ("fp64", "fp32", "fp16"):
            ent = {}
            for fld in ("cuda_core_tflops", "tensor_core_tflops"):
                r = rng.random()
                if r < 0.45:
                    continue
                ent[fld] = 0 if r < 0.5 else (-1.5 if r < 0.53 else round(rng.uniform(0.1, 2000), 3))
            if ent or rng.random() < 0.2:
                peaks[rng.choice([pk, pk.upper()])] = ent
        doc = json.dumps({"name": "r", "memory_bandwidth_tbps": round(rng.uniform(0.5, 9), 4),
                          "l2_cache_mb": rng.choice([0, 40, 126]), "peaks": peaks})
        for what in range(4):
            for unit in (0, 1):
                for prec in (0, 1, 2):
                    o = C.c_double()
                    rc = R.ref_spec_eval(doc.encode(), what, unit, prec, 0.3, C.byref(o))
                    fns = (lambda s: P.machine_balance(s, unit, prec), lambda s: P.tensor_alpha(s, prec),
                           lambda s: P.attainable(s, 0.3, unit, prec), lambda s: P.ridge_point(s, unit, prec))
                    try:
                        got, grc = fns[what](P.load_spec(doc)), 0
                    except P.RooflensError as e:
                        grc, got = e.code, None
                    assert grc == rc, (doc, what, unit, prec)
                    if rc == 0:
                        assert got == o.value, (doc, what, unit, prec)
        buf = C.create_string_buffer(4096)
        rc = R.ref_serialize_spec(doc.encode(), buf, 4096)
        if rc == 0:
            assert P.serialize_spec(P.load_spec(doc)) == buf.value.decode()


# ---------------------------------------------------------------------------
# SpeedupBound text (bounds.hpp:27-45) and the analysis report (report.hpp)
# ---------------------------------------------------------------------------
def _ref_bound(kind, a, b=0.0, c=0.0, d=0.0):
    import ctypes as C

    v, k, na, nw = C.c_double(), C.c_int(), C.c_int(), C.c_int()
    text, kname = C.create_string_buffer(4096), C.create_string_buffer(64)
    rc = O.ref().ref_bound_text(kind, a, b, c, d, C.byref(v), C.byref(k), C.byref(na), C.byref(nw), text, 4096,
                                kname, 64)
    if rc:
        return rc
    lines = text.value.decode().split("\n")[:-1]
    return {"value": v.value, "kind": k.value, "kind_name": kname.value.decode(),
            "assumptions": lines[:na.value], "warnings": lines[na.value:]}


BOUND_CASES = [
    ("unoverlapped", 0, (1.0, 3.0, 0.5, 2.0)), ("unoverlapped", 0, (0.0, 1.0, 0.0, 4.0)),
    ("kernel", 1, (2.01, 5.0, 0.0625)), ("kernel", 1, (1.97, 8.5, 9.0)), ("kernel", 1, (1.0, 5.0, 5.0)),
    ("tensor_core", 2, (2.0,)), ("tensor_core", 2, (1.0172,)),
    ("workload", 3, (0.25, 5.0)), ("workload", 3, (6.75, 5.56)),
]


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("which,kind,args", BOUND_CASES)
def test_speedup_bound_text_matches_reference(which, kind, args):
    ours = P.speedup_bound(which, *args)
    ref = _ref_bound(kind, *args)
    assert ours == ref


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("which,kind,args", [("kernel", 1, (0.5, 5.0, 1.0)), ("kernel", 1, (2.0, 5.0, 0.0)),
                                             ("workload", 3, (1.0, 0.0)), ("unoverlapped", 0, (-1.0, 1.0, 0.0, 2.0)),
                                             ("unoverlapped", 0, (0.0, 0.0, 0.0, 2.0))])
def test_speedup_bound_errors_match_reference(which, kind, args):
    with pytest.raises(P.RooflensError) as e:
        P.speedup_bound(which, *args)
    assert e.value.code == _ref_bound(kind, *args)


def test_analysis_report_fields():
    """build_analysis (report.hpp:40-44): the verdict's X is the min bound to
    3 significant digits; the json/csv numbers are the C-ABI's own values;
    text is 4 significant digits; output is deterministic."""
    import csv
    import io
    import json

    spec = P.builtin_spec("A100-80GB")
    kc = P.spmv_csr_model(1 << 22, 1 << 22, 1 << 26)
    j = json.loads(P.analysis_report(spec, "spmv-csr", kc, "json"))
    a = P.tensor_alpha(spec)
    B = P.machine_balance(spec)
    vals = {b["kind"]: b["value"] for b in j["bounds"]}
    assert vals["kernel ceiling"] == P.kernel_speedup_ceiling(a, B, kc.intensity)[0]
    assert vals["tensor-core ceiling"] == P.tensor_core_ceiling(a)
    assert vals["workload ceiling"] == P.workload_ceiling(kc.intensity, B)
    assert j["verdict"] == f"tensor cores cannot exceed {min(vals.values()):.3g}x on this kernel/machine"
    assert j["boundedness"] == "memory-bound" and j["alpha"] == a and j["balance"] == B
    assert [b["assumptions"] for b in j["bounds"]] == [
        P.speedup_bound("kernel", a, B, kc.intensity)["assumptions"], P.speedup_bound("tensor_core", a)["assumptions"],
        P.speedup_bound("workload", kc.intensity, B)["assumptions"]]
    rows = list(csv.reader(io.StringIO(P.analysis_report(spec, "spmv-csr", kc, "csv"))))
    d = {k: v for k, v in rows[1:]}
    assert float(d["kernel ceiling"]) == vals["kernel ceiling"] and int(d["traffic_bytes"]) == kc.traffic_bytes
    txt = P.analysis_report(spec, "spmv-csr", kc, "text")
    assert f"{vals['kernel ceiling']:.4g}" in txt and txt == P.analysis_report(spec, "spmv-csr", kc, "text")
    # compute-bound kernel: the kernel-ceiling warning travels into the report
    j = json.loads(P.analysis_report(spec, "2d49pt", P.stencil_model("2d49pt"), "json"))
    assert j["boundedness"] == "compute-bound" and j["bounds"][0]["warnings"]
    # stencil section (t > 15.98 on GH200 at B = 9.99)
    j = json.loads(P.analysis_report(P.builtin_spec("GH200"), "2d5pt", P.stencil_model("2d5pt"), "json",
                                     balance_override=9.99, single_step_intensity=0.625))
    assert j["min_temporal_depth"] == 16 and j["balance_overridden"] and j["balance"] == 9.99
    # a spec without a tensor-core peak: workload ceiling only, with a note
    j = json.loads(P.analysis_report(P.HardwareSpec("cc-only", 1e12, 1e6, 1e13), "scale", P.scale_model(10), "json"))
    assert [b["kind"] for b in j["bounds"]] == ["workload ceiling"] and "alpha" not in j
    with pytest.raises(P.RooflensError) as e:
        P.analysis_report(spec, "scale", P.scale_model(10), "json", balance_override=0.0)
    assert e.value.kind == "ZeroBalance"
    with pytest.raises(P.RooflensError) as e:
        P.analysis_report(spec, "scale", P.scale_model(10), "json", precision=P.FP16)
    assert e.value.kind == "MissingPeak"
