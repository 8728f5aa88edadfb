"""Generate tests/golden/accounting.json from the REFERENCE library itself.

Runs the unmodified reference (rooflens, /root/reference/proj/src) through the
oracle/_ref shim built by oracle/Makefile, over the SPEC.md examples, the
BASELINE.json configs and the error edge cases, and records every result (or
error kind).  tests/test_accounting.py checks the product C-ABI against these
fixtures on every machine (the GPU box has no /root/reference) and against the
live reference library wherever oracle/_ref is present.

    make -C oracle && python tests/golden/make_golden.py
"""
import ctypes as C
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle as O  # noqa: E402

KINDS = ["MissingPeak", "ParseError", "ValidationError", "MissingField", "UnknownHardware",
         "InvalidCount", "InvalidIndexSize", "ZeroIntensity", "InvalidAlpha", "ZeroBalance",
         "InvalidRange", "BadBanner", "UnsupportedFormat", "MalformedEntry", "IndexOutOfRange",
         "TruncatedFile", "IoError"]

A100 = '{"name": "A100-80GB", "memory_bandwidth_tbps": 1.94, "l2_cache_mb": 40, "peaks": {"fp64": {"cuda_core_tflops": 9.7, "tensor_core_tflops": 19.5}}}'
B200_DOC = '{"name": "B200", "memory_bandwidth_tbps": 6.5431, "l2_cache_mb": 126, "peaks": {"fp64": {"cuda_core_tflops": 36.43, "tensor_core_tflops": 37.15}}}'
SPEC_DOCS = {
    "a100": A100,
    "b200_measured": B200_DOC,
    "gh200": '{"name": "GH200", "memory_bandwidth_tbps": 4.0, "l2_cache_mb": 50, "peaks": {"fp64": {"cuda_core_tflops": 34.0, "tensor_core_tflops": 67.0}}}',
    "fp32_only": '{"name": "x", "memory_bandwidth_tbps": 1, "l2_cache_mb": 1, "peaks": {"FP32": {"cuda_core_tflops": 2}}}',
    "unknown_key": '{"name": "x", "memory_bandwidth_tbps": 1, "l2_cache_mb": 1, "peaks": {}, "extra": 1}',
    "unknown_peak_key": '{"name": "x", "memory_bandwidth_tbps": 1, "l2_cache_mb": 1, "peaks": {"fp64": {"cuda_core_tflops": 1, "foo": 2}}}',
    "missing_field": '{"name": "x", "memory_bandwidth_tbps": 1, "peaks": {"fp64": {"cuda_core_tflops": 1}}}',
    "zero_bw": '{"name": "x", "memory_bandwidth_tbps": 0, "l2_cache_mb": 1, "peaks": {"fp64": {"cuda_core_tflops": 1}}}',
    "tc_without_cc": '{"name": "x", "memory_bandwidth_tbps": 1, "l2_cache_mb": 1, "peaks": {"fp64": {"tensor_core_tflops": 1}}}',
    "empty_peaks": '{"name": "x", "memory_bandwidth_tbps": 1, "l2_cache_mb": 1, "peaks": {}}',
    "bad_precision": '{"name": "x", "memory_bandwidth_tbps": 1, "l2_cache_mb": 1, "peaks": {"fp8": {"cuda_core_tflops": 1}}}',
    "string_bw": '{"name": "x", "memory_bandwidth_tbps": "1", "l2_cache_mb": 1, "peaks": {"fp64": {"cuda_core_tflops": 1}}}',
    "malformed": '{"name": "x", ',
    "not_object": '[1, 2, 3]',
    "negative_peak": '{"name": "x", "memory_bandwidth_tbps": 1, "l2_cache_mb": 1, "peaks": {"fp64": {"cuda_core_tflops": -1}}}',
    "empty_name": '{"name": "", "memory_bandwidth_tbps": 1, "l2_cache_mb": 1, "peaks": {"fp64": {"cuda_core_tflops": 1}}}',
}
# full peak tables: every precision, partial units, mixed-case keys
MULTI_DOCS = {
    "h100_all": '{"name": "H100-SXM", "memory_bandwidth_tbps": 3.35, "l2_cache_mb": 50, "peaks": {"fp64": {"cuda_core_tflops": 33.5, "tensor_core_tflops": 66.9}, "fp32": {"cuda_core_tflops": 66.9, "tensor_core_tflops": 494.7}, "fp16": {"cuda_core_tflops": 133.8, "tensor_core_tflops": 989.4}}}',
    "fp32_only": SPEC_DOCS["fp32_only"],
    "fp16_cc_only": '{"name": "y", "memory_bandwidth_tbps": 2.5, "l2_cache_mb": 0, "peaks": {"Fp16": {"cuda_core_tflops": 7.25}, "fp64": {"cuda_core_tflops": 1.5}}}',
    "b200_fp32": '{"name": "B200", "memory_bandwidth_tbps": 6.5431, "l2_cache_mb": 126, "peaks": {"fp64": {"cuda_core_tflops": 36.43, "tensor_core_tflops": 37.15}, "fp32": {"cuda_core_tflops": 72.1}}}',
    "zero_fp16_tc": '{"name": "z", "memory_bandwidth_tbps": 1, "l2_cache_mb": 1, "peaks": {"fp16": {"cuda_core_tflops": 3, "tensor_core_tflops": 0}}}',
    "tc_without_cc_fp32": '{"name": "z", "memory_bandwidth_tbps": 1, "l2_cache_mb": 1, "peaks": {"fp64": {"cuda_core_tflops": 3}, "fp32": {"tensor_core_tflops": 9}}}',
}


def err(rc):
    return {"error": KINDS[rc - 1] if 1 <= rc <= len(KINDS) else f"rc{rc}"}


def u64pair(fn, *args):
    w, q = C.c_uint64(), C.c_uint64()
    rc = fn(*args, C.byref(w), C.byref(q))
    return err(rc) if rc else {"work": w.value, "traffic": q.value}


def dbl(fn, *args):
    o = C.c_double()
    rc = fn(*args, C.byref(o))
    return err(rc) if rc else {"value": o.value}


def main():
    R = O.ref()
    cases = []
    for n in (1, 7, 1 << 27, 10 ** 9, (1 << 62), 0):
        for p in (0, 1, 2):
            cases.append({"fn": "scale_model", "args": [n, p], **u64pair(R.ref_scale_model, n, p)})
    for m, n in ((1, 1), (1000, 1000), (4096, 8192), (1 << 32, 1 << 32), (0, 5), (5, 0)):
        cases.append({"fn": "gemv_model", "args": [m, n, 0], **u64pair(R.ref_gemv_model, m, n, 0)})
    for a in ((100, 100, 500, 600, 4, 0, 0, 0), (100, 100, 500, 0, 0, 500, 2, 1), (10, 10, 50, 60, 3, 0, 0, 0),
              (10, 10, 101, 0, 0, 0, 0, 0), (0, 10, 5, 0, 0, 0, 0, 0), (10, 10, 0, 0, 0, 0, 0, 0),
              (1 << 22, 1 << 22, 1 << 26, (1 << 26) + (1 << 22) + 1, 4, 0, 0, 0)):
        cases.append({"fn": "spmv_generic_model", "args": list(a), **u64pair(R.ref_spmv_generic_model, *a)})
    for st in ((1 << 22, 1 << 22, 1 << 26, 4, 0),      # BASELINE configs[1]
               (5558326, 5558326, 59524291, 4, 0),     # circuit5M (SPEC.md:165-167 / survey erratum)
               (1000, 1000, 5000, 2, 0), (1000, 1000, 5000, 8, 1), (1000, 1000, 5000, 3, 0),
               (1000, 1000, 5000, 0, 0), (10, 10, 101, 4, 0), (1, 1, 1, 4, 2),
               ((1 << 40), (1 << 40), (1 << 62), 8, 0)):
        cases.append({"fn": "spmv_csr_model", "args": list(st), **u64pair(R.ref_spmv_csr_model, *st)})
    for preset in ("2d5pt", "2d9pt", "2d13pt", "2d49pt", "3d7pt", "3d27pt", "4d81pt"):
        for t in (1, 4, 16, 0):
            for p in (0, 2):
                w, q, pts = C.c_uint64(), C.c_uint64(), C.c_uint64()
                rc = R.ref_stencil_model(preset.encode(), p, t, C.byref(w), C.byref(q), C.byref(pts))
                res = err(rc) if rc else {"work": w.value, "traffic": q.value, "points": pts.value}
                cases.append({"fn": "stencil_model", "args": [preset, p, t], **res})
    # bounds
    for a, b, i in ((2.0, 5.0, 1 / 16), (2.0, 8.5, 0.625), (1.0198, 5.5677, 1 / 16), (1.0198, 5.5677, 0.150943),
                    (1.0198, 5.5677, 0.625), (1.0198, 5.5677, 0.875), (1.0198, 5.5677, 3.375), (2.0, 1.0, 4.0),
                    (0.5, 5.0, 1.0), (2.0, 5.0, 0.0)):
        o, nw = C.c_double(), C.c_int()
        rc = R.ref_kernel_speedup_ceiling(a, b, i, C.byref(o), C.byref(nw))
        cases.append({"fn": "kernel_speedup_ceiling", "args": [a, b, i],
                      **(err(rc) if rc else {"value": o.value, "warnings": nw.value})})
    for a in (1.0, 1.0198, 2.0, 1e6, 0.9):
        cases.append({"fn": "tensor_core_ceiling", "args": [a], **dbl(R.ref_tensor_core_ceiling, a)})
    for i, b in ((0.25, 5.0), (3.375, 5.5677), (0.0, 5.0), (1.0, 0.0)):
        cases.append({"fn": "workload_ceiling", "args": [i, b], **dbl(R.ref_workload_ceiling, i, b)})
    for b, i in ((9.99, 0.625), (8.5, 0.625), (5.5677, 0.625), (5.5677, 3.375), (0.5, 0.625), (0.625, 0.625),
                 (1.0, 0.0), (1e30, 1e-30)):
        o = C.c_uint64()
        rc = R.ref_min_temporal_depth(b, i, C.byref(o))
        cases.append({"fn": "min_temporal_depth", "args": [b, i], **(err(rc) if rc else {"value": o.value})})
    for p, m, n in ((19.5e12, 8, 4), (67e12, 8, 4), (37.15e12, 8, 4), (1.0, 0, 4), (0.0, 8, 4)):
        cases.append({"fn": "tc_scale_trick_throughput", "args": [p, m, n],
                      **dbl(R.ref_tc_scale_trick_throughput, p, m, n)})
    for tcm, tme, tot, a in ((1.0, 3.0, 0.0, 2.0), (0.0, 1.0, 0.0, 2.0), (1.0, 1.0, 1.0, 1.0), (0, 0, 0, 2.0),
                             (-1.0, 1.0, 0.0, 2.0), (1.0, 1.0, 0.0, 0.5)):
        cases.append({"fn": "unoverlapped_speedup", "args": [tcm, tme, tot, a],
                      **dbl(R.ref_unoverlapped_speedup, tcm, tme, tot, a)})
    # roofline on FP64 specs
    for bw, pcc, ptc in ((1.94e12, 9.7e12, 19.5e12), (6.5431e12, 36.43e12, 37.15e12)):
        for unit in (0, 1):
            cases.append({"fn": "machine_balance", "args": [bw, pcc, ptc, unit],
                          **dbl(R.ref_machine_balance, bw, pcc, ptc, unit)})
            for i in (1 / 16, 0.150943, 5.0, 100.0, -1.0):
                cases.append({"fn": "attainable", "args": [bw, pcc, ptc, unit, i],
                              **dbl(R.ref_attainable, bw, pcc, ptc, unit, i)})
        cases.append({"fn": "tensor_alpha", "args": [bw, pcc, ptc], **dbl(R.ref_tensor_alpha, bw, pcc, ptc)})
    for i, b in ((0.1, 5.0), (5.0, 5.0), (6.0, 5.0)):
        cases.append({"fn": "classify", "args": [i, b], "value": R.ref_classify(i, b)})
    for name, doc in SPEC_DOCS.items():
        vals = [C.c_double() for _ in range(4)]
        rc = R.ref_load_spec(doc.encode(), *[C.byref(v) for v in vals])
        res = err(rc) if rc else dict(zip(("bw", "l2", "p_cc", "p_tc"), (v.value for v in vals)))
        cases.append({"fn": "load_spec", "args": [name], "doc": doc, **res})
    # machine_balance / tensor_alpha / attainable / ridge_point at every (unit,
    # precision) on full peak tables, and serialize_spec, from the reference
    for name, doc in MULTI_DOCS.items():
        for what, fn in enumerate(("machine_balance", "tensor_alpha", "attainable", "ridge_point")):
            for unit in (0, 1):
                for prec in (0, 1, 2):
                    if fn == "tensor_alpha" and unit:
                        continue
                    o = C.c_double()
                    rc = R.ref_spec_eval(doc.encode(), what, unit, prec, 0.75, C.byref(o))
                    cases.append({"fn": "spec_eval", "args": [name, fn, unit, prec, 0.75], "doc": doc,
                                  **(err(rc) if rc else {"value": o.value})})
        buf = C.create_string_buffer(4096)
        rc = R.ref_serialize_spec(doc.encode(), buf, 4096)
        cases.append({"fn": "serialize_spec", "args": [name], "doc": doc,
                      **(err(rc) if rc else {"text": buf.value.decode()})})
    for name in ("A100-80GB", "GH200", "B200"):
        vals = [C.c_double() for _ in range(4)]
        rc = R.ref_builtin_spec(name.encode(), *[C.byref(v) for v in vals])
        res = err(rc) if rc else dict(zip(("bw", "l2", "p_cc", "p_tc"), (v.value for v in vals)))
        cases.append({"fn": "builtin_spec", "args": [name], **res})
    out = {"generator": "tests/golden/make_golden.py",
           "source": "reference rooflens library (/root/reference/proj/src) via oracle/_ref",
           "cases": cases}
    with open(os.path.join(HERE, "accounting.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(f"wrote {len(cases)} cases")


if __name__ == "__main__":
    main()
