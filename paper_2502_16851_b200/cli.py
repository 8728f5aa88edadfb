"""rooflens-b200 command line: analysis report and measured-vs-bound per kernel
(SURVEY.md §8f "next" #3; the reference declares but never implements it:
report.hpp:19-48).

    python -m paper_2502_16851_b200.cli hardware list | show NAME | --spec FILE
    python -m paper_2502_16851_b200.cli analyze --hw NAME|FILE --kernel scale|gemv|spmv-csr|stencil
            [--n N] [--m M] [--nnz NNZ] [--shape 2d5pt] [--t T] [--balance-override B]
            [--format text|json|csv]
    python -m paper_2502_16851_b200.cli matrix --hw NAME FILE.mtx ...
    python -m paper_2502_16851_b200.cli roofline --hw NAME --out FILE.csv|FILE.svg [--points K]
    python -m paper_2502_16851_b200.cli measure --kernel scale|gemv|spmv-csr|2d5pt|2d9pt|2d13pt|2d49pt|
            3d7pt|3d27pt [--unit cc|tc] [--reps R] [--t T (2d5pt)] [--mtx FILE.mtx (spmv-csr)]
            (runs the sm_100a kernel; needs a GPU)

Exit codes (SPEC.md cli_report): 0 success, 1 usage error, 2 input/parse error,
3 internal invariant violation.  Every analysis number comes from the C-ABI
(accounting, bounds, roofline); text prints 4 significant digits, json/csv
full precision.  Output is deterministic (no timestamps).
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import math
import os
import sys

from . import (CUDA_CORE, FP16, FP32, FP64, TENSOR_CORE, HardwareSpec, RooflensError, analysis_report,
               attainable, builtin_spec, load_spec_file,
               classify, gemv_model, sample_curve as _sample_curve, kernel_speedup_ceiling, load_spec, machine_balance, matrix_analysis,
               min_temporal_depth, mtx_stats, scale_model, spmv_csr_model, stencil_model, stencil_preset,
               tensor_alpha, tensor_core_ceiling, workload_ceiling)

BUILTINS = ("A100-80GB", "GH200")
BOUNDEDNESS = ("memory-bound", "compute-bound", "balanced")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class UsageError(Exception):
    pass


SPEC_DOC = os.path.join(ROOT, "profiles", "B200-measured.json")


def measured_b200() -> HardwareSpec:
    """The measured B200: profiles/B200-measured.json, the reference-schema
    document bench.py emits as `hardware_spec` (measured HBM copy bandwidth,
    K11 FP64 DFMA/DMMA peaks), read through load_spec_file
    (hardware.cpp:239-247)."""
    if os.path.exists(SPEC_DOC):
        return load_spec_file(SPEC_DOC)
    bw = 6548.8e9
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            bw = float(json.load(f)["hbm_gbs"]) * 1e9
    except Exception:
        pass
    return HardwareSpec("B200-measured", bw, 126e6, 36.4e12, 37.0e12)


def resolve_hw(name: str) -> HardwareSpec:
    if name in BUILTINS:
        return builtin_spec(name)
    if name in ("B200", "B200-measured"):
        return measured_b200()
    if os.path.exists(name):
        with open(name) as f:
            return load_spec(f.read())
    path = os.environ.get("ROOFLENS_HW_PATH")
    if path and os.path.exists(os.path.join(path, name + ".json")):
        with open(os.path.join(path, name + ".json")) as f:
            return load_spec(f.read())
    return builtin_spec(name)  # raises UnknownHardware


def fmt4(x: float) -> str:
    return f"{x:.4g}"


# ---------------------------------------------------------------------------
# analysis report: rooflens::build_analysis + render_* (report.hpp:19-48) in
# the library (csrc/report.cpp, rl_analysis_render)
# ---------------------------------------------------------------------------
def build_analysis(spec: HardwareSpec, kernel_name: str, kc, balance_override=None,
                   single_step_intensity=None, precision: int = FP64) -> dict:
    return json.loads(analysis_report(spec, kernel_name, kc, "json", balance_override, single_step_intensity,
                                      precision))


def render(spec: HardwareSpec, kernel_name: str, kc, fmt: str, balance_override=None,
           single_step_intensity=None, precision: int = FP64) -> str:
    return analysis_report(spec, kernel_name, kc, fmt, balance_override, single_step_intensity, precision)


def kernel_of(args):
    k, p = args.kernel, getattr(args, "prec", FP64)
    if k == "scale":
        return "scale", scale_model(args.n or 1, p), None
    if k == "gemv":
        if not (args.m and args.n):
            raise UsageError("gemv needs --m and --n")
        return "gemv", gemv_model(args.m, args.n, p), None
    if k == "spmv-csr":
        if not (args.m and args.nnz):
            raise UsageError("spmv-csr needs --m, --nnz (and --n for rectangular)")
        return "spmv-csr", spmv_csr_model(args.m, args.n or args.m, args.nnz, precision=p), None
    if k == "stencil":
        shape = args.shape or "2d5pt"
        t = args.t or 1
        return shape, stencil_model(shape, p, t), stencil_model(shape, p, 1).intensity
    raise UsageError(f"unknown kernel {k}")


# ---------------------------------------------------------------------------
# commands
# ---------------------------------------------------------------------------
def cmd_hardware(args, out):
    if args.action == "list":
        for n in BUILTINS + ("B200-measured",):
            out.write(n + "\n")
        return 0
    spec = load_spec(open(args.spec).read()) if args.spec else resolve_hw(args.name or "")
    rows = [("name", spec.name), ("memory_bandwidth_Bps", spec.memory_bandwidth),
            ("l2_cache_bytes", spec.l2_cache_bytes), ("fp64_cuda_core_flops", spec.peak_cuda_core),
            ("fp64_balance_cuda_core", machine_balance(spec, CUDA_CORE))]
    if spec.peak_tensor_core > 0:
        rows += [("fp64_tensor_core_flops", spec.peak_tensor_core),
                 ("fp64_balance_tensor_core", machine_balance(spec, TENSOR_CORE)),
                 ("fp64_alpha", tensor_alpha(spec))]
    for k, v in rows:
        out.write(f"{k:<26}{fmt4(v) if isinstance(v, float) else v}\n")
    return 0


def cmd_analyze(args, out):
    spec = resolve_hw(args.hw)
    name, kc, i1 = kernel_of(args)
    out.write(render(spec, name, kc, args.format, args.balance_override, i1, args.prec))
    return 0


def cmd_matrix(args, out):
    spec = resolve_hw(args.hw)
    rows, failed = [], False
    for path in args.files:
        try:
            m, n, nnz = mtx_stats(path)
            a = matrix_analysis(m, n, nnz, spec)
            rows.append((nnz, os.path.basename(path), m, n, a))
        except RooflensError as e:
            failed = True
            out.write(f"error {os.path.basename(path)}: {e}\n")
    rows.sort(key=lambda r: (r[0], r[1]))  # Table 2 order: by nnz
    out.write("matrix,rows,cols,nnz,intensity,boundedness,kernel_ceiling,fits_in_l2\n")
    for nnz, name, m, n, a in rows:
        I = a["work_flops"] / a["traffic_bytes"]
        out.write(f"{name},{m},{n},{nnz},{I!r},{BOUNDEDNESS[a['boundedness']]},{a['kernel_ceiling']!r},"
                  f"{bool(a['fits_in_l2'])}\n")
    return 2 if failed else 0


def sample_curve(spec: HardwareSpec, unit: int, i_min: float, i_max: float, n: int):
    """reference roofline.cpp:40-79 through the C-ABI (rl_sample_curve)."""
    if not (i_min > 0 and i_min < i_max) or n < 2:
        raise UsageError("need 0 < i_min < i_max and points >= 2")
    name = "FP64 " + ("CudaCore" if unit == CUDA_CORE else "TensorCore")
    return [(x, y, name) for x, y in _sample_curve(spec, i_min, i_max, n, unit=unit)]


def cmd_roofline(args, out):
    spec = resolve_hw(args.hw)
    units = [CUDA_CORE] + ([TENSOR_CORE] if spec.peak_tensor_core > 0 else [])
    pts = [p for u in units for p in sample_curve(spec, u, args.i_min, args.i_max, args.points)]
    if args.out.endswith(".csv"):
        with open(args.out, "w", newline="") as f:
            w = csv.writer(f, lineterminator="\n")
            w.writerow(["intensity", "attainable", "ceiling_name"])
            for x, y, n in pts:
                w.writerow([repr(x), repr(y), n])
    elif args.out.endswith(".svg"):
        W, H, pad = 640, 420, 50
        lx0, lx1 = math.log10(args.i_min), math.log10(args.i_max)
        ys = [y for _, y, _ in pts]
        ly0, ly1 = math.log10(min(ys)), math.log10(max(ys) * 1.2)
        X = lambda x: pad + (math.log10(x) - lx0) / (lx1 - lx0) * (W - 2 * pad)
        Y = lambda y: H - pad - (math.log10(y) - ly0) / (ly1 - ly0) * (H - 2 * pad)
        parts = [f'<svg xmlns="http://www.w3.org/2000/svg" width="{W}" height="{H}">',
                 f'<text x="{pad}" y="20">{spec.name} FP64 roofline</text>']
        for u, color in zip(units, ("#1f77b4", "#d62728")):
            name = "FP64 " + ("CudaCore" if u == CUDA_CORE else "TensorCore")
            line = " ".join(f"{X(x):.2f},{Y(y):.2f}" for x, y, n in pts if n == name)
            parts.append(f'<polyline fill="none" stroke="{color}" points="{line}"/>')
        for name, kc in (("scale", scale_model(1)), ("spmv", spmv_csr_model(1 << 22, 1 << 22, 1 << 26)),
                         ("2d5pt", stencil_model("2d5pt")), ("3d27pt", stencil_model("3d27pt"))):
            if args.i_min <= kc.intensity <= args.i_max:
                x, y = X(kc.intensity), Y(attainable(spec, kc.intensity))
                parts.append(f'<circle cx="{x:.2f}" cy="{y:.2f}" r="3"/><text x="{x + 4:.2f}" y="{y - 4:.2f}">{name}</text>')
        parts.append("</svg>")
        with open(args.out, "w") as f:
            f.write("\n".join(parts) + "\n")
    else:
        raise UsageError("--out must end in .csv or .svg")
    out.write(f"wrote {args.out} ({len(pts)} points)\n")
    return 0


def cmd_measure(args, out):
    """Run the sm_100a kernel and report measured GB/s against the roofline
    and the TC/CC bound of the measured B200 spec."""
    import torch

    from . import (fill_uniform, gemv, gen_band_csr, mtx_read_csr, scale, spmv_csr, stencil, stencil_init,
                   stencil_temporal)

    unit = CUDA_CORE if args.unit == "cc" else TENSOR_CORE
    spec = measured_b200()
    k = args.kernel
    if args.mtx:
        if k != "spmv-csr":
            raise UsageError("--mtx goes with --kernel spmv-csr")
        rp_h, col_h, val_h, ncols = mtx_read_csr(args.mtx)
        rp, col, val = (torch.from_numpy(a).cuda() for a in (rp_h, col_h, val_h))
        x = torch.empty(ncols, dtype=torch.float64, device="cuda")
        y = torch.empty(rp_h.size - 1, dtype=torch.float64, device="cuda")
        fill_uniform(x, 1, 4, 0, 1)
        fn = lambda: spmv_csr(rp, col, val, x, y, unit=unit)
        k = f"spmv-csr:{os.path.basename(args.mtx)}"
    elif args.t and args.t > 1:
        if k != "2d5pt":
            raise UsageError("--t (temporal depth) is implemented for 2d5pt")
        u = torch.empty((16384, 16384), dtype=torch.float64, device="cuda")
        stencil_init(u, 1, 1)
        v = u.clone()
        fn = lambda: stencil_temporal("2d5pt", u, v, args.t, args.t, unit=unit)[0]
        k = f"2d5pt:t={args.t}"
    elif k == "gemv":
        m, n = args.m or 16384, args.n or 65536
        A = torch.empty((m, n), dtype=torch.float64, device="cuda")
        fill_uniform(A.view(-1), 1, 6, 0, 1)
        x = torch.empty(n, dtype=torch.float64, device="cuda")
        fill_uniform(x, 1, 4, 0, 1)
        y = torch.empty(m, dtype=torch.float64, device="cuda")
        fn = lambda: gemv(A, x, y, unit=unit)
    elif k in ("2d9pt", "2d13pt", "2d49pt"):
        u = torch.empty((16384, 16384), dtype=torch.float64, device="cuda")
        stencil_init(u, stencil_preset(k)[2], 1)
        v = u.clone()
        preset = k
        fn = lambda: stencil(preset, u, v, 1, unit=unit)
    elif k == "scale":
        n = args.n or (1 << 27)
        b = torch.empty(n, dtype=torch.float64, device="cuda")
        fill_uniform(b, 1, 1, 0, 1)
        a = torch.empty_like(b)
        fn = lambda: scale(a, b, 3.0, unit=unit)
    elif k == "spmv-csr":
        n, kk, hb = args.n or (1 << 22), 16, 65536
        rp = torch.empty(n + 1, dtype=torch.int32, device="cuda")
        col = torch.empty(n * kk, dtype=torch.int32, device="cuda")
        val = torch.empty(n * kk, dtype=torch.float64, device="cuda")
        x = torch.empty(n, dtype=torch.float64, device="cuda")
        y = torch.empty(n, dtype=torch.float64, device="cuda")
        gen_band_csr(n, 0, n, kk, min(hb, n - 1), 1, rp, col, val)
        fill_uniform(x, 1, 4, 0, 1)
        fn = lambda: spmv_csr(rp, col, val, x, y, unit=unit)
    elif k in ("2d5pt", "3d7pt", "3d27pt"):
        shape = (16384, 16384) if k == "2d5pt" else (512, 512, 512)
        u = torch.empty(shape, dtype=torch.float64, device="cuda")
        stencil_init(u, 1, 1)
        v = u.clone()
        fn = lambda: stencil(k, u, v, 1, unit=unit)
    else:
        raise UsageError(f"unknown kernel {k}")
    kc = fn()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(args.reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / args.reps
    gbs = kc.traffic_bytes / (ms * 1e-3) / 1e9
    rep = build_analysis(spec, k, kc)
    rep["measured"] = {"unit": args.unit, "ms": ms, "gbs": gbs,
                       "frac_of_hbm": gbs * 1e9 / spec.memory_bandwidth,
                       "achieved_flops": kc.work_flops / (ms * 1e-3)}
    if args.format == "json":
        out.write(json.dumps(rep, indent=1) + "\n")
    else:
        out.write(render(spec, k, kc, "text"))
        out.write(f"measured_gbs  {fmt4(gbs)}\nfrac_of_hbm   {fmt4(rep['measured']['frac_of_hbm'])}\n")
    return 0


def main(argv=None, out=None) -> int:
    out = out or sys.stdout
    ap = argparse.ArgumentParser(prog="rooflens-b200")
    ap.add_argument("--format", default="text", choices=["text", "json", "csv"])
    # SPEC.md cli_report global flag: analysis at any precision the spec has
    # peaks for; the kernels (measure) execute in FP64 only
    ap.add_argument("--precision", default="fp64", choices=["fp64", "fp32", "fp16"])
    sub = ap.add_subparsers(dest="cmd", required=True)
    h = sub.add_parser("hardware")
    h.add_argument("action", choices=["list", "show"])
    h.add_argument("name", nargs="?")
    h.add_argument("--spec")
    a = sub.add_parser("analyze")
    a.add_argument("--hw", required=True)
    a.add_argument("--kernel", required=True, choices=["scale", "gemv", "spmv-csr", "stencil"])
    for opt in ("--n", "--m", "--nnz", "--t"):
        a.add_argument(opt, type=int)
    a.add_argument("--shape")
    a.add_argument("--balance-override", type=float)
    a.add_argument("--format", dest="format", default=None, choices=["text", "json", "csv"])
    m = sub.add_parser("matrix")
    m.add_argument("--hw", required=True)
    m.add_argument("files", nargs="+")
    r = sub.add_parser("roofline")
    r.add_argument("--hw", required=True)
    r.add_argument("--out", required=True)
    r.add_argument("--points", type=int, default=64)
    r.add_argument("--i-min", type=float, default=1.0 / 64)
    r.add_argument("--i-max", type=float, default=64.0)
    me = sub.add_parser("measure")
    me.add_argument("--kernel", required=True)
    me.add_argument("--unit", default="cc", choices=["cc", "tc"])
    me.add_argument("--n", type=int)
    me.add_argument("--m", type=int)
    me.add_argument("--t", type=int, help="temporal depth (2d5pt, CUDA core)")
    me.add_argument("--mtx", help="Matrix Market file for --kernel spmv-csr")
    me.add_argument("--reps", type=int, default=20)
    me.add_argument("--format", dest="format", default=None, choices=["text", "json"])
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:
        return 0 if e.code == 0 else 1
    if getattr(args, "format", None) is None:
        args.format = "text"
    args.prec = {"fp64": FP64, "fp32": FP32, "fp16": FP16}[args.precision]
    if args.precision != "fp64" and args.cmd == "measure":
        print(f"ValidationError: the kernels execute in FP64 only (got {args.precision})", file=sys.stderr)
        return 2
    try:
        return {"hardware": cmd_hardware, "analyze": cmd_analyze, "matrix": cmd_matrix,
                "roofline": cmd_roofline, "measure": cmd_measure}[args.cmd](args, out)
    except UsageError as e:
        print(f"usage error: {e}", file=sys.stderr)
        return 1
    except RooflensError as e:
        print(str(e), file=sys.stderr)
        return 2
    except (OSError, ValueError) as e:
        print(f"IoError: {e}", file=sys.stderr)
        return 2
    except AssertionError as e:  # pragma: no cover
        print(f"internal: {e}", file=sys.stderr)
        return 3


if __name__ == "__main__":
    sys.exit(main())
