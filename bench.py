#!/usr/bin/env python
"""bench.py -- B200 benchmark of the FP64 memory-bound kernels (arXiv 2502.16851).

Metric (BASELINE.json): achieved HBM GB/s (% of B200 peak) per kernel, and the
tensor-core vs CUDA-core speedup against the paper's bound re-derived from
B200's own FP64 peaks and HBM bandwidth.

Headline line (`value`): BASELINE.json configs[1], CSR SpMV FP64, 2^22 rows
per GPU, 16 nnz/row in a +-65536 band, int32 indices, CUDA-core variant; one
step = one y = A x over HBM-resident inputs (889,192,452 algorithmic bytes =
the reference's spmv_csr_model, kernels.cpp:123-135).  At N > 1 each rank
owns 2^22 rows of an N*2^22-row matrix (weak scaling) and every step
exchanges the x band halo with its neighbours over NCCL, overlapped with the
interior rows.  Inputs (889 MB/step) exceed the 126 MB L2; x (32 MiB) stays
L2-resident by design (the model counts it once).

Also on the same JSON line (N = 1): `per_kernel` -- every BASELINE config
(STREAM 2^27 x 20 reps, SpMV x 20, 2d5pt 16384^2 x 100 steps, 3d7pt and
3d27pt 512^3 x 50 steps) on both units, with GB/s, fraction of the measured
HBM peak, TC/CC speedup and the B200-derived bound (K11 FP64 peaks measured
live); `e2e` through the host-buffer C-ABI call; `cpu_baseline` (the oracle
port on this box's cores); `roofline`; `clocks`; `gpu_launches`.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload spmv|stream|2d5pt|3d7pt|3d27pt] [--unit cc|tc]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "achieved HBM GB/s (% of B200 peak) per kernel; TC vs CUDA-core speedup vs bound"
SEED = 2025
HBM_FALLBACK_GBS = 6650.0  # B200_PROFILING.md fallback, used only if MEASURED_PEAKS.json is absent

WORKLOADS = {
    "stream": dict(desc="STREAM Scale FP64 a=q*b, q=3, n=2^27 (BASELINE configs[0])", reps=20),
    "spmv": dict(desc="CSR SpMV FP64, n=2^22 rows/GPU, 16 nnz/row, band +-65536, int32 idx "
                      "(BASELINE configs[1])", reps=20),
    "2d5pt": dict(desc="2d5pt Jacobi FP64 16384^2, c0=0.5 c1=0.125 (BASELINE configs[2])", reps=100),
    "3d7pt": dict(desc="3d7pt Jacobi FP64 512^3, c0=0.4 c1=0.1 (BASELINE configs[3])", reps=50),
    "3d27pt": dict(desc="3d27pt box Jacobi FP64 512^3, w=1/(1+|d|) normalised (BASELINE configs[4])",
                   reps=50),
}


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic():
    """Per-launch DRAM bytes from the committed ncu --set full summary, if any."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return {}


# ---------------------------------------------------------------------------
# clocks: NVML sampled in a thread during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int, period_s: float = 0.01):
        self.samples, self.reasons, self.ok = [], set(), False
        self.max_mhz = None
        self._stop = threading.Event()
        self.period = period_s
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# workloads on the GPU
# ---------------------------------------------------------------------------
class Spmv:
    n_local = 1 << 22
    k = 16
    hb = 65536

    def __init__(self, torch, P, D, rank, world, comm=None, unit=None):
        self.torch, self.P, self.D, self.world = torch, P, D, world
        n_glob = self.n_local * world
        self.part = pt = D.SpmvPartition(n_glob, self.hb, world, rank)
        m = pt.rows
        dev = "cuda"
        self.rp = torch.empty(m + 1, dtype=torch.int32, device=dev)
        self.col = torch.empty(m * self.k, dtype=torch.int32, device=dev)
        self.val = torch.empty(m * self.k, dtype=torch.float64, device=dev)
        self.x = torch.empty(pt.window, dtype=torch.float64, device=dev)
        self.y = torch.empty(m, dtype=torch.float64, device=dev)
        P.gen_band_csr(m, pt.r0, n_glob, self.k, self.hb, SEED, self.rp, self.col, self.val)
        P.fill_uniform(self.x, SEED, 4, pt.col_base, 1)
        # whole-job algorithmic bytes: the reference model on the global matrix;
        # per-rank: the model on the local row block with its own x slice.
        self.job_bytes = P.spmv_csr_model(n_glob, n_glob, n_glob * self.k).traffic_bytes
        self.bytes = P.spmv_csr_model(m, m, m * self.k).traffic_bytes
        self.plans = {}
        self.comm = comm
        self.raw_csr = False  # True: the CSR kernels on the generator's arrays (no plan)
        self.plan_colsort = 1  # the plan's layout choice (tuning key spmv_plan_colsort)

    def step(self, unit):
        P = self.P
        if self.world == 1 and self.raw_csr:
            P.spmv_csr(self.rp, self.col, self.val, self.x, self.y, unit=unit)
        elif self.world == 1:
            # rl_spmv_plan_execute: the plan's layout (K17 column-sorted row
            # blocks on this matrix), built once from the CSR on the first
            # (untimed, warm-up) call -- cusparseSpMV_preprocess-style
            key = (unit, self.plan_colsort)
            if key not in self.plans:
                prev = P.tuning_set("spmv_plan_colsort", self.plan_colsort)
                try:
                    t0 = time.perf_counter()
                    self.plans[key] = P.SpmvPlan(self.rp.cpu(), self.col.cpu(), self.val.cpu(), self.x.numel(),
                                                 unit=unit)
                    self.plan_create_s = time.perf_counter() - t0
                finally:
                    P.tuning_set("spmv_plan_colsort", prev)
            self.plans[key].execute(self.x, self.y)
        else:
            # rl_dist_spmv: NCCL halo exchange overlapped with the interior rows
            if unit not in self.plans:
                self.plans[unit] = self.D.DistSpmv(self.comm, self.n_local * self.world, self.hb,
                                                   [(self.rp, self.col, self.val, self.x, self.y)], unit=unit)
            self.plans[unit].execute()

    def close(self):
        for pl in self.plans.values():
            pl.close()
        self.plans = {}

    def host_buffers(self):
        t = self.torch
        pin = dict(pin_memory=True)
        col = self.col if self.world == 1 else (self.col - self.part.col_base)
        return {"rp": t.empty(self.rp.shape, dtype=t.int32, **pin).copy_(self.rp),
                "col": t.empty(self.col.shape, dtype=t.int32, **pin).copy_(col),
                "val": t.empty(self.val.shape, dtype=t.float64, **pin).copy_(self.val),
                "x": t.empty(self.x.shape, dtype=t.float64, **pin).copy_(self.x),
                "y": t.empty(self.y.shape, dtype=t.float64, **pin)}

    def e2e_step(self, h, unit):
        """The iterative-solver call pattern: A was uploaded once into a plan
        (rl_spmv_plan_create, outside the timed region); each step moves x in
        and y out through pinned host memory (rl_spmv_plan_execute_host).
        N > 1: the owned x goes into the rank's window, rl_dist_spmv_execute,
        y comes back."""
        if self.world > 1:
            self.x[self.part.own_slice()].copy_(h["x"][self.part.own_slice()], non_blocking=True)
            self.step(unit)
            h["y"].copy_(self.y, non_blocking=True)
            self.torch.cuda.current_stream().synchronize()
            return
        if "plan" not in h:
            h["plan"] = self.P.SpmvPlan(h["rp"], h["col"], h["val"], h["x"].numel(), unit=unit)
        h["plan"].execute_host(h["x"], h["y"])

    def full_copy_step(self, h, unit):
        """Everything over PCIe every step (rl_spmv_csr_host)."""
        self.P.spmv_csr_host(h["rp"], h["col"], h["val"], h["x"], h["y"], unit=unit)

    def h2d_d2h(self, h):
        if self.world > 1:
            return self.part.rows * 8, h["y"].numel() * 8
        return h["x"].numel() * 8, h["y"].numel() * 8

    def e2e_stream(self, h, unit, steps):
        """A stream of independent vectors through one plan (N = 1): step k
        uploads its own x (R distinct pinned vectors, rotated), computes, and
        downloads its own y, via rl_spmv_plan_execute_host_async; consecutive
        calls overlap (step k + 1's x upload beside step k's compute and y
        download) and the timed region ends with rl_spmv_plan_wait.  Returns
        (seconds, results bit-identical to one synchronous call each)."""
        t, P, R = self.torch, self.P, 3
        if "plan" not in h:
            h["plan"] = P.SpmvPlan(h["rp"], h["col"], h["val"], h["x"].numel(), unit=unit)
        if "xs" not in h:
            xs = [h["x"]]
            for r in range(1, R):
                d = t.empty_like(self.x)
                P.fill_uniform(d, SEED + r, 4, 0, 1)
                xs.append(t.empty(d.shape, dtype=t.float64, pin_memory=True).copy_(d))
            h["xs"] = xs
            h["ys"] = [t.empty(h["y"].shape, dtype=t.float64, pin_memory=True) for _ in range(R)]
        pl, xs, ys = h["plan"], h["xs"], h["ys"]
        for r in range(R):  # warm: both device slots, every host buffer pair
            pl.execute_host_async(xs[r], ys[r])
        pl.wait()
        t0 = time.perf_counter()
        for k in range(steps):
            pl.execute_host_async(xs[k % R], ys[k % R])
        pl.wait()
        sec = time.perf_counter() - t0
        ok = True
        for r in range(R):  # the last result of each input against a synchronous call
            if steps > r:
                chk = t.empty_like(ys[r])
                pl.execute_host(xs[r], chk)
                ok = ok and bool(t.equal(chk, ys[r]))
        return sec, ok

    def full_copy_bytes(self, h):
        return (sum(h[k].numel() * h[k].element_size() for k in ("rp", "col", "val", "x")),
                h["y"].numel() * 8)


class Stream:
    n = 1 << 27

    def __init__(self, torch, P, D, rank, world, comm=None, unit=None):
        self.torch, self.P, self.D, self.comm, self.world = torch, P, D, comm, world
        lo, hi = D.scale_chunk(self.n * world, world, rank)
        self.b = torch.empty(hi - lo, dtype=torch.float64, device="cuda")
        self.a = torch.empty_like(self.b)
        P.fill_uniform(self.b, SEED, 1, lo, 1)
        self.bytes = P.scale_model(hi - lo).traffic_bytes
        self.job_bytes = P.scale_model(self.n * world).traffic_bytes

    def step(self, unit):
        if self.world == 1:
            self.P.scale(self.a, self.b, 3.0, unit=unit)
        else:
            self.D.dist_scale(self.comm, self.a, self.b, 3.0, self.n * self.world, unit=unit)

    def close(self):
        pass

    def host_buffers(self):
        t = self.torch
        return {"b": t.empty(self.b.shape, dtype=t.float64, pin_memory=True).copy_(self.b),
                "a": t.empty(self.b.shape, dtype=t.float64, pin_memory=True)}

    def e2e_step(self, h, unit):
        if self.world > 1:
            self.b.copy_(h["b"], non_blocking=True)
            self.step(unit)
            h["a"].copy_(self.a, non_blocking=True)
            self.torch.cuda.current_stream().synchronize()
            return
        self.P.scale_host(h["a"], h["b"], 3.0, unit=unit)

    def h2d_d2h(self, h):
        return h["b"].numel() * 8, h["a"].numel() * 8


class Stencil:
    """One step = one full BASELINE run (100 / 50 double-buffered timesteps).
    At N > 1 the global grid grows along the slab axis (weak scaling)."""

    def __init__(self, torch, P, D, rank, world, preset, comm=None, unit=None):
        self.torch, self.P, self.D, self.preset, self.world = torch, P, D, preset, world
        base = (16384, 16384) if preset == "2d5pt" else (512, 512, 512)
        self.tsteps = 100 if preset == "2d5pt" else 50
        self.gshape = gshape = (base[0] * world,) + base[1:]
        self.part = pt = D.SlabPartition(preset, gshape, world, rank)
        self.u = torch.empty(pt.local_shape, dtype=torch.float64, device="cuda")
        P.stencil_init(self.u, 1, SEED, outer_begin=pt.g_lo, global_shape=gshape)
        self.v = self.u.clone()
        inner = lambda shp: __import__("math").prod(s - 2 for s in shp)
        self.job_bytes = 16 * inner(gshape) * self.tsteps
        own_inner = (min(pt.o1, gshape[0] - 1) - max(pt.o0, 1)) * inner((3,) + base[1:])
        self.bytes = 16 * own_inner * self.tsteps
        self.plans = {}
        self.comm = comm

    def step(self, unit):
        P = self.P
        if self.world == 1:
            P.stencil(self.preset, self.u, self.v, self.tsteps, unit=unit)
        else:
            # rl_dist_stencil: per timestep the ghost planes/rows go over NCCL
            # while the slab interior is swept; timestep pairs replay a CUDA graph
            if unit not in self.plans:
                self.plans[unit] = self.D.DistStencil(self.comm, self.preset, self.gshape, [self.u], [self.v],
                                                      unit=unit)
            self.plans[unit].run(self.tsteps)

    def close(self):
        for pl in self.plans.values():
            pl.close()
        self.plans = {}

    def host_buffers(self):
        t = self.torch
        return {"u": t.empty(self.u.shape, dtype=t.float64, pin_memory=True).copy_(self.u),
                "v": t.empty(self.u.shape, dtype=t.float64, pin_memory=True).copy_(self.u)}

    def e2e_step(self, h, unit):
        if self.world > 1:
            self.u.copy_(h["u"], non_blocking=True)
            self.v.copy_(self.u)
            self.step(unit)
            h["v"].copy_(self.u if self.tsteps % 2 == 0 else self.v, non_blocking=True)
            self.torch.cuda.current_stream().synchronize()
            return
        self.P.stencil_host(self.preset, h["u"], h["v"], self.tsteps, unit=unit)

    def h2d_d2h(self, h):
        return h["u"].numel() * 8, h["u"].numel() * 8


def make(name, torch, P, D, rank, world, comm=None):
    if name == "spmv":
        return Spmv(torch, P, D, rank, world, comm)
    if name == "stream":
        return Stream(torch, P, D, rank, world, comm)
    return Stencil(torch, P, D, rank, world, name, comm)


def time_steps(torch, wl, unit, steps, warmup, world):
    """W untimed steps, then exactly K timed steps bracketed by barrier+sync;
    per-step CUDA events on the launching (current) stream.  Returns
    (max-over-ranks total ms, list of per-step ms on this rank)."""
    import torch.distributed as dist

    for _ in range(warmup):
        wl.step(unit)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    ev[0].record()
    for i in range(steps):
        wl.step(unit)
        ev[i + 1].record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    per = [ev[i].elapsed_time(ev[i + 1]) for i in range(steps)]
    total = ev[0].elapsed_time(ev[steps])
    if world > 1:
        t = torch.tensor([total], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total = float(t.item())
    return total, per


def fp64_peaks(torch, P):
    """K11: DFMA and DMMA throughput over all SMs (TFLOP/s)."""
    sink = torch.zeros(256, dtype=torch.float64, device="cuda")
    out = {}
    for name, unit, iters in (("cuda_core", P.CUDA_CORE, 20000), ("tensor_core", P.TENSOR_CORE, 20000)):
        P.fp64_peak_launch(unit, 1000, sink)
        torch.cuda.synchronize()
        best = 0.0
        for _ in range(3):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            fl = P.fp64_peak_launch(unit, iters, sink)
            e.record()
            torch.cuda.synchronize()
            best = max(best, fl / (s.elapsed_time(e) * 1e-3) / 1e12)
        out[name] = round(best, 2)
    return out


def _tc_pure_keys(name):
    """Tuning keys that select the paper's full banded tensor-core form (every
    tap on DMMA) instead of the default x-band hybrid."""
    return {"2d5pt": {"stencil_tc2d_hybrid": 0}, "3d7pt": {"stencil_tc3d_hybrid": 0},
            "3d27pt": {"stencil_tc3d_hybrid": 0}}.get(name, {})


def _with_keys(P, keys, fn):
    prev = {k: P.tuning_set(k, v) for k, v in keys.items()}
    try:
        return fn()
    finally:
        for k, v in prev.items():
            P.tuning_set(k, v)


def _time_e2e(torch, wl, unit, reps):
    h = wl.host_buffers()
    bi, bo = wl.h2d_d2h(h)
    wl.e2e_step(h, unit)
    t0 = time.perf_counter()
    for _ in range(reps):
        wl.e2e_step(h, unit)
    el = time.perf_counter() - t0
    if "plan" in h:
        h["plan"].close()
    return {"value": round(wl.job_bytes * reps / el / 1e9, 1), "unit": "GB/s", "h2d_bytes_per_step": bi,
            "d2h_bytes_per_step": bo, "steps": reps}


def per_kernel_table(torch, P, D, hbm):
    rows = {}
    intensity = {
        "stream": P.scale_model(1).intensity,
        "spmv": P.spmv_csr_model(1 << 22, 1 << 22, 1 << 26).intensity,
        "2d5pt": P.stencil_model("2d5pt").intensity,
        "3d7pt": P.stencil_model("3d7pt").intensity,
        "3d27pt": P.stencil_model("3d27pt").intensity,
    }
    for name, spec in WORKLOADS.items():
        wl = make(name, torch, P, D, 0, 1)
        res = {}
        variants = [("cc", P.CUDA_CORE, {}), ("tc", P.TENSOR_CORE, {})]
        if _tc_pure_keys(name):
            variants.append(("tc_pure", P.TENSOR_CORE, _tc_pure_keys(name)))
        if name == "spmv":
            variants += [("cc_csr", P.CUDA_CORE, {}), ("tc_csr", P.TENSOR_CORE, {})]
        for uname, unit, keys in variants:
            if name == "spmv":
                wl.raw_csr = uname.endswith("_csr")
                wl.plan_colsort = 1
            # stencils: 5 runs of the full timestep count, median run (one run is
            # +-5 % noisy on this box; the spread is reported)
            reps = spec["reps"] if name in ("stream", "spmv") else 5
            total, per = _with_keys(P, keys, lambda: time_steps(torch, wl, unit, reps, 2, 1))
            ms = total / reps if name in ("stream", "spmv") else sorted(per)[len(per) // 2]
            gbs = wl.bytes / (ms * 1e-3) / 1e9
            unit_ms = ms if name in ("stream", "spmv") else ms / wl.tsteps
            res[uname] = {"gbs": round(gbs, 1), "frac_of_measured_peak": round(gbs / hbm, 4),
                          "ms_per_unit": round(unit_ms, 4)}
            if name not in ("stream", "spmv"):
                res[uname]["runs"] = reps
                res[uname]["gbs_min_max"] = [round(wl.bytes / (max(per) * 1e-3) / 1e9, 1),
                                             round(wl.bytes / (min(per) * 1e-3) / 1e9, 1)]
            if keys:
                res[uname]["kernel"] = "full banded DMMA form (every tap on the tensor core), tuning " + \
                    ", ".join(f"{k}={v}" for k, v in keys.items())
        if name == "spmv":
            for u, key in (("cc", (P.CUDA_CORE, 1)), ("tc", (P.TENSOR_CORE, 1))):
                layout, lbytes = wl.plans[key].info()
                res[u]["kernel"] = (f"rl_spmv_plan_execute, layout {layout} ({lbytes} B streamed per call; "
                                    + ("K17 column-sorted row blocks, spmv_colsort.cu)" if layout == "colsort"
                                       else "CSR, spmv.cu)"))
            res["plan_create_s"] = round(wl.plan_create_s, 3)
            for u in ("cc_csr", "tc_csr"):
                res[u]["kernel"] = "rl_spmv_csr on the generator's CSR arrays (spmv.cu)"
            # what caps the CSR kernels on this matrix (profiles/README.md): one
            # L1/L2 request per x gather plus one per 128-byte line of val/col,
            # against the measured random-gather rate (tools/micro/dsmem_gather.cu:
            # 1.0 per SM per cycle, 290 G/s at 1.965 GHz)
            m = Spmv.n_local
            reqs = m * Spmv.k + (m * Spmv.k * 12) // 128
            rate = reqs / (res["cc_csr"]["ms_per_unit"] * 1e-3) / 1e9
            res["cc_csr"]["l2_request_roof"] = {"requests_per_step": reqs, "achieved": round(rate, 1),
                                                "peak": 290.0, "unit": "G requests/s",
                                                "frac": round(rate / 290.0, 4)}
            res["plan_over_csr_cc"] = round(res["cc"]["gbs"] / res["cc_csr"]["gbs"], 4)
        res["tc_over_cc"] = round(res["tc"]["gbs"] / res["cc"]["gbs"], 4)
        if "tc_pure" in res:
            res["tc_pure_over_cc"] = round(res["tc_pure"]["gbs"] / res["cc"]["gbs"], 4)
            res["tc"]["kernel"] = "x-band hybrid (x taps on DMMA, centre/y/z taps on DFMA)"
        res["intensity"] = round(intensity[name], 5)
        if name != "spmv":
            # end to end through the host-buffer C-ABI call (rl_scale_host /
            # rl_stencil_host): H2D of the input and D2H of the result inside
            res["e2e_cc"] = _time_e2e(torch, wl, P.CUDA_CORE, 3 if name == "stream" else 1)
        rows[name] = res
        wl.close()
        del wl
        torch.cuda.empty_cache()
    return rows


def cusparse_yardstick(torch, P, hbm, reps=20):
    """cuSPARSE (the paper's CC SpMV baseline)
    is in the image; it is timed here on the same BASELINE matrix as a
    yardstick only (torch's CSR matvec dispatches to cusparseSpMV).  Never
    on the product path."""
    n, k, hb = 1 << 22, 16, 65536
    rp = torch.empty(n + 1, dtype=torch.int32, device="cuda")
    col = torch.empty(n * k, dtype=torch.int32, device="cuda")
    val = torch.empty(n * k, dtype=torch.float64, device="cuda")
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    P.gen_band_csr(n, 0, n, k, hb, SEED, rp, col, val)
    P.fill_uniform(x, SEED, 4, 0, 1)
    try:
        A = torch.sparse_csr_tensor(rp, col, val, size=(n, n))
        xv = x.view(n, 1)
        y = None
        for _ in range(3):
            y = A @ xv
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            y = A @ xv
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / reps
        ours = torch.empty(n, dtype=torch.float64, device="cuda")
        P.spmv_csr(rp, col, val, x, ours)
        torch.cuda.synchronize()
        rel = float(torch.linalg.norm(y.view(-1) - ours) / torch.linalg.norm(ours))
        gbs = P.spmv_csr_model(n, n, n * k).traffic_bytes / (ms * 1e-3) / 1e9
        out = {"gbs": round(gbs, 1), "frac_of_measured_peak": round(gbs / hbm, 4), "ms": round(ms, 4),
               "rel_diff_vs_ours": rel, "via": f"torch {torch.__version__} sparse CSR matvec (cuSPARSE)"}
    except Exception as ex:  # yardstick only: never fail the bench on it
        out = {"unavailable": f"{type(ex).__name__}: {ex}"[:200]}
    del rp, col, val, x
    torch.cuda.empty_cache()
    return out


def temporal_blocking(torch, P, hbm, t1_ms, balance=None):
    """temporal depth t on the BASELINE grids -- 2d5pt
    (16384^2, 100 timesteps) on both units, 3d7pt and 3d27pt (512^3, 50
    timesteps) on the CUDA core: floor(steps/t) fused sweeps + the remainder
    as single steps.  Model bytes are stencil_model(preset, FP64, t): 16 B per
    point per fused sweep (reference kernels.cpp:137-155).  t1_ms: the
    single-step ms per timestep per (preset, unit) from the kernel table.
    min_temporal_depth (bounds.cpp:111-125) at the measured balance is the
    depth from which the fused sweep is compute-bound."""
    out = {}
    runs = (("2d5pt", (16384, 16384), 100, ((2, 3, 4, 5, 7), (2, 3, 4))),
            ("3d7pt", (512, 512, 512), 50, ((2, 3, 4), ())),
            ("3d27pt", (512, 512, 512), 50, ((2, 3, 4), ())))
    for preset, shape, steps, (ds_cc, ds_tc) in runs:
        u = torch.empty(shape, dtype=torch.float64, device="cuda")
        P.stencil_init(u, 1, SEED)
        v = u.clone()
        for uname, unit, ds in (("cc", P.CUDA_CORE, ds_cc), ("tc", P.TENSOR_CORE, ds_tc)):
            for t in ds:
                P.stencil_temporal(preset, u, v, 2 * t, t, unit=unit)
                torch.cuda.synchronize()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                kc, _ = P.stencil_temporal(preset, u, v, steps, t, unit=unit)
                e.record()
                torch.cuda.synchronize()
                ms = s.elapsed_time(e)
                gbs = kc.traffic_bytes / (ms * 1e-3) / 1e9
                row = {"ms_per_timestep": round(ms / steps, 4), "model_gbs": round(gbs, 1),
                       "frac_of_measured_peak": round(gbs / hbm, 4),
                       "tflops": round(kc.work_flops / (ms * 1e-3) / 1e12, 2)}
                t1 = t1_ms.get((preset, uname))
                if t1:
                    row["timestep_speedup_vs_t1"] = round(t1 / (ms / steps), 3)
                out[f"{preset}_t{t}" + ("" if uname == "cc" else "_tc")] = row
        if balance:
            out[f"{preset}_min_temporal_depth"] = P.min_temporal_depth(balance, P.stencil_model(preset).intensity)
        del u, v
        torch.cuda.empty_cache()
    out["note"] = ("2d5pt CC: register-pipelined strips (stencil_tb.cu); 2d5pt TC: overlapped 64x64 tiles in "
                   "shared memory, each level the x-band-on-DMMA form (stencil_tbtc.cu); 3d7pt: register-blocked "
                   "TMA tiles (stencil_tb3r.cu); 3d27pt: t = 2 register-blocked partial-sum planes (stencil_tb27r.cu), "
                   "t = 3, 4 the z-column kernel (stencil_tb3.cu).  One HBM read + write per t timesteps; bytes = stencil_model(t) per fused "
                   "sweep, so model_gbs falls as t rises while the per-timestep time drops")
    return out


def gemv_rows(torch, P, hbm, reps=10):
    """dense GEMV y = A x (gemv_model bytes, kernels.cpp:88-101),
    A 16384 x 65536 FP64 (8 GiB, row-major)."""
    m, n = 16384, 65536
    A = torch.empty((m, n), dtype=torch.float64, device="cuda")
    P.fill_uniform(A.view(-1), SEED, 6, 0, 1)
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    P.fill_uniform(x, SEED, 4, 0, 1)
    y = torch.empty(m, dtype=torch.float64, device="cuda")
    res = {}
    for uname, unit in (("cc", P.CUDA_CORE), ("tc", P.TENSOR_CORE)):
        kc = P.gemv(A, x, y, unit=unit)
        for _ in range(2):
            P.gemv(A, x, y, unit=unit)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            P.gemv(A, x, y, unit=unit)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / reps
        gbs = kc.traffic_bytes / (ms * 1e-3) / 1e9
        res[uname] = {"gbs": round(gbs, 1), "frac_of_measured_peak": round(gbs / hbm, 4), "ms": round(ms, 4)}
    res["tc_over_cc"] = round(res["tc"]["gbs"] / res["cc"]["gbs"], 4)
    res["intensity"] = round(P.gemv_model(m, n).intensity, 5)
    res["config"] = "16384 x 65536 row-major FP64"
    del A
    torch.cuda.empty_cache()
    return res


def stencil_preset_rows(torch, P, hbm, steps=10):
    """the reference's other presets (kernels.cpp:54-58)
    2d9pt / 2d13pt / 2d49pt on the 16384^2 grid, radius-R Dirichlet ring,
    stencil_model bytes (16 B per updated point per step) and flops
    (2 |S| per point).  2d49pt sits at the FP64 ridge."""
    import math
    u = torch.empty((16384, 16384), dtype=torch.float64, device="cuda")
    v = torch.empty_like(u)
    out = {}
    for preset in ("2d9pt", "2d13pt", "2d49pt"):
        npts, r = P.stencil_preset(preset)[1], P.stencil_preset(preset)[2]
        P.stencil_init(u, r, SEED)
        v.copy_(u)
        pts = math.prod(s - 2 * r for s in u.shape)
        res = {}
        for uname, unit in (("cc", P.CUDA_CORE), ("tc", P.TENSOR_CORE)):
            P.stencil(preset, u, v, 2, unit=unit)
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            kc = P.stencil(preset, u, v, steps, unit=unit)
            e.record()
            torch.cuda.synchronize()
            ms = s.elapsed_time(e) / steps
            gbs = kc.traffic_bytes / steps / (ms * 1e-3) / 1e9
            res[uname] = {"gbs": round(gbs, 1), "frac_of_measured_peak": round(gbs / hbm, 4),
                          "tflops": round(kc.work_flops / steps / (ms * 1e-3) / 1e12, 2),
                          "ms_per_step": round(ms, 4)}
        res["tc_over_cc"] = round(res["tc"]["gbs"] / res["cc"]["gbs"], 4)
        res["intensity"] = round(P.stencil_model(preset).intensity, 5)
        res["config"] = f"16384^2, {steps} steps, radius {r}"
        out[preset] = res
    del u, v
    torch.cuda.empty_cache()
    return out


def add_bounds(P, rows, peaks_runs, hbm):
    """TC/CC speedup ceiling per kernel from the measured B200 figures
    (kernel_speedup_ceiling, reference bounds.cpp:72-85).  K11 runs before and
    after the kernel table; alpha moves with the power state, so every bound is
    reported as the range over those runs and `within_bound` uses its top."""
    alphas = [pk["tensor_core"] / pk["cuda_core"] for pk in peaks_runs]
    balances = [pk["cuda_core"] * 1e12 / (hbm * 1e9) for pk in peaks_runs]
    for name, res in rows.items():
        ceils = [P.kernel_speedup_ceiling(max(a, 1.0), bl, res["intensity"])[0] for a, bl in zip(alphas, balances)]
        res["bound"] = round(max(ceils), 4)
        res["bound_range"] = [round(min(ceils), 4), round(max(ceils), 4)]
        res["within_bound"] = bool(res["tc_over_cc"] <= max(ceils) * 1.02)
        if "tc_pure_over_cc" in res:
            res["tc_pure_within_bound"] = bool(res["tc_pure_over_cc"] <= max(ceils) * 1.02)
    return {"alpha": round(alphas[0], 4), "alpha_range": [round(min(alphas), 4), round(max(alphas), 4)],
            "balance_flop_per_byte": round(balances[0], 4),
            "balance_range": [round(min(balances), 4), round(max(balances), 4)],
            "tensor_core_ceiling": round(P.tensor_core_ceiling(max(max(alphas), 1.0)), 4),
            "note": "alpha = measured DMMA/DFMA FP64 peak (K11 before and after the kernel table); ceilings "
                    "from kernel_speedup_ceiling (bounds.cpp:72-85) with alpha clamped to >= 1"}


def cpu_baseline(name, seconds=10.0):
    """Oracle port timed on this host's cores (bounded sample)."""
    import numpy as np

    import oracle as O

    thr = O.num_threads()
    if name == "spmv":
        n, k, hb = 1 << 22, 16, 65536
        rp, col, val = O.gen_band_csr(n, 0, n, k, hb, SEED)
        x = O.fill_uniform(n, SEED, 4, 0, 1)
        nbytes = (n * k + 2 * n) * 8 + (n * k + n + 1) * 4
        fn = lambda: O.spmv_csr(rp, col, val, x)
        sample = "full 2^22-row matrix, repeated SpMV"
    elif name == "stream":
        n = 1 << 27
        b = O.fill_uniform(n, SEED, 1, 0, 1)
        nbytes = 16 * n
        fn = lambda: O.scale(b, 3.0)
        sample = "full 2^27-element Scale, repeated"
    else:
        shape = (16384, 16384) if name == "2d5pt" else (512, 512, 512)
        u0 = O.stencil_init(shape, 1, SEED)
        inner = 1
        for s in shape:
            inner *= s - 2
        nbytes = 16 * inner
        fn = lambda: O.stencil(name, u0, 1)
        sample = f"full BASELINE {shape} grid, 1 timestep per call"
    fn()
    t0 = time.perf_counter()
    calls = 0
    while True:
        fn()
        calls += 1
        el = time.perf_counter() - t0
        if el >= seconds or calls >= 100000:
            break
    gbs = nbytes * calls / el / 1e9
    return {"value": round(gbs, 3), "unit": "GB/s", "cores": thr, "kind": "port",
            "sample": f"{sample}; {calls} calls in {el:.1f} s"}


def workload_bytes(name, world):
    """Per-GPU algorithmic bytes per step: the reference model of the rank's
    share (spmv_csr_model / scale_model / stencil_model, kernels.cpp:74-155)."""
    import math

    import paper_2502_16851_b200 as P

    if name == "spmv":
        m = Spmv.n_local
        return P.spmv_csr_model(m, m, m * Spmv.k).traffic_bytes
    if name == "stream":
        return P.scale_model(Stream.n).traffic_bytes
    shape = (16384, 16384) if name == "2d5pt" else (512, 512, 512)
    return 16 * math.prod(s - 2 for s in shape) * WORKLOADS[name]["reps"]


def make_config(args, world):
    """The `config` object both arms print (identical keys and values)."""
    return {"workload": WORKLOADS[args.workload]["desc"],
            "unit": "cuda_core" if args.unit == "cc" else "tensor_core",
            "parallelism": f"rows/slabs x{world} (NCCL halo exchange)" if world > 1 else "single GPU",
            "l2": "inputs larger than L2 (no flush needed)",
            "algorithmic_bytes_per_step_per_gpu": workload_bytes(args.workload, world),
            "peak_source": hbm_peak()[1]}


def run_reference(args, rank, world):
    """--impl reference: the reference path on the host cores (the reference
    has no executing kernel, so its CPU path is the oracle port)."""
    if rank != 0:
        return
    # all the host threads this process may use (torchrun exports
    # OMP_NUM_THREADS=1 to every rank; the other ranks do no work here)
    os.environ["OMP_NUM_THREADS"] = str(len(os.sched_getaffinity(0)))
    import oracle as O

    name = args.workload
    spec = WORKLOADS[name]
    thr = O.num_threads()
    if name == "spmv":
        n, k, hb = 1 << 22, 16, 65536
        rp, col, val = O.gen_band_csr(n, 0, n, k, hb, SEED)
        x = O.fill_uniform(n, SEED, 4, 0, 1)
        nbytes = (n * k + 2 * n) * 8 + (n * k + n + 1) * 4
        fn = lambda: O.spmv_csr(rp, col, val, x)
        sample = "full 2^22-row BASELINE matrix, one SpMV per step"
    elif name == "stream":
        n = 1 << 27
        b = O.fill_uniform(n, SEED, 1, 0, 1)
        nbytes = 16 * n
        fn = lambda: O.scale(b, 3.0)
        sample = "full 2^27 Scale per step"
    else:
        shape = (16384, 16384) if name == "2d5pt" else (512, 512, 512)
        u0 = O.stencil_init(shape, 1, SEED)
        inner = 1
        for s in shape:
            inner *= s - 2
        nbytes = 16 * inner
        fn = lambda: O.stencil(name, u0, 1)
        sample = f"full {shape} grid, one timestep per step (of {spec['reps']})"
    if world > 1:
        sample += f"; one rank's share of the {world}-GPU weak-scaled job, on rank 0's host cores"
    for _ in range(args.warmup):
        fn()
    t0 = time.perf_counter()
    steps = 0
    budget = 120.0
    for _ in range(args.steps):
        fn()
        steps += 1
        if time.perf_counter() - t0 > budget:
            break
    el = time.perf_counter() - t0
    gbs = nbytes * steps / el / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(gbs, 3), "unit": "GB/s",
        "n_gpus": world, "steps": steps, "warmup": args.warmup,
        "ms_per_step": round(el / steps * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded splitmix64, BASELINE shapes)",
        "config": make_config(args, world),
        "cpu_baseline": {"value": round(gbs, 3), "unit": "GB/s", "cores": thr, "kind": "port",
                         "sample": sample + (f"; stopped after {steps} of {args.steps} steps "
                                             f"({budget:.0f} s budget)" if steps < args.steps else "")},
        "e2e": {"value": round(gbs, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def dist_table(torch, P, D, comm, world, hbm, reps=10):
    """N > 1: every BASELINE config on both units through rl_dist_* (whole-job
    GB/s = global model bytes / max-over-ranks time)."""
    out = {}
    for name in ("stream", "spmv", "2d5pt", "3d7pt", "3d27pt"):
        wl = make(name, torch, P, D, comm.rank, world, comm)
        res = {}
        for uname, unit in (("cc", P.CUDA_CORE), ("tc", P.TENSOR_CORE)):
            r = reps if name in ("stream", "spmv") else 3
            total, _ = time_steps(torch, wl, unit, r, 2, world)
            gbs = wl.job_bytes * r / (total * 1e-3) / 1e9
            res[uname] = {"gbs": round(gbs, 1), "gbs_per_gpu": round(gbs / world, 1),
                          "frac_of_measured_peak_per_gpu": round(gbs / world / hbm, 4),
                          "ms_per_step": round(total / r, 4)}
        res["tc_over_cc"] = round(res["tc"]["gbs"] / res["cc"]["gbs"], 4)
        out[name] = res
        wl.close()
        del wl
        torch.cuda.empty_cache()
    return out


def dist_one_gpu(torch, P, D, hbm):
    """The sharded path on ONE GPU: two parts per rank on a world-1 NCCL
    communicator, halos through NCCL self send/recv inside the same group a
    multi-GPU run posts.  Measures what the C++ step adds over the
    single-launch kernels and its host cost per step (enqueue time of a
    graph-replayed call, no synchronisation)."""
    import math

    comm = D.Comm.single()
    out = {"nccl": comm.info()}
    # SpMV: BASELINE matrix, 2 parts
    n, k, hb, L = 1 << 22, 16, 65536, 2
    tens = []
    for i in range(L):
        p = D.SpmvPartition(n, hb, L, i)
        rp = torch.empty(p.rows + 1, dtype=torch.int32, device="cuda")
        col = torch.empty(p.rows * k, dtype=torch.int32, device="cuda")
        val = torch.empty(p.rows * k, dtype=torch.float64, device="cuda")
        P.gen_band_csr(p.rows, p.r0, n, k, hb, SEED, rp, col, val)
        x = torch.empty(p.window, dtype=torch.float64, device="cuda")
        P.fill_uniform(x, SEED, 4, p.col_base, 1)
        tens.append((rp, col, val, x, torch.empty(p.rows, dtype=torch.float64, device="cuda")))
    plan = D.DistSpmv(comm, n, hb, tens)
    reps = 20
    for _ in range(3):
        plan.execute()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        plan.execute()
    host = (time.perf_counter() - t0) / 10   # includes the ctypes call (~1-2 us)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        plan.execute()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    gbs = P.spmv_csr_model(n, n, n * k).traffic_bytes / (ms * 1e-3) / 1e9
    # the Python -> ctypes call overhead inside host_us_per_call
    t0 = time.perf_counter()
    for _ in range(1000):
        comm.info()
    ctypes_us = (time.perf_counter() - t0) / 1000 * 1e6
    out["spmv_2parts"] = {"gbs": round(gbs, 1), "frac_of_measured_peak": round(gbs / hbm, 4),
                          "ms_per_call": round(ms, 4), "host_us_per_call": round(host * 1e6, 2),
                          "python_call_overhead_us": round(ctypes_us, 2),
                          "halo_bytes_per_call": 2 * 2 * hb * 8}
    plan.close()
    del tens
    torch.cuda.empty_cache()
    # stencils: 2 slabs per GPU, BASELINE grids and timestep counts
    for preset, shape, steps in (("2d5pt", (16384, 16384), 100), ("3d7pt", (512, 512, 512), 50),
                                 ("3d27pt", (512, 512, 512), 50)):
        parts = [D.SlabPartition(preset, shape, L, i) for i in range(L)]
        us = []
        for p in parts:
            u = torch.empty(p.local_shape, dtype=torch.float64, device="cuda")
            P.stencil_init(u, 1, SEED, outer_begin=p.g_lo, global_shape=shape)
            us.append(u)
        vs = [u.clone() for u in us]
        plan = D.DistStencil(comm, preset, shape, us, vs)
        plan.run(2)
        plan.run(steps)
        torch.cuda.synchronize()
        # host cost: enqueue time of a 10-timestep call (short enough that the
        # launch queue never fills, so the host does not wait for the GPU)
        t0 = time.perf_counter()
        plan.run(10)
        host = (time.perf_counter() - t0) / 10
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        kc, _ = plan.run(steps)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e)
        gbs = kc.traffic_bytes / (ms * 1e-3) / 1e9
        layer = math.prod(shape[1:])
        out[f"{preset}_2parts"] = {"gbs": round(gbs, 1), "frac_of_measured_peak": round(gbs / hbm, 4),
                                   "ms_per_timestep": round(ms / steps, 4),
                                   "host_us_per_timestep": round(host * 1e6, 2),
                                   "halo_bytes_per_timestep": 2 * 2 * layer * 8}
        plan.close()
        del us, vs
        torch.cuda.empty_cache()
    comm.close()
    out["note"] = ("rl_dist_* with 2 parts on one GPU (world-1 NCCL, self send/recv); steady-state calls "
                   "replay a captured CUDA graph, host_us = enqueue time per call / timestep")
    return out


def relaunch(args):
    """--gpus N without a torchrun environment: re-exec this command under
    torch.distributed.run with N ranks on 127.0.0.1."""
    import socket

    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="spmv", choices=list(WORKLOADS))
    ap.add_argument("--unit", default="cc", choices=["cc", "tc"])
    ap.add_argument("--no-per-kernel", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=20)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        relaunch(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU "
              f"(torchrun --nproc-per-node {args.gpus}) or drop WORLD_SIZE", file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    import paper_2502_16851_b200 as P
    from paper_2502_16851_b200 import dist as D

    comm = None
    if world > 1:
        # NCCL's init lines (rank, nranks, transport) go to stderr so the
        # JSON line stays alone on stdout
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        dist.init_process_group("nccl")
        P.lib()
        comm = D.Comm.from_env()
    else:
        torch.cuda.set_device(0)
    P.lib()
    hbm, hbm_src = hbm_peak()
    unit = P.CUDA_CORE if args.unit == "cc" else P.TENSOR_CORE

    wl = make(args.workload, torch, P, D, rank, world, comm)
    dev_index = torch.cuda.current_device()
    peaks_runs = []
    if world == 1 and not args.no_per_kernel:
        peaks_runs.append(fp64_peaks(torch, P))   # K11, first of two (alpha range)
        time.sleep(1.0)
    launches0 = P.kernel_launches()
    with ClockSampler(dev_index) as clk:
        # warm-up inside so the sampler sees the GPU under load before timing
        total_ms, per = time_steps(torch, wl, unit, args.steps, args.warmup, world)
    launches = P.kernel_launches() - launches0
    # launches counted over warmup+timed; report timed share
    timed_launches = int(round(launches * args.steps / (args.steps + args.warmup)))
    bytes_per_step_rank = wl.bytes
    value = wl.job_bytes * args.steps / (total_ms * 1e-3) / 1e9
    ms_per_step = total_ms / args.steps
    per_sorted = sorted(per)
    launch_ms = statistics.mean(per)  # one kernel launch per step at N=1
    achieved = bytes_per_step_rank / (launch_ms * 1e-3) / 1e9

    # end to end through the public API with host buffers
    h = wl.host_buffers()
    h2d, d2h = wl.h2d_d2h(h)
    wl.e2e_step(h, unit)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        wl.e2e_step(h, unit)
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_val = wl.job_bytes * args.e2e_steps / e2e_s / 1e9
    e2e_sync = None
    if hasattr(wl, "e2e_stream") and world == 1:
        # the headline e2e: a stream of independent vectors, calls overlapping;
        # the one-call-at-a-time number (the iterative-solver pattern) beside it
        st_s, st_ok = wl.e2e_stream(h, unit, args.e2e_steps)
        e2e_sync = {"value": round(e2e_val, 3), "unit": "GB/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "steps": args.e2e_steps,
                    "api": "rl_spmv_plan_execute_host, one synchronous call per step (each x may depend on the "
                           "previous y)"}
        e2e_val = wl.job_bytes * args.e2e_steps / st_s / 1e9
        e2e_stream_ok = st_ok
    full_copy = None
    if hasattr(wl, "full_copy_step") and world == 1:
        wl.full_copy_step(h, unit)
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            wl.full_copy_step(h, unit)
        fc_s = time.perf_counter() - t0
        fi, fo = wl.full_copy_bytes(h)
        full_copy = {"value": round(wl.job_bytes * args.e2e_steps / fc_s / 1e9, 3), "unit": "GB/s",
                     "h2d_bytes_per_step": fi, "d2h_bytes_per_step": fo,
                     "api": "rl_spmv_csr_host (CSR + x over PCIe every step)"}
    if "plan" in h:
        h["plan"].close()
    del h

    traffic = ncu_traffic().get(f"{args.workload}_{args.unit}")
    api = {"spmv": ("rl_spmv_plan_execute_host: A resident (uploaded once by rl_spmv_plan_create), "
                    "x H2D and y D2H from pinned host memory inside every timed call"),
           }.get(args.workload, "rl_*_host C-ABI (pinned host buffers, copies inside the timed call)")
    if e2e_sync is not None:
        api = ("rl_spmv_plan_execute_host_async + rl_spmv_plan_wait: A resident (uploaded once by "
               "rl_spmv_plan_create); a stream of independent vectors, every step its own x H2D and its own y "
               "D2H from pinned host memory (3 distinct vectors rotated), consecutive calls overlapping; timed "
               "region ends with the wait; results bit-identical to synchronous calls: " +
               ("yes" if e2e_stream_ok else "NO"))
    if world > 1:
        api = ("rl_dist_* plan: the rank's owned input H2D from pinned host memory, the distributed call "
               "(NCCL halo exchange + kernels), the rank's result D2H; max over ranks")
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 5),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded splitmix64 inputs generated in HBM; BASELINE.json shapes)",
        "config": make_config(args, world),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": hbm, "unit": "GB/s",
                     "frac": round(achieved / hbm, 4), "traffic": traffic,
                     "launch_ms_mean": round(launch_ms, 5),
                     "launch_ms_p50": round(per_sorted[len(per_sorted) // 2], 5)},
        "e2e": {"value": round(e2e_val, 3), "unit": "GB/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "steps": args.e2e_steps, "api": api},
        "e2e_sync": e2e_sync,
        "e2e_full_copy": full_copy,
        "gpu_launches": timed_launches,
        "clocks": clk.summary(),
    }
    wl.close()
    del wl
    torch.cuda.empty_cache()

    if world > 1:
        line["dist"] = {"comm": comm.info(), "per_kernel": dist_table(torch, P, D, comm, world, hbm),
                        "halo": {"spmv_bytes_per_call_per_inner_rank": 2 * 2 * Spmv.hb * 8,
                                 "2d_bytes_per_timestep_per_inner_rank": 2 * 2 * 16384 * 8,
                                 "3d_bytes_per_timestep_per_inner_rank": 2 * 2 * 512 * 512 * 8}}
    if world == 1 and not args.no_per_kernel:
        with ClockSampler(dev_index) as clk2:
            table = per_kernel_table(torch, P, D, hbm)
            table["spmv"]["cusparse_cc_yardstick"] = cusparse_yardstick(torch, P, hbm)
            t1 = {(pr, un): table[pr][un]["ms_per_unit"] for pr in ("2d5pt", "3d7pt", "3d27pt") for un in ("cc", "tc")}
            pk0 = peaks_runs[0] if peaks_runs else None
            line["temporal_blocking"] = temporal_blocking(
                torch, P, hbm, t1, pk0["cuda_core"] * 1e12 / (hbm * 1e9) if pk0 else None)
            line["next_rows"] = {"gemv": gemv_rows(torch, P, hbm), **stencil_preset_rows(torch, P, hbm)}
            line["dist_one_gpu"] = dist_one_gpu(torch, P, D, hbm)
        # K11 again at the end (after the power-capped stretch): alpha range
        peaks_runs.append(fp64_peaks(torch, P))
        bounds = add_bounds(P, table, peaks_runs, hbm)
        add_bounds(P, line["next_rows"], peaks_runs, hbm)
        # temporal rows on both units: TC/CC per depth against the kernel ceiling
        # at the fused sweep's intensity t * I1 (bounds.cpp:72-85)
        tb = line["temporal_blocking"]
        i1 = P.stencil_model("2d5pt").intensity
        for t in (2, 3, 4):
            cc, tc = tb.get(f"2d5pt_t{t}"), tb.get(f"2d5pt_t{t}_tc")
            if cc and tc:
                tb[f"2d5pt_t{t}_tc"]["tc_over_cc"] = round(cc["ms_per_timestep"] / tc["ms_per_timestep"], 4)
                ceils = [P.kernel_speedup_ceiling(max(pk["tensor_core"] / pk["cuda_core"], 1.0),
                                                  pk["cuda_core"] * 1e12 / (hbm * 1e9), t * i1)[0] for pk in peaks_runs]
                tb[f"2d5pt_t{t}_tc"]["bound"] = round(max(ceils), 4)
        peaks = peaks_runs[0]
        balance = peaks["cuda_core"] * 1e12 / (hbm * 1e9)
        for res in line["next_rows"].values():
            # which roof binds the CUDA-core form: HBM below the ridge, the DFMA pipe above
            res["roof"] = "fp64" if res["intensity"] > balance else "hbm"
            if "tflops" in res.get("cc", {}):
                res["cc"]["frac_of_fp64_peak"] = round(res["cc"]["tflops"] / peaks["cuda_core"], 4)
                res["tc"]["frac_of_fp64_peak"] = round(res["tc"]["tflops"] / peaks["tensor_core"], 4)
        line["per_kernel"] = table
        line["fp64_peaks_tflops"] = peaks
        line["fp64_peaks_tflops_runs"] = peaks_runs
        line["bounds"] = bounds
        # the measured B200 as a reference-schema spec document (serialize_spec,
        # hardware.cpp:249-264); profiles/B200-measured.json is this object
        spec = P.HardwareSpec("B200-measured", hbm * 1e9, 126e6, peaks["cuda_core"] * 1e12,
                              peaks["tensor_core"] * 1e12)
        line["hardware_spec"] = json.loads(P.serialize_spec(spec))
        line["per_kernel_clocks"] = clk2.summary()
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.workload)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
