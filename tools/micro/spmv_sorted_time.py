"""BASELINE SpMV: CSR kernel (rl_spmv_csr) vs the plan's column-sorted block
layout (rl_spmv_plan_execute, device x/y), interleaved; checks both."""
import os
os.environ.setdefault("RL_DEV_TUNING", "1")  # sweep knobs (rl_tuning_set developer keys)
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2502_16851_b200 as P  # noqa: E402

n, k, hb = 1 << 22, 16, 65536
rp = torch.empty(n + 1, dtype=torch.int32, device="cuda")
col = torch.empty(n * k, dtype=torch.int32, device="cuda")
val = torch.empty(n * k, dtype=torch.float64, device="cuda")
x = torch.empty(n, dtype=torch.float64, device="cuda")
P.gen_band_csr(n, 0, n, k, hb, 1, rp, col, val)
P.fill_uniform(x, 1, 4, 0, 1)
y0 = torch.empty(n, dtype=torch.float64, device="cuda")
P.spmv_csr(rp, col, val, x, y0)
hrp, hcol, hval = rp.cpu(), col.cpu(), val.cpu()
plans = {}
P.tuning_set("spmv_plan_sorted", 1)
if os.environ.get("ONLY"):  # one plan, three executes (for ncu)
    P.tuning_set("spmv_sorted_cap", int(os.environ["ONLY"]))
    pl = P.SpmvPlan(hrp, hcol, hval, n)
    yy = torch.empty(n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        pl.execute(x, yy)
    torch.cuda.synchronize()
    sys.exit(0)
for cap in (16384, 12288, 8192):
    P.tuning_set("spmv_sorted_cap", cap)
    import time
    t0 = time.time()
    plans[cap] = P.SpmvPlan(hrp, hcol, hval, n)
    print(f"cap {cap}: layout {plans[cap].layout()}, build {time.time() - t0:.1f} s", flush=True)
P.tuning_set("spmv_sorted_cap", 16384)
ys = {c: torch.empty(n, dtype=torch.float64, device="cuda") for c in plans}
fns = {"csr": lambda: P.spmv_csr(rp, col, val, x, y0)}
for c, pl in plans.items():
    fns[f"sorted{c}"] = (lambda pl=pl, c=c: pl.execute(x, ys[c]))
res = {kk: [] for kk in fns}
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rd in range(8):
    for kk, fn in fns.items():
        fn()
        s.record()
        for _ in range(20):
            fn()
        e.record()
        torch.cuda.synchronize()
        if rd:
            res[kk].append(s.elapsed_time(e) / 20)
for kk, t in res.items():
    t.sort()
    ms = t[len(t) // 2]
    print(f"{kk:12s} {ms * 1e3:7.1f} us  {889192452 / ms / 1e6:7.1f} GB/s", flush=True)
for c in plans:
    err = float(torch.linalg.norm(ys[c] - y0) / torch.linalg.norm(y0))
    print(f"sorted{c} rel diff vs CSR kernel {err:.2e}")
