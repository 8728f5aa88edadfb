"""Device-side time of the tiled plan kernel vs the CSR kernel (BASELINE matrix)."""
import os
os.environ.setdefault("RL_DEV_TUNING", "1")  # sweep knobs (rl_tuning_set developer keys)
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import oracle as O
import paper_2502_16851_b200 as P
P.library_path = os.environ.get("RL_LIB", P.library_path)
n, k, hb = 1 << 22, 16, 65536
rp = torch.empty(n + 1, dtype=torch.int32, device="cuda"); col = torch.empty(n * k, dtype=torch.int32, device="cuda")
val = torch.empty(n * k, dtype=torch.float64, device="cuda"); x = torch.empty(n, dtype=torch.float64, device="cuda")
y = torch.empty(n, dtype=torch.float64, device="cuda")
P.gen_band_csr(n, 0, n, k, hb, 1, rp, col, val); P.fill_uniform(x, 1, 4, 0, 1)
t0 = time.perf_counter()
P.tuning_set("spmv_plan_tiled", int(os.environ.get("TILED", "1")))
plan = P.SpmvPlan(rp.cpu(), col.cpu(), val.cpu(), n)
print("plan build s", round(time.perf_counter() - t0, 2), "info", plan.info())
def timeit(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps
nb = P.spmv_csr_model(n, n, n * k).traffic_bytes
ms = timeit(lambda: P.spmv_csr(rp, col, val, x, y)); print(f"csr  {ms:.4f} ms {nb/ms/1e6:.0f} GB/s")
y2 = torch.empty_like(y)
ms = timeit(lambda: plan.execute(x, y2)); print(f"plan {ms:.4f} ms {nb/ms/1e6:.0f} GB/s (layout bytes {plan.info()[1]/1e6:.1f} MB)")
print("relerr", O.rel_err(y2.cpu().numpy(), y.cpu().numpy()))
