"""K16 (column-chunked plan layout) vs the CSR kernel on the BASELINE matrix:
correctness against the CSR kernel and device time per call."""
import os
os.environ.setdefault("RL_DEV_TUNING", "1")  # sweep knobs (rl_tuning_set developer keys)
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2502_16851_b200 as P  # noqa: E402

n, k, hb, seed = 1 << 22, 16, 65536, 2025
rp = torch.empty(n + 1, dtype=torch.int32, device="cuda")
col = torch.empty(n * k, dtype=torch.int32, device="cuda")
val = torch.empty(n * k, dtype=torch.float64, device="cuda")
P.gen_band_csr(n, 0, n, k, hb, seed, rp, col, val)
x = torch.empty(n, dtype=torch.float64, device="cuda")
P.fill_uniform(x, seed, 4, 0, 1)
y = torch.empty(n, dtype=torch.float64, device="cuda")
ref = torch.empty(n, dtype=torch.float64, device="cuda")
P.spmv_csr(rp, col, val, x, ref)
t0 = time.time()
P.tuning_set("spmv_plan_chunked", 1)
plan = P.SpmvPlan(rp.cpu(), col.cpu(), val.cpu(), n)
print("build", round(time.time() - t0, 2), "s layout", plan.layout(), "bytes", plan.info()[1])
model = P.spmv_csr_model(n, n, n * k).traffic_bytes


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


y.fill_(float("nan"))
plan.execute(x, y)
torch.cuda.synchronize()
rel = float(torch.linalg.norm(y - ref) / torch.linalg.norm(ref))
print("rel diff vs CSR kernel", rel, "nan", bool(torch.isnan(y).any()))
for name, fn in (("csr", lambda: P.spmv_csr(rp, col, val, x, ref)), ("chunked", lambda: plan.execute(x, y))):
    ms = timeit(fn)
    print(f"{name}: {ms:.4f} ms  {model / ms / 1e6:.1f} GB/s")
for mode in (1, 2, 3):
    P.tuning_set("spmv_chunked_mode", mode)
    ms = timeit(lambda: plan.execute(x, y))
    print(f"chunked mode {mode}: {ms:.4f} ms")
P.tuning_set("spmv_chunked_mode", 0)
hx = torch.empty(n, dtype=torch.float64).pin_memory().copy_(x)
hy = torch.empty(n, dtype=torch.float64).pin_memory()
plan.execute_host(hx, hy)
t0 = time.perf_counter()
for _ in range(10):
    plan.execute_host(hx, hy)
print("execute_host ms", round((time.perf_counter() - t0) / 10 * 1e3, 3),
      "rel", float(torch.linalg.norm(hy.cuda() - ref) / torch.linalg.norm(ref)))
