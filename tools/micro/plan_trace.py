"""One traced rl_spmv_plan_execute_host call per chunk count (RL_PLAN_TRACE=1
prints event times in us: x pieces on s_in, chunk begin/end on s_cmp, y
chunks on s_out) plus the steady-state time of 20 calls."""
import os
os.environ.setdefault("RL_DEV_TUNING", "1")  # sweep knobs (rl_tuning_set developer keys)
import os, sys, time
if os.environ.get("TRACE", "1") == "1":
    os.environ["RL_PLAN_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2502_16851_b200 as P
n, k, hb = 1 << 22, 16, 65536
rp = torch.empty(n + 1, dtype=torch.int32, device="cuda"); col = torch.empty(n * k, dtype=torch.int32, device="cuda")
val = torch.empty(n * k, dtype=torch.float64, device="cuda"); x = torch.empty(n, dtype=torch.float64, device="cuda")
P.gen_band_csr(n, 0, n, k, hb, 1, rp, col, val); P.fill_uniform(x, 1, 4, 0, 1)
pin = lambda t: t.cpu().pin_memory()
hrp, hcol, hval, hx = pin(rp), pin(col), pin(val), pin(x)
hy = torch.empty(n, dtype=torch.float64).pin_memory()
for arg in (sys.argv[1:] or ["8", "16", "32"]):
    chunks, _, taper = arg.partition(":")
    chunks = int(chunks)
    P.tuning_set("spmv_plan_chunks", chunks)
    P.tuning_set("spmv_plan_colsort_chunks", chunks)
    P.tuning_set("spmv_plan_taper", int(taper or 1))
    plan = P.SpmvPlan(hrp, hcol, hval, n)
    for _ in range(3):
        plan.execute_host(hx, hy)
    sys.stderr.flush()
    t0 = time.perf_counter()
    for _ in range(20):
        plan.execute_host(hx, hy)
    dt = (time.perf_counter() - t0) / 20
    print(f"chunks {arg}: {dt*1e3:.3f} ms/call {889192452/dt/1e9:.1f} GB/s", flush=True)
    plan.close()
