"""rl_spmv_plan_execute_host_async on the BASELINE matrix: host enqueue time
per call, device-side per-call period in a stream of independent vectors, and
the traced copy timeline of the steady state (RL_PLAN_TRACE-like events on
the plan streams are not available here: we time with wall clock + events on
the default stream around waits)."""
import os, sys, time
os.environ.setdefault("RL_DEV_TUNING", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2502_16851_b200 as P
n, k, hb = 1 << 22, 16, 65536
rp = torch.empty(n + 1, dtype=torch.int32, device="cuda"); col = torch.empty(n * k, dtype=torch.int32, device="cuda")
val = torch.empty(n * k, dtype=torch.float64, device="cuda"); x = torch.empty(n, dtype=torch.float64, device="cuda")
P.gen_band_csr(n, 0, n, k, hb, 1, rp, col, val); P.fill_uniform(x, 1, 4, 0, 1)
pin = lambda t: t.cpu().pin_memory()
hrp, hcol, hval = pin(rp), pin(col), pin(val)
xs = [pin(x) for _ in range(3)]
ys = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(3)]
for cfg in sys.argv[1:] or ["8", "4", "16", "2"]:
    P.tuning_set("spmv_plan_colsort_chunks", int(cfg))
    plan = P.SpmvPlan(hrp, hcol, hval, n)
    for r in range(6):
        plan.execute_host_async(xs[r % 3], ys[r % 3])
    plan.wait()
    K = 30
    t0 = time.perf_counter()
    for r in range(K):
        plan.execute_host_async(xs[r % 3], ys[r % 3])
    t1 = time.perf_counter()
    plan.wait()
    t2 = time.perf_counter()
    print(f"chunks {cfg}: host enqueue {(t1 - t0) / K * 1e3:.3f} ms/call, period {(t2 - t0) / K * 1e3:.3f} ms/call "
          f"({889192452 * K / (t2 - t0) / 1e9:.0f} GB/s)", flush=True)
    plan.close()
