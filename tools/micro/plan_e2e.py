"""rl_spmv_plan_execute_host timing vs chunk count / zero-copy (BASELINE matrix)."""
import os
os.environ.setdefault("RL_DEV_TUNING", "1")  # sweep knobs (rl_tuning_set developer keys)
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import oracle as O
import paper_2502_16851_b200 as P
n, k, hb = 1 << 22, 16, 65536
rp = torch.empty(n + 1, dtype=torch.int32, device="cuda"); col = torch.empty(n * k, dtype=torch.int32, device="cuda")
val = torch.empty(n * k, dtype=torch.float64, device="cuda"); x = torch.empty(n, dtype=torch.float64, device="cuda")
P.gen_band_csr(n, 0, n, k, hb, 1, rp, col, val); P.fill_uniform(x, 1, 4, 0, 1)
yref = torch.empty(n, dtype=torch.float64, device="cuda"); P.spmv_csr(rp, col, val, x, yref); yref = yref.cpu().numpy()
pin = lambda t: t.cpu().pin_memory()
hrp, hcol, hval, hx = pin(rp), pin(col), pin(val), pin(x)
for zc in (0, 1):
    for chunks in (2, 4, 8, 16):
        P.tuning_set("spmv_plan_zero_copy", zc)
        P.tuning_set("spmv_plan_chunks", chunks)
        hy = torch.full((n,), float("nan"), dtype=torch.float64).pin_memory()
        plan = P.SpmvPlan(hrp, hcol, hval, n)
        plan.execute_host(hx, hy)
        t0 = time.perf_counter()
        for _ in range(20):
            plan.execute_host(hx, hy)
        dt = (time.perf_counter() - t0) / 20
        err = O.rel_err(hy.numpy(), yref)
        print(f"zero_copy {zc} chunks {chunks:3d}: {dt*1e3:.3f} ms/step  {889192452/dt/1e9:.1f} GB/s  relerr {err:.1e}")
        plan.close()
