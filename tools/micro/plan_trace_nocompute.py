import os, sys
os.environ["RL_DEV_TUNING"] = "1"; os.environ["RL_PLAN_TRACE"] = "1"
sys.path.insert(0, os.getcwd())
import torch, paper_2502_16851_b200 as P
n, k, hb = 1 << 22, 16, 65536
rp = torch.empty(n + 1, dtype=torch.int32, device="cuda"); col = torch.empty(n * k, dtype=torch.int32, device="cuda")
val = torch.empty(n * k, dtype=torch.float64, device="cuda"); x = torch.empty(n, dtype=torch.float64, device="cuda")
P.gen_band_csr(n, 0, n, k, hb, 1, rp, col, val); P.fill_uniform(x, 1, 4, 0, 1)
pin = lambda t: t.cpu().pin_memory()
hrp, hcol, hval, hx = pin(rp), pin(col), pin(val), pin(x)
hy = torch.empty(n, dtype=torch.float64).pin_memory()
plan = P.SpmvPlan(hrp, hcol, hval, n)
for nc in (1, 0):
    P.tuning_set("spmv_plan_probe_nocompute", nc)
    print("nocompute", nc, file=sys.stderr, flush=True)
    for _ in range(3):
        plan.execute_host(hx, hy)
