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
for cfg in sys.argv[1:]:
    ch, eb, tp, nb = (int(v) for v in (cfg + ":0").split(":")[:4])
    P.tuning_set("spmv_plan_colsort_chunks", ch); P.tuning_set("spmv_plan_edge_blocks", eb); P.tuning_set("spmv_plan_taper", tp)
    P.tuning_set("spmv_plan_colsort_blocks", nb)
    plan = P.SpmvPlan(hrp, hcol, hval, n)
    print("cfg", cfg, "xpieces/chunks", file=sys.stderr, flush=True)
    for _ in range(4):
        plan.execute_host(hx, hy)
    plan.close()
