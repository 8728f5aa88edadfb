import os, sys
os.environ["RL_DEV_TUNING"] = "1"
sys.path.insert(0, os.getcwd())
import torch
import paper_2502_16851_b200 as P
n, k, hb = 1 << 22, 16, 65536
rp = torch.empty(n + 1, dtype=torch.int32, device="cuda"); col = torch.empty(n * k, dtype=torch.int32, device="cuda")
val = torch.empty(n * k, dtype=torch.float64, device="cuda"); x = torch.empty(n, dtype=torch.float64, device="cuda")
y = torch.empty(n, dtype=torch.float64, device="cuda")
P.gen_band_csr(n, 0, n, k, hb, 1, rp, col, val); P.fill_uniform(x, 1, 4, 0, 1)
P.tuning_set("spmv_colsort_shape", int(sys.argv[1]))
if len(sys.argv) > 2:
    P.tuning_set("spmv_colsort_window", int(sys.argv[2]))
plan = P.SpmvPlan(rp.cpu(), col.cpu(), val.cpu(), n)
for _ in range(3):
    plan.execute(x, y)
torch.cuda.synchronize()
