"""Three rl_spmv_plan_execute calls on the BASELINE matrix (for ncu captures).
python tools/micro/prof_colsort.py [spmv_colsort_fixed 0|1] [unit cc|tc]"""
import os
import sys

os.environ["RL_DEV_TUNING"] = "1"
sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import paper_2502_16851_b200 as P  # noqa: E402

n, k, hb = 1 << 22, 16, 65536
rp = torch.empty(n + 1, dtype=torch.int32, device="cuda"); col = torch.empty(n * k, dtype=torch.int32, device="cuda")
val = torch.empty(n * k, dtype=torch.float64, device="cuda"); x = torch.empty(n, dtype=torch.float64, device="cuda")
y = torch.empty(n, dtype=torch.float64, device="cuda")
P.gen_band_csr(n, 0, n, k, hb, 1, rp, col, val); P.fill_uniform(x, 1, 4, 0, 1)
if len(sys.argv) > 1:
    P.tuning_set("spmv_colsort_fixed", int(sys.argv[1]))
unit = P.TENSOR_CORE if len(sys.argv) > 2 and sys.argv[2] == "tc" else P.CUDA_CORE
plan = P.SpmvPlan(rp.cpu(), col.cpu(), val.cpu(), n, unit=unit)
for _ in range(3):
    plan.execute(x, y)
torch.cuda.synchronize()
