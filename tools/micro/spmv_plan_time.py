"""Device-resident SpMV on the BASELINE matrix: the plan layouts (K17
column-sorted row blocks, CSR) and the raw CSR kernels, both units."""
import os
os.environ.setdefault("RL_DEV_TUNING", "1")
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2502_16851_b200 as P

n, k, hb = 1 << 22, 16, 65536
rp = torch.empty(n + 1, dtype=torch.int32, device="cuda"); col = torch.empty(n * k, dtype=torch.int32, device="cuda")
val = torch.empty(n * k, dtype=torch.float64, device="cuda"); x = torch.empty(n, dtype=torch.float64, device="cuda")
y = torch.empty(n, dtype=torch.float64, device="cuda")
P.gen_band_csr(n, 0, n, k, hb, 1, rp, col, val); P.fill_uniform(x, 1, 4, 0, 1)
B = 889192452
hrp, hcol, hval = rp.cpu(), col.cpu(), val.cpu()


def timeit(fn, reps=50):
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


for win in (64, 128):
    P.tuning_set("spmv_colsort_window", win)
    plan = P.SpmvPlan(hrp, hcol, hval, n)
    ms = timeit(lambda: plan.execute(x, y))
    print(f"plan {plan.layout()} cc window {win}: {ms:.4f} ms {B / ms / 1e6:.0f} GB/s", flush=True)
    plan.close()
P.tuning_set("spmv_colsort_window", 128)
for unit, uname in ((P.CUDA_CORE, "cc"), (P.TENSOR_CORE, "tc")):
    ms = timeit(lambda: P.spmv_csr(rp, col, val, x, y, unit=unit))
    print(f"csr kernel {uname}: {ms:.4f} ms {B / ms / 1e6:.0f} GB/s", flush=True)
    for cs in (1, 0):
        P.tuning_set("spmv_plan_colsort", cs)
        plan = P.SpmvPlan(hrp, hcol, hval, n, unit=unit)
        ms = timeit(lambda: plan.execute(x, y))
        print(f"plan {plan.layout()} {uname}: {ms:.4f} ms {B / ms / 1e6:.0f} GB/s", flush=True)
        plan.close()
    P.tuning_set("spmv_plan_colsort", 1)
