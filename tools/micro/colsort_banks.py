"""K17 bank-ordering sweep on the BASELINE matrix: group classes (1 = none, 16,
32) x window; python colsort_banks.py [spmv_colsort_fixed] [cc|tc] -- device x
and y, CUDA events."""
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


def timeit(fn, reps=100):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


fixed = int(sys.argv[1]) if len(sys.argv) > 1 else 1
unit = P.TENSOR_CORE if len(sys.argv) > 2 and sys.argv[2] == "tc" else P.CUDA_CORE
P.tuning_set("spmv_colsort_fixed", fixed)
for rnd in range(2):
    for cls in (1, 16, 32):
        for win in (64, 128):
            P.tuning_set("spmv_colsort_classes", cls)
            P.tuning_set("spmv_colsort_window", win)
            plan = P.SpmvPlan(hrp, hcol, hval, n, unit=unit)
            ms = timeit(lambda: plan.execute(x, y))
            print(f"{sys.argv[2:]} fixed {fixed} classes {cls} window {win}: {ms:.4f} ms {B / ms / 1e6:.0f} GB/s", flush=True)
            plan.close()
