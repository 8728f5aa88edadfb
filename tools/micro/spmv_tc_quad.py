"""K17 tensor-core step: two quadrant DMMA per warp step on the 64-bit grid
(spmv_colsort_fixed = 2) against the FP64 tensor-core pass (fixed = 1: the
tensor-core plan keeps FP64 atomics, 4 masked DMMA after two unpermuting
shuffles) and the CUDA-core plan.  BASELINE matrix, device x/y, CUDA events."""
import os
os.environ.setdefault("RL_DEV_TUNING", "1")
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2502_16851_b200 as P

n, k, hb = 1 << 22, 16, 65536
rp = torch.empty(n + 1, dtype=torch.int32, device="cuda"); col = torch.empty(n * k, dtype=torch.int32, device="cuda")
val = torch.empty(n * k, dtype=torch.float64, device="cuda"); x = torch.empty(n, dtype=torch.float64, device="cuda")
y = torch.empty(n, dtype=torch.float64, device="cuda"); yref = torch.empty_like(y)
P.gen_band_csr(n, 0, n, k, hb, 1, rp, col, val); P.fill_uniform(x, 1, 4, 0, 1)
B = 889192452
hrp, hcol, hval = rp.cpu(), col.cpu(), val.cpu()
P.spmv_csr(rp, col, val, x, yref, unit=P.CUDA_CORE)
torch.cuda.synchronize()


def timeit(fn, reps=200):
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


shapes = {0: "1024x3", 1: "768x3", 2: "512x4", 3: "512x6", 4: "1024x2"}
runs = [(2, P.TENSOR_CORE, f"tc grid (2 quadrant DMMA) CTA {v}", sh) for sh, v in shapes.items()]
runs += [(1, P.TENSOR_CORE, "tc fp64 (shuffles + 4 DMMA)", 0), (2, P.CUDA_CORE, "cc grid", 0)]
for fixed, unit, name, sh in runs:
    P.tuning_set("spmv_colsort_fixed", fixed)
    P.tuning_set("spmv_colsort_tc_shape", sh)
    plan = P.SpmvPlan(hrp, hcol, hval, n, unit=unit)
    plan.execute(x, y)
    torch.cuda.synchronize()
    y1 = y.clone()
    ms = min(timeit(lambda: plan.execute(x, y)) for _ in range(3))
    rel = float((y - yref).norm() / yref.norm())
    same = bool(torch.equal(y, y1))
    print(f"{name}: {ms:.4f} ms {B / ms / 1e6:.0f} GB/s rel {rel:.2e} repeat-identical {same}", flush=True)
    plan.close()
P.tuning_set("spmv_colsort_fixed", 2)
