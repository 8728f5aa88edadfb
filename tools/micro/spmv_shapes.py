"""K17 CTA shapes (spmv_colsort_{cc,tc}_shape) for both units on the BASELINE
matrix: plan execute, device x/y, CUDA events, best of 3 x 200 calls, plus
norm-wise error against the CSR kernel and call-to-call identity."""
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
shapes = [int(a) for a in sys.argv[1].split(",")] if len(sys.argv) > 1 else [0, 1, 4, 5, 6, 7, 8, 9]
units = sys.argv[2].split(",") if len(sys.argv) > 2 else ["tc", "cc"]


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


plans = {u: P.SpmvPlan(hrp, hcol, hval, n, unit=P.TENSOR_CORE if u == "tc" else P.CUDA_CORE) for u in units}
res = {}
for rnd in range(int(os.environ.get("ROUNDS", "15"))):  # interleaved short bursts: clocks drift under load
    for u in units:
        for sh in shapes:
            P.tuning_set(f"spmv_colsort_{u}_shape", sh)
            ms = timeit(lambda: plans[u].execute(x, y), reps=30)
            res.setdefault((u, sh), []).append(ms)
for u in units:
    for sh in shapes:
        P.tuning_set(f"spmv_colsort_{u}_shape", sh)
        plans[u].execute(x, y); torch.cuda.synchronize(); y1 = y.clone()
        plans[u].execute(x, y); torch.cuda.synchronize()
        rel = float((y - yref).norm() / yref.norm())
        ms = sorted(res[(u, sh)])[len(res[(u, sh)]) // 2]
        print(f"{u} shape {sh}: median {ms:.4f} ms min {min(res[(u, sh)]):.4f} {B / ms / 1e6:.0f} GB/s "
              f"rel {rel:.2e} identical {bool(torch.equal(y, y1))}", flush=True)
    P.tuning_set(f"spmv_colsort_{u}_shape", 0)
