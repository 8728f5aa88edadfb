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
# configs "unit:vec:shape,..." (default: the sweep below)
cfgs = [tuple(c.split(":")) for c in sys.argv[1].split(",")] if len(sys.argv) > 1 else \
    [("cc", "2", "11", "2"), ("cc", "4", "10", "2"), ("cc", "4", "16", "2"), ("tc", "2", "13", "2"),
     ("tc", "4", "16", "2")]
cfgs = [(c[0], int(c[1]), int(c[2]), int(c[3]) if len(c) > 3 else 1, int(c[4]) if len(c) > 4 else 1)
        for c in cfgs]  # unit, vec, shape, spread, fuse


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


plans = {}
for u, v, sp in sorted({(c[0], c[1], c[3]) for c in cfgs}):
    P.tuning_set("spmv_colsort_vec", v)
    P.tuning_set("spmv_colsort_spread", sp)
    plans[(u, v, sp)] = P.SpmvPlan(hrp, hcol, hval, n, unit=P.TENSOR_CORE if u == "tc" else P.CUDA_CORE)
P.tuning_set("spmv_colsort_vec", 2)
P.tuning_set("spmv_colsort_spread", 1)
res = {}
# interleaved at call granularity (clocks and power drift under load): every
# round calls each config once between its own pair of events
N = int(os.environ.get("ROUNDS", "400"))
evs = {c: [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(N)] for c in cfgs}
for c in cfgs:  # warm
    P.tuning_set(f"spmv_colsort_{c[0]}_shape", c[2])
    P.tuning_set("spmv_colsort_fuse", c[4])
    for _ in range(3):
        plans[(c[0], c[1], c[3])].execute(x, y)
torch.cuda.synchronize()
BURST = int(os.environ.get("BURST", "1"))  # back-to-back calls between one event pair (bench-like when > 1)
for r in range(N):
    for c in cfgs:
        u, v, sh, sp, fu = c
        P.tuning_set(f"spmv_colsort_{u}_shape", sh)
        P.tuning_set("spmv_colsort_fuse", fu)
        a, b = evs[c][r]
        a.record()
        for _ in range(BURST):
            plans[(u, v, sp)].execute(x, y)
        b.record()
torch.cuda.synchronize()
for c in cfgs:
    res[c] = [a.elapsed_time(b) / BURST for a, b in evs[c]]
for u, v, sh, sp, fu in cfgs:
    P.tuning_set(f"spmv_colsort_{u}_shape", sh)
    P.tuning_set("spmv_colsort_fuse", fu)
    pl = plans[(u, v, sp)]
    pl.execute(x, y); torch.cuda.synchronize(); y1 = y.clone()
    pl.execute(x, y); torch.cuda.synchronize()
    rel = float((y - yref).norm() / yref.norm())
    r = sorted(res[(u, v, sh, sp, fu)])
    ms = r[len(r) // 2]
    print(f"{u} vec {v} shape {sh} spread {sp} fuse {fu}: median {ms:.4f} ms min {r[0]:.4f} {B / ms / 1e6:.0f} GB/s "
          f"rel {rel:.2e} identical {bool(torch.equal(y, y1))}", flush=True)
