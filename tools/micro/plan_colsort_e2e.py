"""rl_spmv_plan_execute_host on the column-sorted layout (K17): chunk count x
compute streams x taper, BASELINE matrix, pinned x/y (graph replay)."""
import os
os.environ.setdefault("RL_DEV_TUNING", "1")  # sweep knobs (rl_tuning_set developer keys)
import sys, time
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
t0 = time.perf_counter()
configs = [(c, s, t) for c in (6, 8, 10, 12) for t in (0, 1, 3, 7) for s in (1,)]
if len(sys.argv) > 1:  # e.g. "8,1,1 6,1,1": chunks,streams,taper triples
    configs = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]]
for chunks, streams, taper in configs:
    zc = 0
    P.tuning_set("spmv_plan_taper", taper)
    P.tuning_set("spmv_plan_colsort_chunks", chunks)
    P.tuning_set("spmv_plan_streams", streams)
    P.tuning_set("spmv_plan_taper", taper)
    hy = torch.full((n,), float("nan"), dtype=torch.float64).pin_memory()
    t1 = time.perf_counter()
    plan = P.SpmvPlan(hrp, hcol, hval, n)
    tc = time.perf_counter() - t1
    plan.execute_host(hx, hy)
    t1 = time.perf_counter()
    for _ in range(20):
        plan.execute_host(hx, hy)
    dt = (time.perf_counter() - t1) / 20
    err = O.rel_err(hy.numpy(), yref)
    print(f"{plan.layout()} chunks {chunks:3d} streams {streams} taper {taper}: {dt*1e3:.3f} ms/call "
          f"{889192452/dt/1e9:.1f} GB/s relerr {err:.1e} (create {tc:.2f} s)", flush=True)
    plan.close()
