"""rl_spmv_plan_execute_host (BASELINE matrix, pinned x/y, graph path): time per
call vs row chunks, x upload pieces and y copy groups; checks y each config.
python tools/micro/plan_pieces.py "chunks,xpieces,ygroups" ..."""
import os
os.environ.setdefault("RL_DEV_TUNING", "1")  # sweep knobs (rl_tuning_set developer keys)
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2502_16851_b200 as P  # noqa: E402

n, k, hb = 1 << 22, 16, 65536
rp = torch.empty(n + 1, dtype=torch.int32, device="cuda")
col = torch.empty(n * k, dtype=torch.int32, device="cuda")
val = torch.empty(n * k, dtype=torch.float64, device="cuda")
x = torch.empty(n, dtype=torch.float64, device="cuda")
P.gen_band_csr(n, 0, n, k, hb, 1, rp, col, val)
P.fill_uniform(x, 1, 4, 0, 1)
yref = torch.empty(n, dtype=torch.float64, device="cuda")
P.spmv_csr(rp, col, val, x, yref)
yref = yref.cpu().numpy()
hrp, hcol, hval, hx = (t.cpu().pin_memory() for t in (rp, col, val, x))
configs = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]] or [(16, 0, 0)]
plans = []
for ch, xp, yg in configs:
    P.tuning_set("spmv_plan_chunks", ch)
    P.tuning_set("spmv_plan_xpieces", xp)
    P.tuning_set("spmv_plan_ygroups", yg)
    hy = torch.full((n,), float("nan"), dtype=torch.float64).pin_memory()
    plan = P.SpmvPlan(hrp, hcol, hval, n)
    plan.execute_host(hx, hy)
    err = O.rel_err(hy.numpy(), yref)
    plans.append((ch, xp, yg, plan, hy, err, []))
for rd in range(8):  # interleaved rounds
    for ch, xp, yg, plan, hy, err, ts in plans:
        t0 = time.perf_counter()
        for _ in range(5):
            plan.execute_host(hx, hy)
        ts.append((time.perf_counter() - t0) / 5)
for ch, xp, yg, plan, hy, err, ts in plans:
    ts.sort()
    dt = ts[len(ts) // 2]
    print(f"chunks {ch:3d} xpieces {xp:2d} ygroups {yg:2d}: {dt * 1e3:.3f} ms/call  "
          f"{889192452 / dt / 1e9:.1f} GB/s  relerr {err:.1e}", flush=True)
    plan.close()
