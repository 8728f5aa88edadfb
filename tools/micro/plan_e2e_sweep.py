"""rl_spmv_plan_execute_host on the BASELINE matrix (pinned x / y, graph
replay): pipeline chunks x x-upload pieces x y-download groups, plus the PCIe
copy floors (x alone up, y alone down, both at once) in the same process."""
import os
os.environ.setdefault("RL_DEV_TUNING", "1")
import sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2502_16851_b200 as P
n, k, hb = 1 << 22, 16, 65536
rp = torch.empty(n + 1, dtype=torch.int32, device="cuda"); col = torch.empty(n * k, dtype=torch.int32, device="cuda")
val = torch.empty(n * k, dtype=torch.float64, device="cuda"); x = torch.empty(n, dtype=torch.float64, device="cuda")
P.gen_band_csr(n, 0, n, k, hb, 1, rp, col, val); P.fill_uniform(x, 1, 4, 0, 1)
pin = lambda t: t.cpu().pin_memory()
hrp, hcol, hval, hx = pin(rp), pin(col), pin(val), pin(x)
hy = torch.empty(n, dtype=torch.float64).pin_memory()
dy = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def wall(fn, reps=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


def up():
    with torch.cuda.stream(s1):
        x.copy_(hx, non_blocking=True)
    s1.synchronize()


def down():
    with torch.cuda.stream(s2):
        hy.copy_(dy, non_blocking=True)
    s2.synchronize()


def both():
    with torch.cuda.stream(s1):
        x.copy_(hx, non_blocking=True)
    with torch.cuda.stream(s2):
        hy.copy_(dy, non_blocking=True)
    s1.synchronize(); s2.synchronize()


print(f"floors: H2D 32 MiB {wall(up):.3f} ms, D2H {wall(down):.3f} ms, both {wall(both):.3f} ms", flush=True)
cfgs = [a.split(":") for a in sys.argv[1:]] or [["8", "0", "0"], ["8", "2", "0"], ["8", "3", "0"], ["8", "4", "0"],
                                                 ["8", "0", "2"], ["8", "0", "4"], ["4", "0", "0"], ["4", "2", "2"],
                                                 ["6", "0", "0"], ["6", "3", "3"], ["12", "0", "0"], ["12", "3", "3"]]
for c in cfgs:
    ch, xp, yg = (int(v) for v in c[:3])
    nb, eb = (int(c[3]) if len(c) > 3 else 0), (int(c[4]) if len(c) > 4 else 0)
    tp = int(c[5]) if len(c) > 5 else 0
    zc = int(c[6]) if len(c) > 6 else 0
    P.tuning_set("spmv_plan_probe_nocompute", int(c[7]) if len(c) > 7 else 0)
    P.tuning_set("spmv_plan_taper", tp)
    P.tuning_set("spmv_plan_zero_copy", zc)
    P.tuning_set("spmv_plan_colsort_blocks", nb)
    P.tuning_set("spmv_plan_edge_blocks", eb)
    P.tuning_set("spmv_plan_colsort_chunks", ch)
    P.tuning_set("spmv_plan_xpieces", xp)
    P.tuning_set("spmv_plan_ygroups", yg)
    plan = P.SpmvPlan(hrp, hcol, hval, n)
    ms = min(wall(lambda: plan.execute_host(hx, hy)) for _ in range(3))
    dev = min(wall(lambda: plan.execute(x, dy), reps=200) for _ in range(3))
    print(f"chunks {ch} xpieces {xp} ygroups {yg} blocks {nb} edge {eb} taper {tp} zero-copy y {zc} no-compute {int(c[7]) if len(c) > 7 else 0}: e2e {ms:.3f} ms/call "
          f"{889192452 / ms / 1e6:.1f} GB/s; device {dev:.4f} ms", flush=True)
    plan.close()
