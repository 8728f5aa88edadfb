"""Device-resident time of the execute_host chunk launches alone (no copies):
the whole-matrix launch against the same plan's chunks launched one after
another (spmv_plan_dev_chunks), per block layout."""
import os, sys
os.environ.setdefault("RL_DEV_TUNING", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2502_16851_b200 as P
n, k, hb = 1 << 22, 16, 65536
rp = torch.empty(n + 1, dtype=torch.int32, device="cuda"); col = torch.empty(n * k, dtype=torch.int32, device="cuda")
val = torch.empty(n * k, dtype=torch.float64, device="cuda"); x = torch.empty(n, dtype=torch.float64, device="cuda")
y = torch.empty(n, dtype=torch.float64, device="cuda")
P.gen_band_csr(n, 0, n, k, hb, 1, rp, col, val); P.fill_uniform(x, 1, 4, 0, 1)
hrp, hcol, hval = rp.cpu(), col.cpu(), val.cpu()


def timed(fn, reps=50):
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


for cfg in sys.argv[1:] or ["8:0", "8:1184", "8:2368", "16:2368", "4:0"]:
    ch, nb = (int(v) for v in cfg.split(":"))
    P.tuning_set("spmv_plan_colsort_chunks", ch); P.tuning_set("spmv_plan_colsort_blocks", nb)
    plan = P.SpmvPlan(hrp, hcol, hval, n)
    P.tuning_set("spmv_plan_dev_chunks", 0)
    whole = timed(lambda: plan.execute(x, y))
    P.tuning_set("spmv_plan_dev_chunks", 1)
    chunked = timed(lambda: plan.execute(x, y))
    P.tuning_set("spmv_plan_dev_chunks", 0)
    print(f"chunks {ch} blocks {nb}: whole {whole:.4f} ms, chunk launches {chunked:.4f} ms ({chunked / ch * 1e3:.1f} us per chunk)", flush=True)
    plan.close()
