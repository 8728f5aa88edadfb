"""K17 stress: random CSR matrices (ragged rows, empty rows, dense and sparse
bands, rectangular, spikes and cancelling rows) through SpmvPlan on both
units x layout knobs (vec 1/2/4, parity order 0/1/2, fused flagged rows 0/1),
each result against the oracle at 1e-12 and bit-identical on a repeat."""
import os, sys
os.environ.setdefault("RL_DEV_TUNING", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import oracle as O
import paper_2502_16851_b200 as P

rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
cases = int(sys.argv[2]) if len(sys.argv) > 2 else 60
bad = 0
for c in range(cases):
    m = int(rng.integers(1, 60000))
    n = int(rng.integers(1, 60000)) if rng.random() < 0.3 else m
    maxlen = int(rng.choice([1, 4, 16, 40, 200]))
    lens = rng.integers(0, maxlen + 1, size=m)
    lens[rng.random(m) < rng.random() * 0.5] = 0
    lens = np.minimum(lens, n)
    band = int(rng.choice([8, 300, 5000, n]))
    rp = np.zeros(m + 1, np.int64); rp[1:] = np.cumsum(lens)
    cols = []
    for i, L in enumerate(lens):
        lo, hi = max(0, min(i, n - 1) - band), min(n, min(i, n - 1) + band + 1)
        L = min(L, hi - lo)
        cols.append(np.sort(rng.choice(np.arange(lo, hi), size=L, replace=False)) if L else np.zeros(0, np.int64))
        lens[i] = L
    rp[1:] = np.cumsum(lens)
    col = np.concatenate(cols).astype(np.int32) if rp[-1] else np.zeros(0, np.int32)
    val = rng.uniform(-1, 1, rp[-1])
    if rng.random() < 0.3:  # cancelling rows
        for i in range(0, m, 7):
            a, b = rp[i], rp[i + 1]; h = (b - a) // 2
            val[a + h:a + 2 * h] = -val[a:a + h]
    x = rng.uniform(-1, 1, n)
    if rng.random() < 0.3:
        x[rng.integers(0, n, 5)] = 1e10
    rp = rp.astype(np.int32)
    if rp[-1] == 0:
        continue
    want = O.spmv_csr(rp, col, val, x)
    vec, spread, fuse = int(rng.choice([1, 2, 4])), int(rng.choice([0, 1, 2])), int(rng.choice([0, 1]))
    for unit in (P.CUDA_CORE, P.TENSOR_CORE):
        prev = [P.tuning_set("spmv_colsort_vec", vec), P.tuning_set("spmv_colsort_spread", spread)]
        try:
            plan = P.SpmvPlan(rp, col, val, n, unit=unit)
        finally:
            P.tuning_set("spmv_colsort_vec", prev[0]); P.tuning_set("spmv_colsort_spread", prev[1])
        pf = P.tuning_set("spmv_colsort_fuse", fuse)
        try:
            dx = torch.from_numpy(x).cuda()
            outs = []
            for _ in range(2):
                dy = torch.full((m,), float("nan"), dtype=torch.float64, device="cuda")
                plan.execute(dx, dy); torch.cuda.synchronize(); outs.append(dy.cpu().numpy())
            err = O.rel_err(outs[0], want)
            same = np.array_equal(outs[0], outs[1])
            if not (err <= 1e-12 and same):
                bad += 1
                print(f"BAD case {c}: m={m} n={n} maxlen={maxlen} band={band} unit={unit} vec={vec} spread={spread} "
                      f"fuse={fuse} layout={plan.layout()} err={err:.3e} same={same}", flush=True)
        finally:
            P.tuning_set("spmv_colsort_fuse", pf)
            plan.close()
print(f"done: {cases} cases, {bad} bad", flush=True)
