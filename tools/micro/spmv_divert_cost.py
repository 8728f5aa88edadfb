"""Cost of diverting rows: 2^21 rows of 1 nonzero, every k-th row L long.
L = 64 stays in the per-row kernel, L = 65 is diverted (one list append
each).  Prints ms per call for each (k, L)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import paper_2502_16851_b200 as P

m = n = 1 << 21
rng = np.random.default_rng(0)
for k in (1000, 100, 20):
    for L in (64, 65):
        lens = np.ones(m, np.int64)
        lens[::k] = L
        rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
        col = rng.integers(0, n, int(rp[-1])).astype(np.int32)
        val = rng.uniform(-1, 1, int(rp[-1]))
        t = [torch.from_numpy(a).cuda() for a in (rp, col, val)]
        x = torch.from_numpy(rng.uniform(-1, 1, n)).cuda()
        y = torch.empty(m, dtype=torch.float64, device="cuda")
        for _ in range(3):
            P.spmv_csr(t[0], t[1], t[2], x, y)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(20):
            P.spmv_csr(t[0], t[1], t[2], x, y)
        e.record()
        torch.cuda.synchronize()
        print(f"every {k}th row {L} long ({m // k} such rows): {s.elapsed_time(e) / 20:.4f} ms", flush=True)
