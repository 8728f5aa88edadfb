"""Zipf-matrix SpMV a few times (for an ncu launch list of the per-row and
long-row kernels)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2502_16851_b200 as P
rng = np.random.default_rng(0)
m = n = 1 << 21
z = np.minimum(rng.zipf(1.7, m), 200000)
lens = (z * (16 * m / z.sum())).astype(np.int64).clip(0, n)
rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
nnz = int(rp[-1])
raw = rng.integers(0, n, nnz, dtype=np.int64)
rowid = np.repeat(np.arange(m), lens)
col = raw[np.lexsort((raw, rowid))].astype(np.int32)
t = [torch.from_numpy(a).cuda() for a in (rp.astype(np.int32), col, rng.uniform(-1, 1, nnz))]
x = torch.from_numpy(rng.uniform(-1, 1, n)).cuda()
y = torch.empty(m, dtype=torch.float64, device="cuda")
print("rows > 64:", int((lens > 64).sum()), "nnz in them:", int(lens[lens > 64].sum()), "of", nnz)
for _ in range(4):
    P.spmv_csr(t[0], t[1], t[2], x, y)
torch.cuda.synchronize()
