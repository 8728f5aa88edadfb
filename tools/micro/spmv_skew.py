"""SpMV on skewed row-length matrices (power-law, a few dense rows) vs
cuSPARSE via torch: checks the CSR kernels' load balance beyond the
uniform BASELINE matrix."""
import os
os.environ.setdefault("RL_DEV_TUNING", "1")  # sweep knobs (rl_tuning_set developer keys)
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import paper_2502_16851_b200 as P
P.library_path = os.environ.get("RL_LIB", P.library_path)


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def build(lens, n, rng):
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    nnz = int(rp[-1])
    col = np.empty(nnz, np.int32)
    # random sorted columns per row (vectorised: random then sort within rows via key)
    raw = rng.integers(0, n, nnz, dtype=np.int64)
    rowid = np.repeat(np.arange(len(lens)), lens)
    order = np.lexsort((raw, rowid))
    col[:] = raw[order]
    return rp.astype(np.int32), col, rng.uniform(-1, 1, nnz)


rng = np.random.default_rng(0)
m = n = 1 << 21
cases = {}
cases["uniform16"] = np.full(m, 16)
z = np.minimum(rng.zipf(1.7, m), 200000)
cases["zipf1.7"] = (z * (16 * m / z.sum())).astype(np.int64).clip(0, n)
d = np.full(m, 12)
d[rng.choice(m, 16, replace=False)] = 200000
cases["dense_rows"] = d
for k, v in os.environ.items():  # RLT_<tuning key>=<int>, e.g. RLT_SPMV_LONG_HUGE=2048
    if k.startswith("RLT_"):
        P.tuning_set(k[4:].lower(), int(v))
for name, lens in cases.items():
    rp, col, val = build(lens, n, rng)
    x = torch.from_numpy(rng.uniform(-1, 1, n)).cuda()
    t = [torch.from_numpy(a).cuda() for a in (rp, col, val)]
    y = torch.empty(m, dtype=torch.float64, device="cuda")
    nb = P.spmv_csr_model(m, n, int(rp[-1])).traffic_bytes
    out = {"case": name, "nnz": int(rp[-1]), "max_row": int(lens.max())}
    for uname, unit in (("cc", P.CUDA_CORE), ("tc", P.TENSOR_CORE)):
        ms = timeit(lambda: P.spmv_csr(t[0], t[1], t[2], x, y, unit=unit))
        out[uname] = {"ms": round(ms, 4), "gbs": round(nb / ms / 1e6, 1)}
    A = torch.sparse_csr_tensor(t[0], t[1], t[2], size=(m, n))
    ms = timeit(lambda: A @ x.view(n, 1))
    out["cusparse"] = {"ms": round(ms, 4), "gbs": round(nb / ms / 1e6, 1)}
    ref = (A @ x.view(n, 1)).view(-1)
    P.spmv_csr(t[0], t[1], t[2], x, y)
    out["relerr"] = float(torch.linalg.norm(y - ref) / torch.linalg.norm(ref))
    print(out, flush=True)
