"""CSR SpMV at the BASELINE size (2^22 rows, 16 nnz/row, +-65536 band):
ms per call for each library in RL_LIBS (comma list; default: the in-tree
build), CUDA core and tensor core, interleaved to cancel clock drift."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import ctypes
import torch
import paper_2502_16851_b200 as P

libs = [l for l in os.environ.get("RL_LIBS", "").split(",") if l] or [P.library_path]
m = n = 1 << 22
rp = torch.empty(m + 1, dtype=torch.int32, device="cuda")
col = torch.empty(16 * m, dtype=torch.int32, device="cuda")
val = torch.empty(16 * m, dtype=torch.float64, device="cuda")
x = torch.empty(n, dtype=torch.float64, device="cuda")
y = torch.empty(m, dtype=torch.float64, device="cuda")
P.gen_band_csr(m, 0, n, 16, 65536, 1, rp, col, val)
P.fill_uniform(x, 1, 4, -1, 1)
model = (16 * m + m + n) * 8 + (16 * m + m + 1) * 4
res = {}
for rnd in range(3):
    for path in libs:
        P.library_path = path
        P._lib = None
        for unit in (P.CUDA_CORE, P.TENSOR_CORE):
            for _ in range(3):
                P.spmv_csr(rp, col, val, x, y, unit=unit)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            s.record()
            for _ in range(20):
                P.spmv_csr(rp, col, val, x, y, unit=unit)
            e.record()
            torch.cuda.synchronize()
            ms = s.elapsed_time(e) / 20
            key = (os.path.basename(path), unit)
            res[key] = min(res.get(key, 1e9), ms)
for (lib, unit), ms in res.items():
    print(f"{lib} unit={unit} {ms:.4f} ms {model / ms / 1e6:.0f} GB/s")
