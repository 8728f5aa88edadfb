"""Does a concurrent SpMV (L2-gather heavy) slow the PCIe copy engines?"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2502_16851_b200 as P
n, k, hb = 1 << 22, 16, 65536
rp = torch.empty(n + 1, dtype=torch.int32, device="cuda"); col = torch.empty(n * k, dtype=torch.int32, device="cuda")
val = torch.empty(n * k, dtype=torch.float64, device="cuda"); x = torch.empty(n, dtype=torch.float64, device="cuda")
y = torch.empty(n, dtype=torch.float64, device="cuda")
P.gen_band_csr(n, 0, n, k, hb, 1, rp, col, val); P.fill_uniform(x, 1, 4, 0, 1)
hx = torch.empty(n, dtype=torch.float64).pin_memory(); hy = torch.empty(n, dtype=torch.float64).pin_memory()
dx = torch.empty(n, dtype=torch.float64, device="cuda"); dy = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
def run(copy_h2d, copy_d2h, spmv_calls, ctas=None):
    torch.cuda.synchronize()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record(s1)
    s2.wait_event(e0); s3.wait_event(e0)
    if copy_h2d:
        with torch.cuda.stream(s1): dx.copy_(hx, non_blocking=True)
    e1.record(s1)
    if copy_d2h:
        with torch.cuda.stream(s3): hy.copy_(dy, non_blocking=True)
    e3 = torch.cuda.Event(enable_timing=True); e3.record(s3)
    with torch.cuda.stream(s2):
        for _ in range(spmv_calls): P.spmv_csr(rp, col, val, x, y, stream=s2)
    e2.record(s2)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), e0.elapsed_time(e3), e0.elapsed_time(e2)
for _ in range(2): run(True, True, 3)
print("h2d alone ms %.3f" % min(run(True, False, 0)[0] for _ in range(5)))
print("d2h alone ms %.3f" % min(run(False, True, 0)[1] for _ in range(5)))
print("both, no spmv: h2d %.3f d2h %.3f" % min(run(True, True, 0)[:2] for _ in range(5)))
for calls in (1, 2, 4):
    r = min(run(True, False, calls) for _ in range(5))
    print(f"h2d with {calls} spmv: h2d {r[0]:.3f} ms, spmv total {r[2]:.3f} ms")
    r = min(run(True, True, calls) for _ in range(5))
    print(f"both with {calls} spmv: h2d {r[0]:.3f} d2h {r[1]:.3f}, spmv total {r[2]:.3f} ms")
