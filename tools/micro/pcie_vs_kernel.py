"""Does PCIe traffic (32 MiB H2D + 32 MiB D2H on the copy engines) slow the
K17 SpMV kernel running beside it?  Device-resident plan.execute timed alone
and under continuous bidirectional copies (CUDA events on the compute stream)."""
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
plan = P.SpmvPlan(rp.cpu(), col.cpu(), val.cpu(), n)
hx = torch.empty(4 * n, dtype=torch.float64).pin_memory(); hy = torch.empty(4 * n, dtype=torch.float64).pin_memory()
dx = torch.empty(4 * n, dtype=torch.float64, device="cuda"); dy2 = torch.empty(4 * n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(reps=40):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        plan.execute(x, y)
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


for _ in range(3):
    plan.execute(x, y)
torch.cuda.synchronize()
print(f"alone: {timed():.4f} ms per call", flush=True)
with torch.cuda.stream(s1):
    for _ in range(6):
        dx.copy_(hx, non_blocking=True)
with torch.cuda.stream(s2):
    for _ in range(6):
        hy.copy_(dy2, non_blocking=True)
print(f"beside H2D + D2H copies: {timed():.4f} ms per call", flush=True)
torch.cuda.synchronize()
with torch.cuda.stream(s1):
    for _ in range(6):
        dx.copy_(hx, non_blocking=True)
print(f"beside H2D copies: {timed():.4f} ms per call", flush=True)
torch.cuda.synchronize()
with torch.cuda.stream(s2):
    for _ in range(6):
        hy.copy_(dy2, non_blocking=True)
print(f"beside D2H copies: {timed():.4f} ms per call", flush=True)
torch.cuda.synchronize()
