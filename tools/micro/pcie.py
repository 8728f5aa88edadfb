"""H2D / D2H / bidirectional pinned-copy bandwidth (torch streams)."""
import time
import torch

n = 32 << 20  # bytes per direction per trial (x/y of the SpMV plan)
for size in (n, 8 * n):
    h_in = torch.empty(size // 8, dtype=torch.float64).pin_memory()
    h_out = torch.empty(size // 8, dtype=torch.float64).pin_memory()
    d_in = torch.empty(size // 8, dtype=torch.float64, device="cuda")
    d_out = torch.empty(size // 8, dtype=torch.float64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for name in ("h2d", "d2h", "both"):
        for rep in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if name in ("h2d", "both"):
                with torch.cuda.stream(s1):
                    d_in.copy_(h_in, non_blocking=True)
            if name in ("d2h", "both"):
                with torch.cuda.stream(s2):
                    h_out.copy_(d_out, non_blocking=True)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
        moved = size * (2 if name == "both" else 1)
        print(f"{size>>20:5d} MiB {name:5s} {dt*1e3:7.3f} ms  {moved/dt/1e9:6.1f} GB/s")
