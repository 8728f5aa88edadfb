"""Bidirectional pinned copies as the SpMV plan issues them: x in P pieces on
one stream, y out in P pieces on another, D2H piece i released after H2D
piece i+lag (the compute dependency)."""
import time
import torch

n = 32 << 20
h_in = torch.empty(n // 8, dtype=torch.float64).pin_memory()
h_out = torch.empty(n // 8, dtype=torch.float64).pin_memory()
d_in = torch.empty(n // 8, dtype=torch.float64, device="cuda")
d_out = torch.empty(n // 8, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(pieces, lag, both=True):
    m = (n // 8) // pieces
    evs = [torch.cuda.Event() for _ in range(pieces)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(pieces):
        with torch.cuda.stream(s1):
            d_in[i * m:(i + 1) * m].copy_(h_in[i * m:(i + 1) * m], non_blocking=True)
            evs[i].record(s1)
    if both:
        for i in range(pieces):
            with torch.cuda.stream(s2):
                s2.wait_event(evs[min(pieces - 1, i + lag)])
                h_out[i * m:(i + 1) * m].copy_(d_out[i * m:(i + 1) * m], non_blocking=True)
    torch.cuda.synchronize()
    return time.perf_counter() - t0


for pieces in (1, 2, 4, 8, 16, 32):
    for lag in (0, 1):
        best = min(run(pieces, lag) for _ in range(5))
        print(f"pieces {pieces:3d} lag {lag}: {best*1e3:.3f} ms  ({2*n/best/1e9:.1f} GB/s total)", flush=True)
best = min(run(8, 0, both=False) for _ in range(5))
print(f"h2d only, 8 pieces: {best*1e3:.3f} ms ({n/best/1e9:.1f} GB/s)")
