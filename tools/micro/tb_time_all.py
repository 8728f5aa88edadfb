"""Temporal-blocking timings on the BASELINE grids: per-timestep ms for each
(preset, unit, t) the library implements, beside the single-step kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch

import paper_2502_16851_b200 as P

which = sys.argv[1:] or ["2d5pt:tc", "3d27pt:cc"]
for spec in which:
    preset, un = spec.split(":")
    unit = P.CUDA_CORE if un == "cc" else P.TENSOR_CORE
    shape = (16384, 16384) if preset.startswith("2d") else (512, 512, 512)
    steps = 100 if preset.startswith("2d") else 50
    u = torch.empty(shape, dtype=torch.float64, device="cuda")
    P.stencil_init(u, 1, 1)
    v = u.clone()
    for t in (1, 2, 3, 4):
        fn = (lambda: P.stencil(preset, u, v, steps, unit=unit)) if t == 1 else \
             (lambda: P.stencil_temporal(preset, u, v, steps, t, unit=unit))
        fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        print(f"{preset} {un} t={t}: {s.elapsed_time(e) / steps:.4f} ms/timestep", flush=True)
    del u, v
    torch.cuda.empty_cache()
