import os
os.environ.setdefault("RL_DEV_TUNING", "1")  # sweep knobs (rl_tuning_set developer keys)
import os, sys
sys.path.insert(0, ".")
import torch
import paper_2502_16851_b200 as P
u = torch.empty((512, 512, 512), dtype=torch.float64, device="cuda")
P.stencil_init(u, 1, 1)
v = u.clone()
for t in (2, 3, 4):
    for promo in (0, 1, 2, 3):
        P.tuning_set("stencil_tb3_l2promo", promo)
        P.stencil_temporal("3d7pt", u, v, 2 * t, t)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(3):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(); P.stencil_temporal("3d7pt", u, v, 10 * t, t); e.record(); torch.cuda.synchronize()
            best = min(best, s.elapsed_time(e) / (10 * t))
        print(f"t={t} l2promo={promo} {best:.4f} ms/timestep", flush=True)
