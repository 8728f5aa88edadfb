"""ms per timestep of 3d7pt temporal blocking at 512^3 for each (t, shape):
python tools/micro/tb3_time.py [t,...] [shape,...]"""
import os
os.environ.setdefault("RL_DEV_TUNING", "1")  # sweep knobs (rl_tuning_set developer keys)
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2502_16851_b200 as P

ts = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,2,3,4").split(",")]
shapes = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "0").split(",")]
u = torch.empty((512, 512, 512), dtype=torch.float64, device="cuda")
P.stencil_init(u, 1, 1)
v = u.clone()
for t in ts:
    for shp in shapes:
        P.tuning_set("stencil_tb3_shape", shp)
        steps = 10 * t
        run = (lambda: P.stencil("3d7pt", u, v, steps)) if t == 1 else (lambda: P.stencil_temporal("3d7pt", u, v, steps, t))
        run()
        best = 1e9
        for _ in range(3):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            s.record()
            run()
            e.record()
            torch.cuda.synchronize()
            best = min(best, s.elapsed_time(e) / steps)
        print(f"t={t} shape={shp} ms/timestep={best:.4f} GB/s-equiv={16 * 510**3 / best / 1e6:.0f}", flush=True)
P.tuning_set("stencil_tb3_shape", 0)
