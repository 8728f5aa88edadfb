"""3d27pt t = 2: register-blocked kernel shapes vs the z-column kernel vs one sweep (512^3, 50 steps)."""
import os
os.environ.setdefault("RL_DEV_TUNING", "1")
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2502_16851_b200 as P
u = torch.empty((512, 512, 512), dtype=torch.float64, device="cuda")
P.stencil_init(u, 1, 1)
v = u.clone()
def t50(fn):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); fn(); e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / 50
print(f"single sweep: {t50(lambda: P.stencil('3d27pt', u, v, 50)):.4f} ms/timestep", flush=True)
P.tuning_set("stencil_tb27r", 0)
print(f"z-column t=2: {t50(lambda: P.stencil_temporal('3d27pt', u, v, 50, 2)):.4f} ms/timestep", flush=True)
P.tuning_set("stencil_tb27r", 1)
for shape in (0, 3):
    P.tuning_set("stencil_tb3_shape", shape)
    print(f"register t=2 shape {shape}: {t50(lambda: P.stencil_temporal('3d27pt', u, v, 50, 2)):.4f} ms/timestep", flush=True)
