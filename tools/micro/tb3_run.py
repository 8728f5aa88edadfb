"""One 3d7pt temporal-blocking call (512^3) for ncu: python tools/micro/tb3_run.py T"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2502_16851_b200 as P
t = int(sys.argv[1]) if len(sys.argv) > 1 else 2
u = torch.empty((512, 512, 512), dtype=torch.float64, device="cuda")
P.stencil_init(u, 1, 1)
v = u.clone()
P.stencil_temporal("3d7pt", u, v, t, t)
torch.cuda.synchronize()
print("ok", t)
