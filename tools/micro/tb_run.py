"""One temporal-blocking call (2d5pt 16384^2) for ncu: python tools/micro/tb_run.py T"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2502_16851_b200 as P
t = int(sys.argv[1]) if len(sys.argv) > 1 else 6
u = torch.empty((16384, 16384), dtype=torch.float64, device="cuda")
P.stencil_init(u, 1, 1)
v = u.clone()
P.stencil_temporal("2d5pt", u, v, 2 * t, t)
torch.cuda.synchronize()
print("ok", t)
