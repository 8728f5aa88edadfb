"""One radius-R preset sweep (16384^2) for ncu: python tools/micro/r_run.py PRESET UNIT"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2502_16851_b200 as P
preset = sys.argv[1] if len(sys.argv) > 1 else "2d49pt"
unit = int(sys.argv[2]) if len(sys.argv) > 2 else 1
u = torch.empty((16384, 16384), dtype=torch.float64, device="cuda")
P.stencil_init(u, P.stencil_preset(preset)[2], 1)
v = u.clone()
P.stencil(preset, u, v, 2, unit=unit)
torch.cuda.synchronize()
print("ok", preset, unit)
