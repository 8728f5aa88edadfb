import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2502_16851_b200 as P
preset, un, t = sys.argv[1], sys.argv[2], int(sys.argv[3])
unit = P.CUDA_CORE if un == "cc" else P.TENSOR_CORE
shape = (16384, 16384) if preset.startswith("2d") else (512, 512, 512)
u = torch.empty(shape, dtype=torch.float64, device="cuda")
P.stencil_init(u, 1, 1)
v = u.clone()
P.stencil_temporal(preset, u, v, 2 * t, t, unit=unit)
torch.cuda.synchronize()
