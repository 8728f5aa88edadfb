import sys, os
sys.path.insert(0, "/root/repo")
import torch, paper_2502_16851_b200 as P
P.tuning_set("stencil_tc3d_mode", 6)
u = torch.empty((512, 512, 512), dtype=torch.float64, device="cuda"); P.stencil_init(u, 1, 1); v = u.clone()
P.stencil("3d27pt", u, v, 2, unit=1); torch.cuda.synchronize(); print("ok")
