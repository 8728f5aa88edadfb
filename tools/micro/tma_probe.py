"""Run one stencil variant in isolation (fresh process per call)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import oracle as O, paper_2502_16851_b200 as P
preset, unit, shape = sys.argv[1], int(sys.argv[2]), tuple(int(s) for s in sys.argv[3].split("x"))
u0 = O.stencil_init(shape, 1, 7)
u = torch.from_numpy(u0.copy()).cuda(); v = torch.from_numpy(u0.copy()).cuda()
try:
    P.stencil(preset, u, v, 1, unit=unit)
    torch.cuda.synchronize()
    print(preset, unit, shape, "relerr", O.rel_err(v.cpu().numpy(), O.stencil(preset, u0, 1)))
except Exception as e:
    print(preset, unit, shape, "FAIL", str(e).splitlines()[0])
