"""3d27pt TC sustained (bench-style: 5 runs of 50 timesteps, median) for a few
launch shapes, interleaved so the power state is shared."""
import os
os.environ.setdefault("RL_DEV_TUNING", "1")
import statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2502_16851_b200 as P
u = torch.empty((512, 512, 512), dtype=torch.float64, device="cuda")
P.stencil_init(u, 1, 1)
v = u.clone()
B = P.stencil_model("3d27pt").traffic_bytes * 510 ** 3
shapes = {"default": {}, "ctas8": {"stencil_tch_ctas_per_sm": 8}, "ctas12": {"stencil_tch_ctas_per_sm": 12},
          "ctas24": {"stencil_tch_ctas_per_sm": 24}, "stages3": {"stencil_tch_stages": 3},
          "tpw2": {"stencil_tch_tpw": 2, "stencil_tch_ctas_per_sm": 8}, "cc": None}
if len(sys.argv) > 1:  # name=key:val,key:val ...
    shapes = {"default": {}, "cc": None}
    for a in sys.argv[1:]:
        name, _, kv = a.partition("=")
        shapes[name] = {k: int(v) for k, v in (x.split(":") for x in kv.split(","))}
res = {k: [] for k in shapes}
for rnd in range(int(os.environ.get('ROUNDS', '7'))):
    for name, keys in shapes.items():
        prev = {}
        for k, val in (keys or {}).items():
            prev[k] = P.tuning_set(k, val)
        unit = P.CUDA_CORE if keys is None else P.TENSOR_CORE
        P.stencil("3d27pt", u, v, 2, unit=unit)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        P.stencil("3d27pt", u, v, 50, unit=unit)
        e.record()
        torch.cuda.synchronize()
        res[name].append(s.elapsed_time(e) / 50)
        for k, val in prev.items():
            P.tuning_set(k, val)
for name, ms in res.items():
    med = statistics.median(ms)
    print(f"{name}: median {med:.4f} ms/step {B / med / 1e6:.0f} GB/s  runs {[round(m, 4) for m in ms]}", flush=True)
