"""3d27pt tensor-core (x-band hybrid, st3d_tma_tch KIND 1) launch-shape sweep on 512^3."""
import os
os.environ.setdefault("RL_DEV_TUNING", "1")
import itertools, json, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2502_16851_b200 as P
u = torch.empty((512, 512, 512), dtype=torch.float64, device="cuda")
P.stencil_init(u, 1, 1)
v = u.clone()
B = P.stencil_model("3d27pt").traffic_bytes * 510 ** 3
def timeit(fn, reps=10):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps
for tpw, cps, st, k8 in itertools.product((1, 2, 4), (2, 4, 8, 16, 32), (4, 6), (0, 1)):
    if st == 6 and k8: continue
    for k, val in (("stencil_tch_tpw", tpw), ("stencil_tch_ctas_per_sm", cps), ("stencil_tch_stages", st), ("stencil_tch_k8", k8)):
        P.tuning_set(k, val)
    ms = timeit(lambda: P.stencil("3d27pt", u, v, 2, unit=P.TENSOR_CORE)) / 2
    print(json.dumps({"tpw": tpw, "ctas_per_sm": cps, "stages": st, "k8": k8, "ms": round(ms, 4), "gbs": round(B / ms / 1e6, 1)}), flush=True)
