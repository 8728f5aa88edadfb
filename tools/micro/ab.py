"""Interleaved A/B timing of tuning variants (cancels the drift that
back-to-back sweeps see on this box): for each round, every variant runs one
`steps`-timestep stencil call; medians over rounds.

python tools/micro/ab.py 3d27pt tc "stencil_tc3d_hybrid=1" "stencil_tc3d_hybrid=0" ...
(a variant "cc" runs the CUDA-core unit with default tuning)"""
import os
os.environ.setdefault("RL_DEV_TUNING", "1")  # sweep knobs (rl_tuning_set developer keys)
import math
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2502_16851_b200 as P  # noqa: E402

SHAPES = {"2d5pt": (16384, 16384), "3d7pt": (512, 512, 512), "3d27pt": (512, 512, 512),
          "2d9pt": (16384, 16384), "2d13pt": (16384, 16384), "2d49pt": (16384, 16384)}


def apply(variant):
    old = {}
    for kv in filter(None, variant.split(",")):
        if kv == "cc":
            continue
        k, v = kv.split("=")
        old[k] = P.tuning_set(k, int(v))
    return old


def main(preset, unit, variants, rounds=int(os.environ.get("AB_ROUNDS", "7")),
         steps=int(os.environ.get("AB_STEPS", "20"))):
    shape = SHAPES[preset]
    r = P.stencil_preset(preset)[2]
    u = torch.empty(shape, dtype=torch.float64, device="cuda")
    P.stencil_init(u, r, 1)
    v = u.clone()
    nbytes = steps * 16 * math.prod(s - 2 * r for s in shape)
    res = {vr: [] for vr in variants}
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for rd in range(rounds + 1):
        for vr in variants:
            un = P.CUDA_CORE if (unit == "cc" or "cc" in vr.split(",")) else P.TENSOR_CORE
            old = apply(vr)
            P.stencil(preset, u, v, 2, unit=un)  # warm (tensor maps, attributes)
            s.record()
            P.stencil(preset, u, v, steps, unit=un)
            e.record()
            torch.cuda.synchronize()
            for k, val in old.items():
                P.tuning_set(k, val)
            if rd:
                res[vr].append(nbytes / s.elapsed_time(e) / 1e6)
    for vr in variants:
        g = res[vr]
        print(f"{preset} {unit} {vr or 'default':48s} median {statistics.median(g):7.1f} GB/s  "
              f"min {min(g):7.1f} max {max(g):7.1f}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3:] or [""])
