"""Tuning sweeps over the rl_tuning_set knobs (CUDA-event timing, GB/s of
algorithmic bytes).  python tools/sweep.py stream|spmv|... > out.jsonl"""
import os
os.environ.setdefault("RL_DEV_TUNING", "1")  # sweep knobs (rl_tuning_set developer keys)
import itertools
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2502_16851_b200 as P  # noqa: E402

P.library_path = os.environ.get("RL_LIB", P.library_path)


def timeit(fn, reps=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def sweep(name, fn, nbytes, grid):
    keys = list(grid)
    for vals in itertools.product(*[grid[k] for k in keys]) if keys else [()]:
        for k, v in zip(keys, vals):
            P.tuning_set(k, v)
        ms = timeit(fn)
        print(json.dumps({"kernel": name, **dict(zip(keys, vals)), "ms": round(ms, 5),
                          "gbs": round(nbytes / ms / 1e6, 1)}), flush=True)


def main(which):
    if which == "stream":
        n = 1 << 27
        b = torch.empty(n, dtype=torch.float64, device="cuda")
        P.fill_uniform(b, 1, 1, 0, 1)
        a = torch.empty_like(b)
        for unit in (0, 1):
            sweep(f"stream_{'cc' if unit == 0 else 'tc'}", lambda: P.scale(a, b, 3.0, unit=unit), 16 * n,
                  {"scale_unroll": [1, 2, 4, 8] if unit == 0 else [4],
                   "scale_blocks_per_sm": [1, 2, 4, 8, 16, 32]})
    elif which == "spmv":
        n, k, hb = 1 << 22, 16, 65536
        rp = torch.empty(n + 1, dtype=torch.int32, device="cuda")
        col = torch.empty(n * k, dtype=torch.int32, device="cuda")
        val = torch.empty(n * k, dtype=torch.float64, device="cuda")
        x = torch.empty(n, dtype=torch.float64, device="cuda")
        y = torch.empty(n, dtype=torch.float64, device="cuda")
        P.gen_band_csr(n, 0, n, k, hb, 1, rp, col, val)
        P.fill_uniform(x, 1, 4, 0, 1)
        nbytes = P.spmv_csr_model(n, n, n * k).traffic_bytes
        sweep("spmv_cc", lambda: P.spmv_csr(rp, col, val, x, y, unit=0), nbytes,
              {"spmv_l1_carveout": [-1, 0, 25, 50], "spmv_xhint": [0, 1], "spmv_threads": [512, 1024],
               "spmv_blocks_per_sm": [1, 2]})
        sweep("spmv_tc", lambda: P.spmv_csr(rp, col, val, x, y, unit=1), nbytes,
              {"spmv_tc_rows": [1, 2], "spmv_tc_threads": [256, 1024], "spmv_tc_blocks_per_sm": [1, 2, 4, 8],
               "spmv_sched": [0, 1]})


def gemv():
    m, n = 16384, 65536
    A = torch.empty((m, n), dtype=torch.float64, device="cuda")
    P.fill_uniform(A.view(-1), 1, 6, 0, 1)
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    P.fill_uniform(x, 1, 4, 0, 1)
    y = torch.empty(m, dtype=torch.float64, device="cuda")
    nbytes = P.gemv_model(m, n).traffic_bytes
    for unit in (0, 1):
        sweep(f"gemv_{'cc' if unit == 0 else 'tc'}", lambda: P.gemv(A, x, y, unit=unit), nbytes, {})


def temporal_t():
    """2d5pt at 16384^2: ms per timestep for temporal depth 1..8 (register
    kernel)."""
    u = torch.empty((16384, 16384), dtype=torch.float64, device="cuda")
    P.stencil_init(u, 1, 1)
    v = u.clone()
    waves_list = [int(x) for x in os.environ.get("TB_WAVES", "1").split(",")]
    cases = [(1, 1, 1)] + [(t, 1, w) for t in range(2, 9) for w in waves_list]
    for t, tb, waves in cases:
        P.tuning_set("stencil_tb_waves", waves)
        steps = 8 * t
        fn = (lambda: P.stencil("2d5pt", u, v, steps)) if t == 1 else \
            (lambda: P.stencil_temporal("2d5pt", u, v, steps, t))
        ms = timeit(fn, reps=5, warm=2) / steps
        print(json.dumps({"kernel": "2d5pt_temporal", "t": t, "register_kernel": tb, "waves": waves,
                          "ms_per_timestep": round(ms, 4),
                          "timestep_gbs_equiv": round(16 * 16382 ** 2 / ms / 1e6, 1)}), flush=True)


def temporal_3d():
    """3d7pt at 512^3: ms per timestep for temporal depth 1..4 (register-blocked
    kernel), z-chunk counts from TB3_CHUNKS (0 = auto)."""
    u = torch.empty((512, 512, 512), dtype=torch.float64, device="cuda")
    P.stencil_init(u, 1, 1)
    v = u.clone()
    modes = [1]
    chunks = [int(x) for x in os.environ.get("TB3_CHUNKS", "0").split(",")]
    shapes = [int(x) for x in os.environ.get("TB3_SHAPES", "0").split(",")]
    for t in (1, 2, 3, 4):
        for mode in (modes if t > 1 else [1]):
          for shp in (shapes if t > 1 and mode == 1 else [0]):
            for ch in (chunks if t > 1 and mode == 1 else [0]):
                P.tuning_set("stencil_tb3_shape", shp)
                P.tuning_set("stencil_tb3_chunks", ch)
                steps = 4 * t
                fn = (lambda: P.stencil("3d7pt", u, v, steps)) if t == 1 else \
                    (lambda: P.stencil_temporal("3d7pt", u, v, steps, t))
                ms = timeit(fn, reps=5, warm=2) / steps
                print(json.dumps({"kernel": "3d7pt_temporal", "t": t, "mode": mode, "shape": shp, "chunks": ch,
                                  "ms_per_timestep": round(ms, 4),
                                  "timestep_gbs_equiv": round(16 * 510 ** 3 / ms / 1e6, 1)}), flush=True)
    P.tuning_set("stencil_tb3_chunks", 0)
    P.tuning_set("stencil_tb3_shape", 0)


def stencils():
    import math
    for preset, shape in (("2d5pt", (16384, 16384)), ("3d7pt", (512, 512, 512)), ("3d27pt", (512, 512, 512))):
        u = torch.empty(shape, dtype=torch.float64, device="cuda")
        P.stencil_init(u, 1, 1)
        v = u.clone()
        nbytes = 2 * 16 * math.prod(s - 2 for s in shape)
        for unit in (0, 1):
            if preset == "2d5pt" or unit == 0:
                continue
            grid = {"stencil_tc3d_mode": [0, 1], "stencil_tc1_ctas_per_sm": [1, 2, 4, 8, 16]}
            sweep(f"{preset}_{'cc' if unit == 0 else 'tc'}", lambda: P.stencil(preset, u, v, 2, unit=unit),
                  nbytes, grid)
        del u, v
        torch.cuda.empty_cache()


def stencil2d():
    import math
    u = torch.empty((16384, 16384), dtype=torch.float64, device="cuda")
    P.stencil_init(u, 1, 1)
    v = u.clone()
    nbytes = 4 * 16 * math.prod(s - 2 for s in u.shape)
    sweep("2d5pt_tc", lambda: P.stencil("2d5pt", u, v, 4, unit=1), nbytes,
          {"stencil_tc_ctas_per_sm": [1, 2, 3, 4, 6, 8]})
    sweep("2d5pt_cc", lambda: P.stencil("2d5pt", u, v, 4, unit=0), nbytes,
          {"stencil_ctas_per_sm": [1, 2, 4], "stencil2d_rows_per_thread": [2, 4, 8]})


def stencil3d_cc():
    import math
    for preset in ("3d7pt", "3d27pt"):
        u = torch.empty((512, 512, 512), dtype=torch.float64, device="cuda")
        P.stencil_init(u, 1, 1)
        v = u.clone()
        nbytes = 4 * 16 * math.prod(s - 2 for s in u.shape)
        sweep(f"{preset}_cc", lambda: P.stencil(preset, u, v, 4, unit=0), nbytes,
              {"stencil3d_cc_stages": [4, 6, 8, 4], "stencil_rows_per_thread": [4, 2, 0]})
        sweep(f"{preset}_cc", lambda: P.stencil(preset, u, v, 4, unit=0), nbytes,
              {"stencil_ctas_per_sm": [1, 2, 3, 4, 6, 8, 1]})
        del u, v
        torch.cuda.empty_cache()


def stencil3d_tc():
    import math
    u = torch.empty((512, 512, 512), dtype=torch.float64, device="cuda")
    P.stencil_init(u, 1, 1)
    v = u.clone()
    nbytes = 4 * 16 * math.prod(s - 2 for s in u.shape)
    sweep("3d27pt_tc", lambda: P.stencil("3d27pt", u, v, 4, unit=1), nbytes,
          {"stencil_tc_concat": [0, 1, 0, 1], "stencil_tc1_ctas_per_sm": [4, 8]})
    sweep("3d7pt_tc", lambda: P.stencil("3d7pt", u, v, 4, unit=1), nbytes,
          {"stencil_tc3d_mode": [2], "stencil_tc3d_ctas_per_sm": [6, 8, 12, 16, 24, 8]})
    sweep("3d27pt_cc", lambda: P.stencil("3d27pt", u, v, 4, unit=0), nbytes,
          {"stencil_cc27x2": [0, 1, 0, 1], "stencil_rows_per_thread": [2, 4]})


def stencil3d_tch():
    """3D tensor core: x-band hybrid (st3d_tma_tch) vs the full banded kernels, 50 timesteps."""
    import math
    for preset in ("3d7pt", "3d27pt"):
        u = torch.empty((512, 512, 512), dtype=torch.float64, device="cuda")
        P.stencil_init(u, 1, 1)
        v = u.clone()
        nbytes = 50 * 16 * math.prod(s - 2 for s in u.shape)
        for hy in (1, 0):
            P.tuning_set("stencil_tc3d_hybrid", hy)
            grid = {"stencil_tch_ctas_per_sm": [2, 3, 4, 8]} if hy else {}
            sweep(f"{preset}_tc_hybrid{hy}", lambda: P.stencil(preset, u, v, 50, unit=1), nbytes, grid)
        P.tuning_set("stencil_tc3d_hybrid", 1)
        sweep(f"{preset}_cc", lambda: P.stencil(preset, u, v, 50, unit=0), nbytes, {})
        del u, v
        torch.cuda.empty_cache()


def stencil_r():
    """2d9pt / 2d13pt / 2d49pt at 16384^2; GB/s of algorithmic bytes and the
    FP64 rate (W = 2 |S| per point)."""
    import math
    u = torch.empty((16384, 16384), dtype=torch.float64, device="cuda")
    v = torch.empty_like(u)
    for preset in ("2d9pt", "2d13pt", "2d49pt"):
        npts, r = P.stencil_preset(preset)[1], P.stencil_preset(preset)[2]
        P.stencil_init(u, r, 1)
        v.copy_(u)
        pts = math.prod(s - 2 * r for s in u.shape)
        for unit, st, cps, sym in ((0, 0, 32, 0), (0, 0, 32, 1), (0, 3, 32, 1), (0, 2, 32, 1), (1, 0, 32, 1)):
            P.tuning_set("stencil_r_cc_stages", st)
            P.tuning_set("stencil_r_sym", sym)
            promo = 1
            P.tuning_set("stencil_r_sym", sym)
            P.tuning_set("stencil_r_ctas_per_sm", cps)
            ms = timeit(lambda: P.stencil(preset, u, v, 2, unit=unit), reps=5) / 2
            print(json.dumps({"kernel": f"{preset}_{'cc' if unit == 0 else 'tc'}", "stages": st, "ctas_per_sm": cps, "sym": sym,
                              "ms_per_step": round(ms, 4),
                              "gbs": round(16 * pts / ms / 1e6, 1),
                              "tflops": round(2 * npts * pts / ms / 1e9, 2)}), flush=True)


if __name__ == "__main__":
    for w in sys.argv[1:]:
        if w == "stencil_r":
            stencil_r()
        elif w == "stencil2d":
            stencil2d()
        elif w == "stencil3d_cc":
            stencil3d_cc()
        elif w == "stencil3d_tch":
            stencil3d_tch()
        elif w == "stencil3d_tc":
            stencil3d_tc()
        elif w == "stencil":
            stencils()
        elif w == "temporal_t":
            temporal_t()
        elif w == "temporal_3d":
            temporal_3d()
        elif w == "gemv":
            gemv()
        else:
            main(w)
