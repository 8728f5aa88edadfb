"""Run each hot kernel a few times at its BASELINE config (for ncu captures).

  python tools/prof_kernels.py [names...]   names: stream_cc stream_tc spmv_cc spmv_tc (the
        plan: K17 column-sorted blocks) spmvcsr_cc spmvcsr_tc (raw CSR kernels) 2d5pt_cc 2d5pt_tc
        3d7pt_cc 3d7pt_tc 3d27pt_cc 3d27pt_tc (default: all of these);
        also 2d9pt_* 2d13pt_* 2d49pt_* gemv_*, temporal tb<preset>t<depth>_<unit>
        (e.g. tb2d5ptt4_cc, tb2d5ptt4_tc, tb3d7ptt2_cc, tb3d27ptt2_cc)
"""
import os
os.environ.setdefault("RL_DEV_TUNING", "1")  # sweep knobs (rl_tuning_set developer keys)
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2502_16851_b200 as P  # noqa: E402

REPS = int(os.environ.get("PROF_REPS", "3"))


def run(name):
    kern, unit = name.rsplit("_", 1)
    unit = P.CUDA_CORE if unit == "cc" else P.TENSOR_CORE
    if kern == "stream":
        n = 1 << 27
        b = torch.empty(n, dtype=torch.float64, device="cuda")
        P.fill_uniform(b, 1, 1, 0, 1)
        a = torch.empty_like(b)
        for _ in range(REPS):
            P.scale(a, b, 3.0, unit=unit)
    elif kern == "spmvcsr":
        n, k, hb = 1 << 22, 16, 65536
        rp = torch.empty(n + 1, dtype=torch.int32, device="cuda")
        col = torch.empty(n * k, dtype=torch.int32, device="cuda")
        val = torch.empty(n * k, dtype=torch.float64, device="cuda")
        x = torch.empty(n, dtype=torch.float64, device="cuda")
        y = torch.empty(n, dtype=torch.float64, device="cuda")
        P.gen_band_csr(n, 0, n, k, hb, 1, rp, col, val)
        P.fill_uniform(x, 1, 4, 0, 1)
        for _ in range(REPS):
            P.spmv_csr(rp, col, val, x, y, unit=unit)
    elif kern == "gemv":
        m, n = 16384, 65536
        A = torch.empty((m, n), dtype=torch.float64, device="cuda")
        P.fill_uniform(A.view(-1), 1, 6, 0, 1)
        x = torch.empty(n, dtype=torch.float64, device="cuda")
        P.fill_uniform(x, 1, 4, 0, 1)
        y = torch.empty(m, dtype=torch.float64, device="cuda")
        for _ in range(REPS):
            P.gemv(A, x, y, unit=unit)
    elif kern == "spmv":
        n, k, hb = 1 << 22, 16, 65536
        rp = torch.empty(n + 1, dtype=torch.int32, device="cuda")
        col = torch.empty(n * k, dtype=torch.int32, device="cuda")
        val = torch.empty(n * k, dtype=torch.float64, device="cuda")
        x = torch.empty(n, dtype=torch.float64, device="cuda")
        y = torch.empty(n, dtype=torch.float64, device="cuda")
        P.gen_band_csr(n, 0, n, k, hb, 1, rp, col, val)
        P.fill_uniform(x, 1, 4, 0, 1)
        plan = P.SpmvPlan(rp.cpu(), col.cpu(), val.cpu(), n, unit=unit)
        for _ in range(REPS):
            plan.execute(x, y)
        plan.close()
    elif kern.startswith("tb"):
        preset, t = kern[2:].rsplit("t", 1)
        shape = (16384, 16384) if preset.startswith("2d") else (512, 512, 512)
        u = torch.empty(shape, dtype=torch.float64, device="cuda")
        P.stencil_init(u, 1, 1)
        v = u.clone()
        P.stencil_temporal(preset, u, v, REPS * int(t), int(t), unit=unit)
    else:
        shape = (16384, 16384) if kern.startswith("2d") else (512, 512, 512)
        u = torch.empty(shape, dtype=torch.float64, device="cuda")
        P.stencil_init(u, P.stencil_preset(kern)[2], 1)
        v = u.clone()
        P.stencil(kern, u, v, REPS, unit=unit)
    torch.cuda.synchronize()


if __name__ == "__main__":
    names = sys.argv[1:] or ["stream_cc", "stream_tc", "spmv_cc", "spmv_tc", "spmvcsr_cc", "spmvcsr_tc",
                             "2d5pt_cc", "2d5pt_tc", "3d7pt_cc", "3d7pt_tc", "3d27pt_cc", "3d27pt_tc"]
    # PROF_TUNE="key=val,key=val": rl_tuning_set before the runs
    for kv in filter(None, os.environ.get("PROF_TUNE", "").split(",")):
        k, v = kv.split("=")
        P.tuning_set(k, int(v))
    for nm in names:
        run(nm)
        torch.cuda.empty_cache()
    print("ok", names)
