"""Per-timestep times of a sustained 3D stencil run, with the SM clock and
power sampled by NVML, to separate kernel cost from power-cap throttling.

python tools/micro/stencil_sustain.py 3d27pt tc [key=val ...] (steps=200)"""
import os
os.environ.setdefault("RL_DEV_TUNING", "1")  # sweep knobs (rl_tuning_set developer keys)
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2502_16851_b200 as P  # noqa: E402


def main(preset, unit, kv):
    import pynvml

    steps = 200
    for s in kv:
        k, v = s.split("=")
        if k == "steps":
            steps = int(v)
        else:
            P.tuning_set(k, int(v))
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    samples, stop = [], threading.Event()

    def sampler():
        while not stop.is_set():
            samples.append((time.time(), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0))
            time.sleep(0.02)

    u = torch.empty((512, 512, 512), dtype=torch.float64, device="cuda")
    P.stencil_init(u, 1, 1)
    v = u.clone()
    un = P.CUDA_CORE if unit == "cc" else P.TENSOR_CORE
    P.stencil(preset, u, v, 2, unit=un)
    torch.cuda.synchronize()
    time.sleep(1.0)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    th = threading.Thread(target=sampler)
    th.start()
    ev[0].record()
    for i in range(steps):
        P.stencil(preset, u, v, 1, unit=un)
        ev[i + 1].record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(steps)]
    gbs = [16 * 510 ** 3 / t / 1e6 for t in ms]
    q = max(1, steps // 10)
    print(preset, unit, kv)
    for i in range(0, steps, q):
        seg = gbs[i:i + q]
        print(f"  steps {i:4d}-{i + len(seg) - 1:4d}: {sum(seg) / len(seg):7.1f} GB/s")
    if samples:
        sm = sorted(s[1] for s in samples)
        pw = sorted(s[2] for s in samples)
        print(f"  SM clock median {sm[len(sm) // 2]} MHz (min {sm[0]}), power median {pw[len(pw) // 2]:.0f} W "
              f"(max {pw[-1]:.0f}), {len(samples)} samples")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3:])
