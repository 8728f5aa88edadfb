"""Markdown table of the key metrics of ncu --set full captures:
python tools/ncu_summary.py "label::path.ncu-rep[#kernel regex][@algorithmic GB per launch]" ..."""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "time µs", 1e-3, "{:.1f}"),
    ("dram__bytes_read.sum", "DRAM read GB", 1e-9, "{:.3f}"),
    ("dram__bytes_write.sum", "DRAM write GB", 1e-9, "{:.3f}"),
    ("dram__cycles_active.avg.pct_of_peak_sustained_elapsed", "DRAM active %", 1, "{:.1f}"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %", 1, "{:.1f}"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1 %", 1, "{:.1f}"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %", 1, "{:.1f}"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %", 1, "{:.1f}"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %", 1, "{:.1f}"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "dmma pipe %", 1, "{:.1f}"),
    ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", "stall mio", 1, "{:.2f}"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long sb", 1, "{:.2f}"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall math", 1, "{:.2f}"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall barrier", 1, "{:.2f}"),
    ("launch__registers_per_thread", "regs", 1, "{:.0f}"),
]
UNITS = {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
         "%": 1, "register/thread": 1, "": 1}


def read(path):
    import re
    path, _, pat = path.partition("#")  # "file.ncu-rep#kernel-name regex": first matching launch
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    ki = head.index("Kernel Name")
    vals = next(r for r in rows[2:] if not pat or re.search(pat, r[ki]))
    res = {"kernel": vals[head.index("Kernel Name")]}
    for m, *_ in METRICS:
        if m in head:
            i = head.index(m)
            scale = UNITS.get(units[i], 1)
            if units[i] in ("us", "usecond", "ms"):
                scale = UNITS[units[i]]  # to ns
            res[m] = float(vals[i].replace(",", "")) * scale
    return res


def main(args):
    cols = ["launch"] + [h for _, h, _, _ in METRICS] + ["DRAM / algorithmic"]
    print("| " + " | ".join(cols) + " |")
    print("|" + "---|" * len(cols))
    for a in args:
        label, rest = a.split("::", 1)
        path, alg = (rest.split("@") + [None])[:2]
        r = read(path)
        cells = [f"{label} (`{r['kernel'].split('(')[0].replace('void ', '')}`)"]
        for m, _, scale, fmt in METRICS:
            cells.append(fmt.format(r[m] * scale) if m in r else "-")
        dram = (r.get("dram__bytes_read.sum", 0) + r.get("dram__bytes_write.sum", 0)) * 1e-9
        cells.append(f"{dram / float(alg):.3f}" if alg else "-")
        print("| " + " | ".join(cells) + " |")


if __name__ == "__main__":
    main(sys.argv[1:])
