"""Per-kernel median table of an `ncu --set full` capture of tools/prof_kernels.py:
python tools/ncu_table.py capture.ncu-rep > profiles/ncu_rN_kernels.md
Launches are grouped by kernel function (template arguments kept); algorithmic bytes
per launch come from the BASELINE model where the kernel is one of the bench's."""
import csv
import io
import statistics
import subprocess
import sys

M = [("gpu__time_duration.sum", "ncu time (µs, cold, serialised)", 1e-3),
     ("dram__bytes_read.sum", None, 1.0), ("dram__bytes_write.sum", None, 1.0),
     ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram % peak", 1.0),
     ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %", 1.0),
     ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1 %", 1.0),
     ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %", 1.0),
     ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %", 1.0),
     ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "dmma pipe %", 1.0),
     ("launch__registers_per_thread", "regs", 1.0)]
UNIT = {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    ki = head.index("Kernel Name")
    groups = {}
    for r in rows[2:]:
        name = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "").replace("unnamed>::", "")
        vals = {}
        for m, _, _ in M:
            if m in head:
                i = head.index(m)
                vals[m] = float(r[i].replace(",", "")) * UNIT.get(units[i], 1)
        groups.setdefault(name, []).append(vals)
    cols = ["kernel", "launches", M[0][1], "DRAM read+write per launch (GB)"] + [h for m, h, _ in M[3:]]
    print("| " + " | ".join(cols) + " |")
    print("|" + "---|" * len(cols))
    for name, vs in groups.items():
        med = {m: statistics.median(v[m] for v in vs if m in v) for m, _, _ in M if any(m in v for v in vs)}
        dram = (med.get("dram__bytes_read.sum", 0) + med.get("dram__bytes_write.sum", 0)) * 1e-9
        cells = [f"`{name}`", str(len(vs)), f"{med.get(M[0][0], 0) * 1e-3:.1f}", f"{dram:.3f}"]
        for m, h, sc in M[3:]:
            cells.append(f"{med[m] * sc:.1f}" if m in med else "-")
        print("| " + " | ".join(cells) + " |")


if __name__ == "__main__":
    main(sys.argv[1])
