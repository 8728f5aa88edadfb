"""Summarise an ncu --set full report into profiles/ (markdown + traffic.json).

  python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/ncu_rNN.md [profiles/traffic.json]
"""
import csv
import io
import json
import re
import statistics
import subprocess
import sys

METRICS = {
    "dur_us": "gpu__time_duration.sum",
    "dram_rd": "dram__bytes_read.sum",
    "dram_wr": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1_pct": "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "warps_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "dmma_pipe_pct": "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "dmma_inst": "sm__inst_executed_pipe_tensor_subpipe_dmma.sum",
    "fp64_inst": "sm__inst_executed_pipe_fp64.sum",
}

ALGO = {  # algorithmic bytes per launch (reference models)
    "stream": 2147483648, "spmv": 889192452, "2d5pt": 4293918784, "3d7pt": 2122416000,
    "3d27pt": 2122416000, "2d9pt": 16 * 16382 ** 2, "2d13pt": 16 * 16378 ** 2, "2d49pt": 16 * 16378 ** 2,
    "gemv": (16384 * 65536 + 16384 + 65536) * 8, "spmvtiled": 889192452,
}


def workload(name):
    m = re.search(r"st2dr_tma_(cc|tc)<(?:\(\w+\))?(\d+), *(?:\(\w+\))?(\w+)", name)
    if m:
        r, box = int(m.group(2)), m.group(3) in ("true", "1")
        return {(1, True): "2d9pt", (3, False): "2d13pt", (3, True): "2d49pt"}[(r, box)] + "_" + m.group(1)
    if "gemv_cc" in name: return "gemv_cc"
    if "gemv_tc" in name: return "gemv_tc"
    if "spmv_tiled" in name: return "spmvtiled_cc"
    if "scale_cc" in name: return "stream_cc"
    if "scale_tc" in name: return "stream_tc"
    if "spmv_cc" in name: return "spmv_cc"
    if "spmv_tc" in name: return "spmv_tc"
    if "st2d_tma_cc" in name or "st2d5_cc" in name: return "2d5pt_cc"
    if "st2d_tma_tc" in name or "st2d5_tc" in name: return "2d5pt_tc"
    m = re.search(r"st3d_tma_(cc|tc1|tc)<(\d)", name)
    if m:
        u, k = m.group(1), int(m.group(2))
        if u == "cc": return {0: "3d7pt_cc", 1: "3d27pt_cc", 2: "3d27pt_cc"}[k]
        return {0: "3d7pt_tc", 1: "3d27pt_tc", 2: "3d27pt_tc"}[k] + ("1" if u == "tc1" else "")
    return None


def main(rep, out_md, out_json=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    per = {}
    for r in rows[2:]:
        w = workload(r[idx["Kernel Name"]])
        if not w:
            continue
        rec = {}
        for k, m in METRICS.items():
            if m in idx:
                try:
                    rec[k] = float(r[idx[m]].replace(",", ""))
                except ValueError:
                    rec[k] = float("nan")
        rec["unit_dram"] = units[idx[METRICS["dram_rd"]]]
        tu = units[idx[METRICS["dur_us"]]]
        rec["dur_us"] *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}.get(tu, 1.0)
        per.setdefault(w, []).append(rec)
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
    lines = ["| kernel | launches | ncu time (µs, cold, serialised) | DRAM read+write per launch (GB) | algorithmic (GB) | traffic / algorithmic | dram % peak | L2 % | L1 % | warps active % | fp64 pipe % | dmma pipe % | regs |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    traffic = {}
    for w in sorted(per):
        recs = per[w]
        med = lambda k: statistics.median(x[k] for x in recs if k in x)
        s = scale.get(recs[0]["unit_dram"], 1.0)
        dram = (med("dram_rd") + med("dram_wr")) * s
        algo = ALGO[w.split("_")[0]]
        w = w.replace("_tc1", "_tc")
        if w.startswith(("2d5pt", "3d")):
            pass  # one launch = one sweep
        traffic[w] = int(dram)
        lines.append(f"| {w} | {len(recs)} | {med('dur_us'):.1f} | {dram/1e9:.3f} | {algo/1e9:.3f} | "
                     f"{dram/algo:.3f} | {med('dram_pct'):.1f} | {med('lts_pct'):.1f} | {med('l1_pct'):.1f} | "
                     f"{med('warps_pct'):.1f} | {med('fp64_pipe_pct'):.1f} | {med('dmma_pipe_pct'):.1f} | "
                     f"{med('regs'):.0f} |")
    with open(out_md, "w") as f:
        f.write(f"# ncu summary of `{rep}`\n\n")
        f.write("`ncu --set full --clock-control none`; medians over the captured launches of "
                "`tools/prof_kernels.py` (BASELINE sizes). Durations under ncu are cold-cache and "
                "serialised: compare shares and bytes, not absolute speed.\n\n")
        f.write("\n".join(lines) + "\n")
    if out_json:
        with open(out_json, "w") as f:
            json.dump(traffic, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(*sys.argv[1:])
