"""Regenerate the per-kernel tables of README.md and profiles/README.md from
profiles/bench_r1.json (run after replacing the bench line)."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HBM = 6543.1  # MEASURED_PEAKS.json hbm_gbs


def replace_table(text, header, rows):
    a = text.index(header)
    a = text.index("\n", text.index("\n", a) + 1) + 1  # skip header + separator
    b = text.index("\n\n", a)
    return text[:a] + "\n".join(rows) + text[b:]


def main():
    d = json.load(open(os.path.join(ROOT, "profiles", "bench_r1.json")))
    pk, nr = d["per_kernel"], d["next_rows"]
    names = {"stream": "STREAM Scale 2^27", "spmv": "CSR SpMV 2^22, 16 nnz/row", "2d5pt": "2d5pt 16384², 100 steps",
             "3d7pt": "3d7pt 512³, 50 steps", "3d27pt": "3d27pt 512³, 50 steps"}
    rows = []
    for k, n in names.items():
        cc, tc = pk[k]["cc"]["gbs"], pk[k]["tc"]["gbs"]
        rows.append(f"| {n} | {cc:.0f} | {cc / HBM * 100:.0f} % | {tc:.0f} | {tc / HBM * 100:.0f} % | "
                    f"{tc / cc:.2f} | {pk[k]['bound']:.4f} |")
    nn = {"gemv": ("GEMV 16384×65536", "HBM"), "2d9pt": ("2d9pt 16384²", "HBM"), "2d13pt": ("2d13pt 16384²", "HBM"),
          "2d49pt": ("2d49pt 16384²", "FP64 (I = 6.125 > balance)")}
    rows2 = []
    for k, (n, roof) in nn.items():
        cc, tc = nr[k]["cc"]["gbs"], nr[k]["tc"]["gbs"]
        rows2.append(f"| {n} | {roof} | {cc:.0f} GB/s ({cc / HBM * 100:.0f} %) | {tc:.0f} GB/s ({tc / HBM * 100:.0f} %) | "
                     f"{tc / cc:.2f} | {nr[k]['bound']:.4f} |")
    p = os.path.join(ROOT, "profiles", "README.md")
    s = open(p).read()
    s = replace_table(s, "| kernel (BASELINE config) | CUDA core GB/s |", rows)
    s = replace_table(s, "| kernel | roof | CUDA core | tensor core | TC/CC | bound |", rows2)
    open(p, "w").write(s)
    names2 = {"stream": "STREAM 2^27", "spmv": "CSR SpMV 2^22, 16 nnz/row (headline)", "2d5pt": "2d5pt 16384²",
              "3d7pt": "3d7pt 512³", "3d27pt": "3d27pt 512³"}
    rows3 = []
    for k, n in names2.items():
        cc, tc = pk[k]["cc"]["gbs"], pk[k]["tc"]["gbs"]
        rows3.append(f"| {n} | {cc:.0f} ({cc / HBM * 100:.0f} %) | {tc:.0f} ({tc / HBM * 100:.0f} %) |")
    p = os.path.join(ROOT, "README.md")
    s = open(p).read()
    s = replace_table(s, "| kernel | CC GB/s (% HBM) | TC GB/s (% HBM) |", rows3)
    open(p, "w").write(s)
    print("peaks", d["fp64_peaks_tflops"], "clocks", d["per_kernel_clocks"], "e2e", d["e2e"]["value"],
          "cpu", d["cpu_baseline"]["value"])


if __name__ == "__main__":
    main()
