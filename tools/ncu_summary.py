"""Summarise an ncu --set full report (.ncu-rep) as a markdown table: duration, DRAM bytes and
throughput, L1/TEX throughput, occupancy, registers and the top warp-stall reasons per kernel.

    python tools/ncu_summary.py gpurun_out/prof_cg_r01g.ncu-rep > profiles/r01g_ncu_summary.md
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]


def col(r, name):
    try:
        return r[h.index(name)]
    except ValueError:
        return ""


def num(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return float("nan")


print(f"# ncu --set full summary of `{rep.split('/')[-1]}`\n")
print("| kernel | us | DRAM MB (r+w) | dram % | l1tex % | issue busy % | warps active % | regs | top stalls (cycles per issue) |")
print("|---|---|---|---|---|---|---|---|---|")
for r in rows[2:]:
    name = col(r, "Kernel Name").split("(")[0].replace("void ", "").split("::")[-1]
    stalls = []
    for n, x in zip(h, r):
        if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio"):
            k = n[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]
            if k not in ("selected",):
                stalls.append((num(x), k))
    stalls.sort(reverse=True)
    us = num(col(r, "gpu__time_duration.sum")) / 1e3 if num(col(r, "gpu__time_duration.sum")) > 1e3 else num(col(r, "gpu__time_duration.sum"))
    unit = {"Gbyte": 1e3, "Mbyte": 1.0, "Kbyte": 1e-3, "byte": 1e-6}
    dram = sum(num(col(r, m)) * unit.get(rows[1][h.index(m)], float("nan"))
               for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    print(f"| {name} | {us:.2f} | {dram:.1f} | {num(col(r, 'dram__bytes_read.sum.pct_of_peak_sustained_elapsed')) + num(col(r, 'dram__bytes_write.sum.pct_of_peak_sustained_elapsed')):.1f} | "
          f"{num(col(r, 'l1tex__throughput.avg.pct_of_peak_sustained_active')):.1f} | "
          f"{num(col(r, 'sm__inst_issued.avg.pct_of_peak_sustained_active')):.1f} | "
          f"{num(col(r, 'sm__warps_active.avg.pct_of_peak_sustained_active')):.1f} | "
          f"{col(r, 'launch__registers_per_thread')} | "
          + ", ".join(f"{k} {v:.1f}" for v, k in stalls[:3]) + " |")
