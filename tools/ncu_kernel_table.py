"""Markdown table of the key ncu metrics of every kernel in one or more
.ncu-rep files (--set full captures), against the measured HBM peak.

    python tools/ncu_kernel_table.py <rep>... > profiles/<tag>_kernels.md
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
try:
    PEAK = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
except Exception:  # noqa: BLE001
    PEAK = 6650.0


def rows_of(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return [dict(zip(r[0], row)) for row in r[2:]]


def f(row, k):
    try:
        return float(row.get(k, "nan").replace(",", ""))
    except ValueError:
        return float("nan")


print("| kernel | ms | DRAM GB/s | % HBM peak | L2 hit % | L1 hit % | issue % | warps % | FP64 pipe % | regs | top stalls |")
print("|---|---:|---:|---:|---:|---:|---:|---:|---:|---:|---|")
for rep in sys.argv[1:]:
    for row in rows_of(rep):
        name = row.get("Kernel Name", "?").split("(")[0].replace("void ", "")
        if "cub::" in name:
            name = "cub::" + name.split("cub::")[1].split("<")[0]
        ms = f(row, "gpu__time_duration.sum")
        dram = (f(row, "dram__bytes_read.sum") + f(row, "dram__bytes_write.sum"))   # Gbyte (ncu units)
        gbs = dram / (ms * 1e-3) if ms > 0 else float("nan")
        st = [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), f(row, k)) for k in row
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")]
        tot = sum(v for _, v in st if v == v) or 1
        top = ", ".join(f"{k} {v / tot:.0%}" for k, v in sorted(st, key=lambda t: -t[1])[:3])
        print(f"| {name} | {ms:.3f} | {gbs:.0f} | {100 * gbs / PEAK:.1f} | "
              f"{f(row, 'lts__t_sector_hit_rate.pct'):.1f} | {f(row, 'l1tex__t_sector_hit_rate.pct'):.1f} | "
              f"{f(row, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f} | "
              f"{f(row, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} | "
              f"{f(row, 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active'):.1f} | "
              f"{row.get('launch__registers_per_thread', '?').split()[0]} | {top} |")
print(f"\nHBM peak = {PEAK} GB/s (MEASURED_PEAKS.json). DRAM GB/s = (dram__bytes_read + dram__bytes_write) / duration "
      "(ncu-serialised, cold-cache launches: shares and ratios, not absolute throughput).")
