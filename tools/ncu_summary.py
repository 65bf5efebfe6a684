"""Key metrics + instruction mix of one kernel in an .ncu-rep.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [steps]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
steps = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, v = rows[0], rows[2]
want = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "launch__registers_per_thread",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct"]
for i, n in enumerate(h):
    if n in want:
        print(f"{n:70s} {v[i]}")
st = [(n, float(v[i].replace(",", ""))) for i, n in enumerate(h)
      if n.startswith("smsp__pcsamp_warps_issue_stalled") and not n.endswith("not_issued")]
tot = sum(x for _, x in st) or 1
print("stalls:", ", ".join(f"{n.replace('smsp__pcsamp_warps_issue_stalled_', '')} {x / tot:.0%}"
                           for n, x in sorted(st, key=lambda t: -t[1])[:8]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(src)))
c = {n: i for i, n in enumerate(r[1])}
op = collections.Counter()
for row in r[2:]:
    toks = row[c["Source"]].strip().split()
    if not toks:
        continue
    k = toks[1] if toks[0].startswith("@") else toks[0]
    try:
        op[k.split(".")[0]] += float(row[c["Instructions Executed"]].replace(",", ""))
    except ValueError:
        pass
tot = sum(op.values())
print(f"instructions {tot:.4g}" + (f", {tot / steps:.1f} per step" if steps else ""))
print("  ".join(f"{k} {x / tot:.1%}" + (f"({x / steps:.1f})" if steps else "") for k, x in op.most_common(24)))
