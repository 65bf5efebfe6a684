"""Turn ncu outputs under gpurun_out/ into the committed summaries in profiles/.

    python tools/summarize_profiles.py <launches.csv> <lookup.ncu-rep> <tag>
"""
import collections
import csv
import io
import json
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}.get(r[ui], 1e-9)
        name = r[ki].split("(")[0].replace("void ", "")
        if "cub::" in name:
            name = "cub::" + name.split("cub::")[1].split("<")[0] + " (radix sort)"
        agg[name][0] += 1
        agg[name][1] += v
    return agg


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return [dict(zip(r[0], row)) for row in r[2:]], dict(zip(r[0], r[1]))


def main():
    launches_csv, rep, tag = sys.argv[1], sys.argv[2], sys.argv[3]
    agg = launches(launches_csv)
    tot = sum(v[1] for v in agg.values())
    lines = [f"# {tag}: ncu launch list (bench.py --steps 1 --warmup 1 --no-cpu-baseline, C4, 40M particles)",
             "", "Per-launch device times are ncu-serialised and cold-cache: compare shares, not absolutes.",
             "", "| kernel | launches | total ms | share |", "|---|---:|---:|---:|"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| {k} | {v[0]} | {v[1] * 1e3:.2f} | {100 * v[1] / tot:.1f}% |")
    open(f"profiles/{tag}_launches.md", "w").write("\n".join(lines) + "\n")
    rows, units = raw_metrics(rep)
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "launch__grid_size",
            "launch__block_size", "smsp__inst_executed.sum"]
    row = [r for r in rows if "k_lookup" in r.get("Kernel Name", "")][0]
    summ = {k: row.get(k) + " " + units.get(k, "") for k in keys if k in row}
    st = [(k, float(v)) for k, v in row.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_")
          and not k.endswith("not_issued") and v not in ("", "n/a")]
    tot_s = sum(v for _, v in st) or 1
    summ["stall_share"] = {k[33:]: round(v / tot_s, 3) for k, v in sorted(st, key=lambda x: -x[1])[:6]}
    json.dump(summ, open(f"profiles/{tag}_ncu_lookup.json", "w"), indent=1)
    print("\n".join(lines))
    print(json.dumps(summ, indent=1))


if __name__ == "__main__":
    main()
