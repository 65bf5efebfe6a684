"""Copy one final measurement run (tools/gpu_runs/r2_final*.sh, tag T) from
gpurun_out/ into profiles/: bench lines, launch list (csv + markdown), ncu
kernel table, lookup counters; print the numbers the docs quote.

    python tools/finalize_profiles.py <tag>
"""
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
sys.path.insert(0, ROOT)

WORKLOADS = ("c1", "c2", "c3", "c3pin", "c4", "c4pin", "c5", "reference")


def main():
    tag = sys.argv[1]
    out, prof = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
    from summarize_profiles import launches
    agg = launches(os.path.join(out, f"{tag}_launches.csv"))
    tot = sum(v[1] for v in agg.values())
    lines = [f"# Kernel launch list, C4 on the HM core (round 2 final, `{tag}`)", "",
             "`ncu --metrics gpu__time_duration.sum --clock-control none` over "
             "`python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-counters`",
             "(2 batches of 40M particles: 1 inactive + 1 active; serialised, cold-cache per-launch times — "
             "shares, not absolutes).", "", "| kernel | launches | time (ms) | share |", "|---|---:|---:|---:|"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{k}` | {v[0]} | {v[1] * 1e3:.2f} | {100 * v[1] / tot:.1f}% |")
    lines.append(f"| total | {sum(v[0] for v in agg.values())} | {tot * 1e3:.2f} | |")
    with open(os.path.join(prof, f"{tag}_launches.md"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    table = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_kernel_table.py"),
                            os.path.join(out, f"{tag}_kernels.ncu-rep")], capture_output=True, text=True).stdout
    with open(os.path.join(prof, f"{tag}_kernels.md"), "w") as fh:
        fh.write(table)
    for w in WORKLOADS:
        shutil.copy(os.path.join(out, f"{tag}_bench_{w}.json"), prof)
    shutil.copy(os.path.join(out, f"{tag}_launches.csv"), prof)
    shutil.copy(os.path.join(out, "r2_lookup_counters.json"), os.path.join(prof, "r2_lookup_counters.json"))
    from bench import csrc_hash
    cnt = json.load(open(os.path.join(prof, "r2_lookup_counters.json")))
    print("counters hash", cnt["csrc_hash"], "tree", csrc_hash())
    print("\n".join(lines[7:16]))
    print(table)
    for w in WORKLOADS:
        d = json.load(open(os.path.join(prof, f"{tag}_bench_{w}.json")))
        cb = d.get("cpu_baseline") or {}
        print(w, round(d["value"] / 1e6, 3), "M/s", "cpu", round(cb.get("value") or 0),
              "frac", (d.get("roofline") or {}).get("frac"))


if __name__ == "__main__":
    main()
