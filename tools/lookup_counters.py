"""ncu counters of the XS lookup of the CURRENT build, normalised per
nuclide-lookup -> JSON read by bench.py's roofline block.

Two modes, both profiling `tools/profile_step.py` (one active batch of a
bench workload, default C4 on the HM core, 40M particles):

* full (default): every lookup launch of the batch (k_lookup_piped on the
  sorted sweeps, k_lookup_staged / k_lookup_warp on the tail) -- the batch's
  nuclide-lookups come from the run's counters;
* --sample S C: only k_lookup_piped launches S .. S+C-1 (the full-population
  sorted sweeps that dominate the step); their nuclide-lookups come from the
  engine's per-iteration trace (EMC_TRACE: cumulative nuclide-lookups after
  every sorted iteration, iteration i <-> piped launch i).  Fast enough to run
  inside bench.py after its timed region.

Per nuclide-lookup it reports DRAM bytes (read + write), L1TEX data-pipe
wavefronts (all, and shared-memory loads), warp instructions; plus the
time-weighted L1TEX data-pipe utilisation, FP64-pipe and issue activity, and
the data pipe's peak (wavefronts per cycle summed over SMs) and SM clock.

    python tools/lookup_counters.py [--out F] [--particles N] [--sample S C] [--workload W]
"""
import argparse
import ast
import csv
import io
import json
import os
import re
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

METRICS = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
           "l1tex__data_pipe_lsu_wavefronts.sum", "l1tex__data_pipe_lsu_wavefronts.sum.peak_sustained",
           "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
           "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
           "sm__cycles_elapsed.avg.per_second",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "smsp__inst_executed.sum"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "hz": 1.0, "Khz": 1e3, "Mhz": 1e6,
         "Ghz": 1e9, "cycle/nsecond": 1e9, "cycle/usecond": 1e6, "cycle/second": 1.0}
# design minimum of L1 data-pipe wavefronts per (warp, nuclide) in the staged
# fast path, all loads broadcast within a warp: window header 16 B (LDS.128: 2),
# (E0, r) 2, next E0 1, (t0,dt) (c0,dc) (f0,df) 6, (den, den*nu) 2
DESIGN_MIN_WAVEFRONTS = 13


def parse(csv_text: str):
    rows = list(csv.reader(io.StringIO(csv_text)))
    hi = [i for i, r in enumerate(rows) if "Metric Name" in r][0]
    h = rows[hi]
    ci, kn, cn, cv, cu = (h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"),
                          h.index("Metric Value"), h.index("Metric Unit"))
    launches = {}
    for r in rows[hi + 1:]:
        if len(r) <= cv:
            continue
        d = launches.setdefault(int(r[ci]), {"kernel": r[kn]})
        try:
            d[r[cn]] = float(r[cv].replace(",", "")) * SCALE.get(r[cu], 1.0)
        except ValueError:
            pass
    return [launches[k] for k in sorted(launches)]


def summarise(launches, nl: float, command: str) -> dict:
    def tot(k):
        return sum(x.get(k, 0.0) for x in launches)
    t = tot("gpu__time_duration.sum")

    def tw(k):     # time-weighted average
        return sum(x.get(k, 0.0) * x.get("gpu__time_duration.sum", 0.0) for x in launches) / t if t else None
    dram = tot("dram__bytes_read.sum") + tot("dram__bytes_write.sum")
    wf = tot("l1tex__data_pipe_lsu_wavefronts.sum")
    wf_sh = tot("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum")
    per_kernel = {}
    for x in launches:
        k = x["kernel"].split("<")[0].split("(")[0].replace("void ", "")
        p = per_kernel.setdefault(k, {"launches": 0, "time_s": 0.0})
        p["launches"] += 1
        p["time_s"] += x.get("gpu__time_duration.sum", 0.0)
    from bench import csrc_hash
    return {"command": command, "csrc_hash": csrc_hash(), "launches": len(launches), "per_kernel": per_kernel,
            "nuclide_lookups": nl, "serialised_kernel_s": t,
            "dram_bytes_read": tot("dram__bytes_read.sum"), "dram_bytes_write": tot("dram__bytes_write.sum"),
            "dram_bytes_per_nuclide_lookup": dram / nl,
            "dram_bytes_per_launch": dram / len(launches),
            "algorithmic_bytes_per_nuclide_lookup": 64,
            "l1_wavefronts_per_nuclide_lookup": wf / nl,
            "l1_wavefront_peak_per_cycle": tw("l1tex__data_pipe_lsu_wavefronts.sum.peak_sustained"),
            "sm_clock_hz": tw("sm__cycles_elapsed.avg.per_second"),
            "l1tex_data_pipe_pct": tw("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
            "fp64_pipe_pct": tw("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "issue_active_pct": tw("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "shared_ld_wavefronts": wf_sh,
            "shared_wavefronts_per_warp_nuclide": wf_sh / (nl / 32.0),
            "l1_wavefronts_per_warp_nuclide": wf / (nl / 32.0),
            "design_min_wavefronts_per_warp_nuclide": DESIGN_MIN_WAVEFRONTS,
            "warp_instructions_per_warp_nuclide": tot("smsp__inst_executed.sum") / (nl / 32.0)}


def sampled_nuclide_lookups(trace: str, skip: int, count: int) -> float:
    """Nuclide-lookups of sorted iterations skip..skip+count-1 of the first
    batch (cumulative counter after each iteration, reset per batch)."""
    rows = [(int(m.group(1)), int(m.group(2)), int(m.group(3))) for m in
            re.finditer(r"emc-trace iter (\d+) nL \d+ lookup_ms \S+ sorted (\d) nl_cum (\d+)", trace)]
    out, prev, k = 0, 0, 0
    for it, sorted_, c in rows:
        if it == 0:
            prev = 0
        if sorted_:
            if skip <= k < skip + count:
                out += c - prev
            k += 1
        prev = c
    return float(out)


def capture(particles: int, workload: str, sample=None, timeout: int = 900, log: str | None = None) -> dict:
    log = log or os.path.join(ROOT, "gpurun_out", "lookup_counters.csv")
    os.makedirs(os.path.dirname(log), exist_ok=True)
    kern = "k_lookup_piped" if sample else "k_lookup_(piped|staged|warp)"
    cmd = ["ncu", "--clock-control", "none", "--metrics", ",".join(METRICS), "-k", f"regex:{kern}", "--csv",
           "--log-file", log]
    if sample:
        cmd += ["-s", str(sample[0]), "-c", str(sample[1])]
    cmd += [sys.executable, os.path.join(ROOT, "tools", "profile_step.py"), "--particles", str(particles),
            "--workload", workload]
    env = dict(os.environ, EMC_TRACE="1") if sample else dict(os.environ)
    t0 = time.time()
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT, env=env)
    if p.returncode:
        raise RuntimeError(f"ncu failed ({p.returncode}): {p.stderr[-1500:]}")
    with open(log) as fh:
        launches = parse(fh.read())
    if sample:
        nl = sampled_nuclide_lookups(p.stderr, sample[0], len(launches))
    else:
        out = p.stdout
        timings = ast.literal_eval(out[out.index("timings ") + 8:].strip().splitlines()[0])
        nl = float(timings["nuclide_lookups_active"])
    what = (f"k_lookup_piped launches {sample[0]}..{sample[0] + len(launches) - 1}" if sample else
            "every lookup launch") + f" of one {workload} batch ({particles} particles), profile_step.py"
    res = summarise(launches, nl, "ncu --metrics ... " + what)
    res["workload"] = workload
    res["capture_wall_s"] = time.time() - t0
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2_lookup_counters.json"))
    ap.add_argument("--particles", type=int, default=40_000_000)
    ap.add_argument("--workload", default="c4")
    ap.add_argument("--sample", type=int, nargs=2, default=None, metavar=("SKIP", "COUNT"))
    ap.add_argument("--timeout", type=int, default=900)
    args = ap.parse_args()
    res = capture(args.particles, args.workload, args.sample, args.timeout)
    with open(args.out, "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
