"""ncu counters of the XS lookup over one whole C4 batch (40M particles) of
the CURRENT build -> profiles/<name>.json, read by bench.py's roofline
`binding` block.

Runs (on the GPU box)

    ncu --metrics <M> -k regex:"k_lookup_(piped|staged|warp)" --csv
        python tools/profile_step.py --particles 40000000

and aggregates every lookup launch: DRAM bytes (read + write), kernel time,
shared-memory LSU wavefronts, L1TEX throughput (time-weighted), FP64 pipe and
issue activity; divides by the batch's nuclide-lookups.  The result records
the hash of csrc/ it was captured on (bench.py reports whether it is current).

    python tools/lookup_counters.py [--out profiles/r2_lookup_counters.json] [--particles N]
"""
import argparse
import ast
import csv
import io
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

METRICS = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
           "l1tex__throughput.avg.pct_of_peak_sustained_active",
           "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
           "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
           "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "smsp__inst_executed.sum"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}
# design minimum of shared-memory wavefronts per (warp, nuclide) in the staged
# consumer: the 64-byte interval record as four 16-byte loads + the (den, den*nu)
# pair, all conflict-free broadcasts over <= 3 distinct intervals per warp
DESIGN_MIN_WAVEFRONTS = 5


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
        d = launches.setdefault(r[ci], {"kernel": r[kn]})
        d[r[cn]] = float(r[cv].replace(",", "")) * SCALE.get(r[cu], 1.0)
    return list(launches.values())


def summarise(launches, nl: float, command: str) -> dict:
    def tot(k):
        return sum(x.get(k, 0.0) for x in launches)
    t = tot("gpu__time_duration.sum")

    def tw(k):     # time-weighted average of a percentage
        return sum(x.get(k, 0.0) * x.get("gpu__time_duration.sum", 0.0) for x in launches) / t if t else None
    dram = tot("dram__bytes_read.sum") + tot("dram__bytes_write.sum")
    wf = tot("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum")
    per_kernel = {}
    for x in launches:
        k = x["kernel"].split("<")[0].split("(")[0]
        p = per_kernel.setdefault(k, {"launches": 0, "time_s": 0.0})
        p["launches"] += 1
        p["time_s"] += x.get("gpu__time_duration.sum", 0.0)
    from bench import csrc_hash
    return {"command": command, "csrc_hash": csrc_hash(), "launches": len(launches),
            "per_kernel": per_kernel,
            "nuclide_lookups": nl, "serialised_kernel_s": t,
            "dram_bytes_read": tot("dram__bytes_read.sum"), "dram_bytes_write": tot("dram__bytes_write.sum"),
            "dram_bytes_per_nuclide_lookup": dram / nl,
            "algorithmic_bytes_per_nuclide_lookup": 64,
            "l1tex_throughput_pct": tw("l1tex__throughput.avg.pct_of_peak_sustained_active"),
            "fp64_pipe_pct": tw("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "issue_active_pct": tw("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "shared_ld_wavefronts": wf,
            "shared_st_wavefronts": tot("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum"),
            "shared_bank_conflicts": tot("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
            "shared_wavefronts_per_warp_nuclide": wf / (nl / 32.0),
            "design_min_wavefronts_per_warp_nuclide": DESIGN_MIN_WAVEFRONTS,
            "warp_instructions_per_warp_nuclide": tot("smsp__inst_executed.sum") / (nl / 32.0)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2_lookup_counters.json"))
    ap.add_argument("--particles", type=int, default=40_000_000)
    ap.add_argument("--kernels", default="k_lookup_(piped|staged|warp)")
    ap.add_argument("--timeout", type=int, default=900)
    args = ap.parse_args()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    log = os.path.join(ROOT, "gpurun_out", "lookup_counters.csv")
    cmd = ["ncu", "--metrics", ",".join(METRICS), "-k", f"regex:{args.kernels}", "--csv", "--log-file", log,
           sys.executable, os.path.join(ROOT, "tools", "profile_step.py"), "--particles", str(args.particles)]
    t0 = time.time()
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=args.timeout, cwd=ROOT)
    if p.returncode:
        sys.exit(f"ncu failed ({p.returncode}): {p.stderr[-2000:]}")
    out = p.stdout
    timings = ast.literal_eval(out[out.index("timings ") + 8:].strip().splitlines()[0])
    nl = float(timings["nuclide_lookups_active"])
    with open(log) as fh:
        launches = parse(fh.read())
    res = summarise(launches, nl, " ".join(cmd[:6]) + f" ... profile_step.py --particles {args.particles}")
    res["capture_wall_s"] = time.time() - t0
    with open(args.out, "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
