"""Benchmark: active-batch particles/s on HM-large depleted fuel (C4).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload W]
    torchrun --nproc-per-node N bench.py --gpus N ...     (one rank per GPU, NCCL)

Workload (BASELINE.json configs[3], SURVEY.md section 8 "C4"): library
depleted_pincell generator (272 fuel, 3 moderator nuclides, 11303 grid
points, 100 axial depleted-fuel materials) seed 1 on the Hoogenboom-Martin
core (presets.hm_core: 241 17x17 assemblies, 323x323 pin lattice, 366 cm),
k-eigenvalue, event mode, sorted lookups, fused tallies, fast (atomic)
reduction, 40M particles per GPU per batch (weak scaling: ppb = N x 40M).
--workload c4pin runs the same library on the reference's own pin cell.
A step is one active batch; W warm-up batches (inactive: batch 0 samples the
source from scratch, later ones resample the bank) precede K timed active
batches.  The library (99.5 MB of grid records) is resident in HBM and every
batch re-reads it >100x over, so inputs are far larger than L2 in aggregate
traffic; no flush between batches is needed.

value     = K*ppb / device time of the K active batches (CUDA events on the
            engine stream, max over ranks)
e2e       = RunResult.active_rate of the same run_event() call: the
            reference's own metric definition (replication.py:282-304, host
            wall per batch incl. host merge/reduce/resample and the per-batch
            D2H of counters/tallies), i.e. through the public API.
roofline  = the XS lookup (k_lookup_piped; tail kernels on unsorted queues),
            bound by the L1TEX data pipe that serves the shared-memory-staged
            interval records: ncu wavefronts per nuclide-lookup (sampled on
            this build right after the timed region, tools/lookup_counters.py)
            x the run's nuclide-lookups x 128 B / the run's summed lookup time,
            against the pipe's peak.  `hbm` keeps north_star's gather model
            (64 B per nuclide-lookup: > HBM peak because staged
            records serve ~1000 particles per DRAM read) and measured DRAM.
"""

from __future__ import annotations

import argparse
import json
import os
import shutil
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "particles/s (active batches), HM-large depleted fuel, at 1/2/4/8 B200"
GUARD_NOTE = ("box_guard on (RunConfig extension, include/emc.h): the reference's nudge can lose a particle "
              "outside the reflective box (~1 per 1e9 histories; seed 42 stops batch 22 without it, "
              "profiles/r2_c4_escape_replay.md); histories that stay inside are bit-identical to the reference")
WORKLOAD = dict(workload="C4 HM-large depleted fuel on the Hoogenboom-Martin core: hm_core(272,3,11303,100,seed=1): "
                         "241 assemblies x 264 pins (17x17, 25 tubes), 323x323 pin lattice with water reflector, "
                         "366 cm, 100 axial depleted-fuel zones, reflective",
                ppb_per_gpu=40_000_000, mode="event", reduction="fast", tally_mode="fused",
                sort="on (group, log E, mat) every lookup sweep", seed=42, box_guard=GUARD_NOTE)
# --workload c5: BASELINE configs[4] (SURVEY 8f row 1 extension)
METRIC_C5 = "particles/s (active batches), fixed-source shielding slab with 3D mesh flux tallies"
WORKLOAD_C5 = dict(workload="C5 shielding_slab(8 nuclides/material, 2000 points, 12 layers, 60x60x60 cm, "
                            "vacuum), surface source, mesh 100x100x120 track-length (flux, total)",
                   ppb_per_gpu=10_000_000, mode="event", reduction="fast", run_mode="fixed_source",
                   mesh=(100, 100, 120), seed=42)


# --workload c1: BASELINE configs[0] (the reference's own CPU-runnable case, SURVEY 8 "C1")
METRIC_C1 = "particles/s (active batches), UO2 pincell, 12 fuel nuclides (C1)"
WORKLOAD_C1 = dict(workload="C1 pincell: depleted_pincell(12,3,100,8,seed=1), 10k particles/batch", ppb_per_gpu=10_000,
                   mode="event", reduction="deterministic", seed=42, box_guard=GUARD_NOTE)
# --workload c3: BASELINE configs[2] (Hoogenboom-Martin small: fresh fuel, 34 fuel nuclides, HM core)
METRIC_C3 = "particles/s (active batches), HM-small fresh fuel (34 fuel nuclides), HM core"
WORKLOAD_C3 = dict(workload="C3 HM-small on the Hoogenboom-Martin core: hm_core(34,3,11303,100,seed=1), "
                            "10M particles/batch",
                   ppb_per_gpu=10_000_000, mode="event", reduction="fast", seed=42, box_guard=GUARD_NOTE)
# --workload c2: BASELINE configs[1] (17x17 assembly, SURVEY 8f row 2 extension)
METRIC_C2 = "particles/s (active batches), 2D 17x17 PWR assembly, ~30 nuclides"
WORKLOAD_C2 = dict(workload="C2 pwr_assembly(27 fuel + 3 moderator nuclides, 11303 points, 17x17 lattice, "
                            "25 water holes, 2D reflective), k-eigenvalue",
                   ppb_per_gpu=1_000_000, mode="event", reduction="fast", seed=42, box_guard=GUARD_NOTE)


# --workload c4pin / c3pin: the same libraries on the reference's own geometry,
# the single pin cell (kernels.py:418-492) with 100 axial zones in 10 cm
METRIC_C4PIN = "particles/s (active batches), HM-large depleted fuel library on the reference pin cell"
WORKLOAD_C4PIN = dict(workload="C4 library on the pincell: depleted_pincell(272,3,11303,100,seed=1)",
                      ppb_per_gpu=40_000_000, mode="event", reduction="fast", tally_mode="fused",
                      sort="on (group, log E, mat) every lookup sweep", seed=42, box_guard=GUARD_NOTE)
METRIC_C3PIN = "particles/s (active batches), HM-small fresh fuel library (34 fuel nuclides) on the reference pin cell"
WORKLOAD_C3PIN = dict(workload="C3 library on the pincell: depleted_pincell(34,3,11303,100,seed=1), 10M particles/batch "
                               "(seed 42 stops in batch 5 without the box guard, profiles/r1s5_c3_reference_error.txt)",
                      ppb_per_gpu=10_000_000, mode="event", reduction="fast", seed=42, box_guard=GUARD_NOTE)
METRICS = {"c1": METRIC_C1, "c2": METRIC_C2, "c3": METRIC_C3, "c5": METRIC_C5, "c4pin": METRIC_C4PIN,
           "c3pin": METRIC_C3PIN}
WORKLOADS = {"c1": WORKLOAD_C1, "c2": WORKLOAD_C2, "c3": WORKLOAD_C3, "c5": WORKLOAD_C5, "c4pin": WORKLOAD_C4PIN,
             "c3pin": WORKLOAD_C3PIN}


def problem(args):
    import paper_2403_12345_b200 as P
    if args.workload == "c4pin":
        return P.depleted_pincell(272, 3, 11303, 100, seed=1)
    if args.workload == "c3pin":
        return P.depleted_pincell(34, 3, 11303, 100, seed=1)
    if args.workload == "c5":
        return P.shielding_slab()
    if args.workload == "c2":
        return P.pwr_assembly()
    if args.workload == "c3":
        return P.hm_core(34, 3, 11303, 100, seed=1)
    if args.workload == "c1":
        return P.depleted_pincell(12, 3, 100, 8, seed=1)
    return P.hm_core(272, 3, 11303, 100, seed=1)


BYTES_PER_NUCLIDE_LOOKUP = 64
# ncu counters of the XS-lookup kernels over one C4 batch of the CURRENT build
# (tools/lookup_counters.py writes it with the hash of csrc/ it was captured on)
LOOKUP_COUNTERS = "r2_lookup_counters.json"


def csrc_hash() -> str:
    import hashlib
    h = hashlib.sha256()
    d = os.path.join(ROOT, "paper_2403_12345_b200", "csrc")
    for f in sorted(os.listdir(d)):
        if f.endswith((".cu", ".cuh", ".h")):
            with open(os.path.join(d, f), "rb") as fh:
                h.update(f.encode() + fh.read())
    return h.hexdigest()[:16]


def lookup_counters(args, ppb: int) -> dict:
    """ncu counters of the XS lookup of THIS build, per nuclide-lookup
    (tools/lookup_counters.py): measured right after the timed region on a
    sample of full-population k_lookup_piped launches of one batch of the same
    workload in a child process (counters cannot be read inside a timed run);
    if ncu is unavailable, the committed profiles/LOOKUP_COUNTERS capture,
    flagged `current` when it was taken on this source hash."""
    err = None
    if not args.no_counters and shutil.which("ncu") and not os.environ.get("CUDA_INJECTION64_PATH"):
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        try:
            import lookup_counters as LC
            import tempfile
            with tempfile.TemporaryDirectory() as td:
                prof = LC.capture(ppb, args.workload, sample=(2, 4), timeout=240, log=os.path.join(td, "lc.csv"))
            prof["source"] = "live: " + prof["command"]
            prof["current"] = True
            return prof
        except Exception as e:  # noqa: BLE001
            err = f"{type(e).__name__}: {str(e)[:200]}"
    path = os.path.join(ROOT, "profiles", LOOKUP_COUNTERS)
    try:
        with open(path) as fh:
            prof = json.load(fh)
    except (OSError, ValueError):
        return {"source": None, "error": err}
    if prof.get("workload", "c4") != args.workload:
        return {"source": None, "error": err or f"committed counters are for {prof.get('workload', 'c4')}"}
    prof["source"] = f"profiles/{LOOKUP_COUNTERS} ({prof.get('command', 'ncu')})"
    prof["current"] = prof.get("csrc_hash") == csrc_hash()
    if err:
        prof["live_error"] = err
    return prof


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """Clocks/throttle sampling over the timed region: NVML in-process (the
    library behind nvidia-smi), else `nvidia-smi --query-gpu` (BENCH_CLOCKS=smi).
    The sampling thread is started before the run (its NVML initialisation must
    not land inside the timed region of short batches); `mark()` brackets the
    timed region and only samples inside it (or the two nearest ones, for
    regions shorter than the sampling period) are reported."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    PERIOD = float(os.environ.get("BENCH_CLOCKS_PERIOD", "0.5"))   # faster polling perturbs short batches

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []            # (monotonic time, fields)
        self.window = [None, None]
        self._stop = threading.Event()
        self._t = None

    def _run_nvml(self):
        import pynvml as nv
        nv.nvmlInit()
        try:
            h = nv.nvmlDeviceGetHandleByIndex(self.gpu)
            mx = str(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))   # a slow query (ms): once
            bits = (0x8, 0x40, 0x20, 0x4)      # hw_slowdown, hw_thermal, sw_thermal, sw_power_cap
            while not self._stop.is_set():
                try:
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                except AttributeError:
                    r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                self.rows.append((time.monotonic(),
                                  [str(self.gpu), str(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)), mx,
                                   str(nv.nvmlDeviceGetPowerUsage(h) / 1000.0), hex(r)]
                                  + ["Active" if r & b else "Not Active" for b in bits]))
                self._stop.wait(self.PERIOD)
        finally:
            nv.nvmlShutdown()

    def _run(self):
        if os.environ.get("BENCH_CLOCKS") == "none":
            return
        if os.environ.get("BENCH_CLOCKS", "nvml") == "nvml":
            try:
                self._run_nvml()
                return
            except Exception:  # noqa: BLE001
                self.rows = []
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), "--format=csv,noheader,nounits",
                                      f"--query-gpu={self.FIELDS}"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append((time.monotonic(), [c.strip() for c in out.split(",")]))
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(0.2)

    def start(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def mark(self, which: int):
        self.window[which] = time.monotonic()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        t0, t1 = self.window
        rows = [r for ts, r in self.rows if t0 is not None and t1 is not None and t0 <= ts <= t1]
        if not rows and self.rows and t0 is not None:
            before = [r for ts, r in self.rows if ts < t0][-1:]
            after = [r for ts, r in self.rows if t1 is not None and ts > t1][:1]
            rows = before + after
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for r in rows:
            for name, v in zip(names, r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(rows)}


def init_dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    forced = os.environ.get("EMC_FORCE_COLLECTIVES") == "1" and "RANK" in os.environ
    if ws <= 1 and not forced:
        return 0, 1, 0
    import torch
    import torch.distributed as dist
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, ws, local


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _oracle_ext(args, cell) -> dict:
    """Oracle configuration of the workload's extensions (same as the GPU arm)."""
    ext = {}
    if args.workload == "c5":
        ext = dict(run_mode="fixed_source", mesh=WORKLOAD_C5["mesh"], slab=True, vacuum=True)
    else:
        ext = dict(box_guard=True)
    if cell.lattice > 1:
        ext["lattice"] = (cell.lattice, cell.pitch, cell.pin_map)
    return ext


def _oracle_run(lib, cell, ext, threads, ppb, inactive, active, mode):
    from oracle import driver
    cfg = dict(particles_per_batch=ppb, inactive_batches=inactive, active_batches=active,
               mode=mode, max_in_flight=10000, tally_mode="fused", reduction="deterministic",
               sort_enabled=True, sort_every_n=1, seed=42, workers=threads, **ext)
    return driver.run(cfg, lib.arrays(), cell.as_tuple(), workers=threads)


def cpu_baseline(args, lib, cell, threads: int, ppb_sample: int, batches=(1, 2)) -> dict:
    """The C oracle (restatement of the reference kernels, pinned bit-exact to
    it) on this host's cores, W workers like run_replicated, in both of the
    reference's executors; the faster one is the
    baseline."""
    ext = _oracle_ext(args, cell)
    rates = {}
    for mode in ("event", "history"):
        res = _oracle_run(lib, cell, ext, threads, ppb_sample, batches[0], batches[1], mode)
        rates[mode] = res["active_rate"]
    best = max(rates, key=rates.get)
    return dict(value=rates[best], unit="particles/s", cores=threads, kind="port", mode=best,
                rates=rates, cpu_model=cpu_model(),
                sample=f"{args.workload.upper()} library, {ppb_sample} particles/batch x ({batches[0]} inactive + "
                       f"{batches[1]} active) in event and in history mode, {threads} worker threads, "
                       f"deterministic reduction (reference defaults); value = the faster mode ({best})")


def run_reference(args):
    """--impl reference: the reference's CPU path (oracle port; the reference
    is Python/numba and cannot travel to the GPU box) on all host cores, in
    both of its executors (event: the reference default; history: CPU-optimal,
    PAPER.md:70); the line reports the faster one."""
    # CPU only: no process group (rank 0 works, the other ranks exit at once;
    # an NCCL group the other ranks abandon could hang rank 0's exit)
    rank = int(os.environ.get("RANK", "0"))
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    lib, cell = problem(args)
    c5 = args.workload == "c5"
    threads = os.cpu_count() or 1
    ppb = args.ref_particles or (30000 if c5 else 3000) * threads
    ext = _oracle_ext(args, cell)
    runs = {}
    for mode in ("event", "history"):
        runs[mode] = _oracle_run(lib, cell, ext, threads, ppb, args.warmup, args.steps, mode)
    best = max(runs, key=lambda m: runs[m]["active_rate"])
    res = runs[best]
    v = res["active_rate"]
    line = {"impl": "reference", "metric": METRICS.get(args.workload, METRIC),
            "value": v, "unit": "particles/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * res["active_wall"] / max(args.steps, 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": dict(WORKLOADS.get(args.workload, WORKLOAD),
                           mode=best, reduction="deterministic (reference default)",
                           ppb_sample=ppb,
                           impl="C restatement of the reference kernels (oracle/, bit-exact with the "
                                "numba reference on this image's glibc)"),
            "cpu_baseline": {"value": v, "unit": "particles/s", "cores": threads, "kind": "port",
                             "cpu_model": cpu_model(), "mode": best,
                             "rates": {m: r["active_rate"] for m, r in runs.items()},
                             "sample": f"{ppb} particles/batch x ({args.warmup}+{args.steps}) batches, "
                                       f"event and history executors, the faster reported"},
            "e2e": {"value": v, "unit": "particles/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    rank, ws, local = init_dist()
    import paper_2403_12345_b200 as P
    from paper_2403_12345_b200 import replication
    from paper_2403_12345_b200.distributed import current_world

    t0 = time.perf_counter()
    lib, cell = problem(args)
    t_lib = time.perf_counter() - t0
    c5 = args.workload == "c5"
    wl = WORKLOADS.get(args.workload, WORKLOAD)
    ppb_gpu = args.particles or wl["ppb_per_gpu"]
    ext = dict(run_mode="fixed_source", mesh=WORKLOAD_C5["mesh"]) if c5 else dict(box_guard=True)
    cfg = P.RunConfig(particles_per_batch=ppb_gpu * ws, inactive_batches=args.warmup,
                      active_batches=args.steps, mode="event", sort_enabled=True,
                      max_in_flight=args.max_in_flight or ppb_gpu, tally_mode="fused",
                      reduction=wl["reduction"], seed=wl["seed"], workers=ws, **ext)
    dev = torch.cuda.current_device()
    eng = replication.engine_for(dev, lib, cell)
    stream = torch.cuda.current_stream()
    eng.set_stream(stream.cuda_stream)
    ev = {}
    launches0 = {}
    sampler = ClockSampler(local).start()

    def on_batch(b, phase, e):
        if b == args.warmup and phase == "start":
            if torch.distributed.is_initialized():
                torch.distributed.barrier()
            torch.cuda.synchronize()
            sampler.mark(0)
            ev["start"] = torch.cuda.Event(enable_timing=True)
            ev["start"].record(stream)
            launches0["n"] = e.launch_count
        if b == args.warmup + args.steps - 1 and phase == "end":
            ev["end"] = torch.cuda.Event(enable_timing=True)
            ev["end"].record(stream)
            torch.cuda.synchronize()
            launches0["end"] = e.launch_count
            sampler.mark(1)

    try:
        res = P.run_event(cfg, lib, cell, on_batch=on_batch)
    finally:
        sampler.stop()
    dev_ms = ev["start"].elapsed_time(ev["end"])
    if torch.distributed.is_initialized():
        t = torch.tensor([dev_ms], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        dev_ms = float(t.item())
    value = args.steps * cfg.particles_per_batch / (dev_ms * 1e-3)
    if rank != 0:
        return
    # roofline of the XS-lookup kernel (timings are summed over ranks; per-rank mean)
    n_nl = res.timings["nuclide_lookups_active"]
    peak, peak_src = _peaks()
    lk_time = res.timings["lookup_active_s"] / ws if "lookup_active_s" in res.timings else None
    achieved = (BYTES_PER_NUCLIDE_LOOKUP * n_nl / ws) / lk_time / 1e9 if lk_time else None
    clocks = sampler.summary()
    # roofline: the lookup's binding unit is the L1TEX data pipe (shared-memory
    # staged records), not HBM -- wavefronts per nuclide-lookup from ncu on this
    # build x this run's nuclide-lookups / this run's lookup time (CUDA events)
    # (gather-lookup workloads -- C1, C5 -- have no staged lookup to sample)
    prof = lookup_counters(args, ppb_gpu) if ws == 1 and args.workload not in ("c1", "c5") else {"source": None}
    wf = prof.get("l1_wavefronts_per_nuclide_lookup")
    l1_peak = l1_ach = None
    if wf and prof.get("l1_wavefront_peak_per_cycle") and lk_time:
        clk = (clocks.get("sm_mhz") or 0) * 1e6 or prof.get("sm_clock_hz")
        l1_peak = prof["l1_wavefront_peak_per_cycle"] * 128 * clk / 1e9
        l1_ach = wf * 128 * (n_nl / ws) / lk_time / 1e9
    nlaunch = res.timings.get("lookup_launches_active", 0) / ws
    dram_nl = prof.get("dram_bytes_per_nuclide_lookup")
    dram_gbs = dram_nl * (n_nl / ws) / lk_time / 1e9 if dram_nl and lk_time else None
    line = {
        "metric": METRICS.get(args.workload, METRIC), "value": value,
        "unit": "particles/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": dict(wl, global_batch=cfg.particles_per_batch,
                       parallelism=f"domain replication x{ws}", l2="inputs >> L2 in traffic; no flush",
                       library_build_s=round(t_lib, 2)),
        "e2e": {"value": res.active_rate, "unit": "particles/s",
                "h2d_bytes_per_step": res.timings.get("h2d_bytes_active", 0) / max(args.steps, 1),
                "d2h_bytes_per_step": res.timings.get("d2h_bytes_active", 0) / max(args.steps, 1),
                "d2h_bytes_final_bank": res.timings.get("d2h_bytes_final_bank", 0)},
        "gpu_launches": int(launches0["end"] - launches0["n"]),
        "roofline": {"bound": "l1tex", "achieved": l1_ach, "peak": l1_peak, "unit": "GB/s",
                     "frac": (l1_ach / l1_peak) if l1_ach and l1_peak else None,
                     "traffic": dram_nl * (n_nl / ws) / nlaunch if dram_nl and nlaunch else None,
                     "kernel": "XS lookup: every lookup launch of the active batches (k_lookup_piped on sorted "
                               "sweeps, k_lookup_staged / k_lookup_warp on unsorted tail queues), time summed "
                               "from CUDA events on the engine stream",
                     "meaning": "L1TEX data-pipe bytes delivered (128 B per wavefront; ncu wavefronts per "
                                "nuclide-lookup of this build x this run's nuclide-lookups) / lookup time, vs the "
                                "data pipe's peak (wavefronts per cycle x 128 B x live SM clock): the staged "
                                "lookup serves every interval record from shared memory, so this pipe -- not "
                                "HBM -- binds it",
                     "counters": {k: prof.get(k) for k in (
                         "source", "current", "live_error", "l1_wavefronts_per_warp_nuclide",
                         "shared_wavefronts_per_warp_nuclide", "design_min_wavefronts_per_warp_nuclide",
                         "l1tex_data_pipe_pct", "fp64_pipe_pct", "issue_active_pct",
                         "warp_instructions_per_warp_nuclide", "dram_bytes_per_nuclide_lookup") if k in prof},
                     "hbm": {"peak": peak, "peak_source": peak_src, "unit": "GB/s",
                             "algorithmic": achieved,
                             "algorithmic_frac": (achieved / peak) if achieved else None,
                             "algorithmic_bytes": "64 B x nuclide-lookups (grid pair + sigma_t,c,f pairs, "
                                                  "SURVEY 8d); > peak because each staged record byte read from "
                                                  "DRAM serves ~1000 particles",
                             "dram_measured": dram_gbs,
                             "dram_frac": (dram_gbs / peak) if dram_gbs else None},
                     "nuclide_lookups_per_step": n_nl / args.steps},
        "clocks": clocks,
        "k_mean": res.k_mean, "k_stderr": res.k_stderr,
        "box_guard_events": res.counters.get("box_guard"),
        "timings_s": {k: v for k, v in res.timings.items() if isinstance(v, float)},
    }
    if l1_ach is None:
        # no staged-lookup counters (gather-lookup workloads, or ncu unavailable):
        # the HBM gather model of SURVEY 8d is the roofline reported
        r = line["roofline"]
        r.update(bound="hbm", achieved=achieved, peak=peak, unit="GB/s",
                 frac=(achieved / peak) if achieved else None, traffic=None,
                 meaning="north_star's HBM gather model: 64 B per nuclide-lookup / summed lookup time vs the "
                         "measured HBM peak (no L1TEX counters for this workload)")
    if ws == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        line["cpu_baseline"] = cpu_baseline(args, lib, cell, threads, args.cpu_particles or (
            10000 if args.workload in ("c4", "c3", "c4pin", "c3pin") else 4000) * threads)
    if c5:
        line["mesh"] = {"cells": int(np.prod(WORKLOAD_C5["mesh"])),
                        "flux_first_layer": float(res.mesh_mean[0, ..., 0].sum()),
                        "leaks": res.counters.get("leaks")}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--particles", type=int, default=0,
                    help="particles per GPU per batch (default 40M for c4, 10M for c5)")
    ap.add_argument("--workload", default="c4", choices=("c4", "c1", "c2", "c3", "c5", "c4pin", "c3pin"),
                    help="c4: headline HM-large eigenvalue (BASELINE metric); c2: 17x17 assembly; "
                         "c3: HM-small; c5: fixed-source slab + mesh")
    ap.add_argument("--max-in-flight", type=int, default=0)
    ap.add_argument("--cpu-particles", type=int, default=0)
    ap.add_argument("--ref-particles", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-counters", action="store_true",
                    help="skip the post-run ncu sample of the lookup (roofline counters)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)
    try:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            dist.destroy_process_group()
    except Exception:  # noqa: BLE001
        pass


if __name__ == "__main__":
    main()
