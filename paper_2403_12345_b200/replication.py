"""Batch coordinator: the drop-in ``run_replicated`` (eventmc/replication.py,
R:<line>) over the GPU engine, plus the weak-scaling harness.

Per batch (R:198-286): run this rank's particle block on its GPU
(emc_run_batch: source, event loop, canonical bank sort), map device error
codes to exceptions (R:214-219), gather the bank and reduce tallies across
ranks (distributed.py), compute k (R:243-249), check neutron bookkeeping
(R:250-257), accumulate counters (R:259-269) and resample the next source
from the global canonical bank (R:271-280).

Ranks and GPUs.  Under torch.distributed (torchrun, one process per GPU)
each rank drives its own GPU.  In a single process ``config.workers = W``
(the reference's worker-thread count) drives min(W, visible GPUs) devices,
one host thread per device, with the collectives of distributed.ThreadGroup
(peer copies for the bank windows); physics is worker-invariant (the
reference's acceptance criterion 2), so W beyond the GPU count only changes
the assignment, never the result.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, replace

import numpy as np

from . import prng, xslib
from .distributed import (BANK_DTYPES, ThreadGroup, World, allgather_array, allreduce_tensor,
                          block_of, chained_fold, combine_counters, current_world, device_view,
                          exchange_bank, gather_bank)
from .engine import DeviceEngine
from .errors import (ConfigurationError, EventMCError, GeometryError, PhysicsError,
                     PopulationCollapseError, RunawayHistoryError, StreamOverlapError)
from .tally import KeffSeries, TallyLayout, batch_statistics
from .transport import FissionBank, RunConfig, RunResult

# device error code -> (exception, message)   (R:28-38)
_ERRORS = {
    1: (GeometryError, "no boundary intersection"),
    2: (GeometryError, "particle outside the cell box"),
    3: (StreamOverlapError, "history consumed a full RNG stride"),
    4: (RunawayHistoryError, "history exceeded the contribution-log cap"),
    5: (EventMCError, "event queue invariant violated"),
    6: (PhysicsError, "sigma_t <= 0 (void materials unsupported)"),
}
# counter indices: kernels.py:81-103
_COUNTER_SUMS = (("captures", 5), ("fissions", 6), ("sourced", 7), ("energy_clamps", 9),
                 ("interp_transport", 10), ("interp_score", 11), ("events_lookup", 12),
                 ("events_advance", 13), ("events_collision", 14), ("invocations_lookup", 15),
                 ("invocations_advance", 16), ("invocations_collision", 17), ("sorts", 18))
_COUNTER_MAXES = (("max_draws_per_history", 8), ("max_log_entries_per_history", 20),
                  ("max_in_flight_observed", 19))
_COUNTER_LEAKS = (("leaks", 22),)          # extension: vacuum boundaries
_COUNTER_GUARD = (("box_guard", 23),)      # extension: RunConfig.box_guard

_ENGINES: dict[tuple[int, int], DeviceEngine] = {}


def engine_for(device: int, library, pincell, slot: int = 0) -> DeviceEngine:
    """Per-(device, slot) engine reused across runs; re-uploads changed
    inputs only.  `slot` > 0 only when several ranks share one GPU (tests)."""
    eng = _ENGINES.get((device, slot))
    if eng is None:
        eng = _ENGINES[(device, slot)] = DeviceEngine(device)
    if eng.library_obj is None or eng.library_obj() is not library:
        eng.upload_library(library)
    if eng.pincell_obj is None or eng.pincell_obj() is not pincell:
        eng.upload_geometry(pincell)
    return eng


def _local_device(world: World) -> int:
    if world.threads:
        return world.device
    if not world.distributed:
        return 0
    import torch
    return torch.cuda.current_device() if world.device_backend else 0


def _device_count() -> int:
    from . import _native
    try:
        return _native.device_count()
    except Exception:  # noqa: BLE001
        return 0


def resolve_devices(config: RunConfig, devices=None) -> list[int]:
    """GPUs a single-process run drives: `devices` if given (a device may be
    listed twice: several ranks on one GPU, for tests), else the first
    min(config.workers, visible GPUs)."""
    if devices is not None:
        devices = [int(d) for d in devices]
        if not devices:
            raise ConfigurationError("devices must not be empty")
        if len(devices) > config.particles_per_batch:
            raise ConfigurationError("more devices than particles per batch")
        return devices
    n = _device_count()
    return list(range(max(1, min(config.workers, n))))


def run_replicated(config: RunConfig, library, pincell, index=None, *,
                   on_batch=None, devices=None) -> RunResult:
    """Run the configured k-eigenvalue (or fixed-source) problem.

    Under torch.distributed: this rank's block on this process's GPU.
    Otherwise: ``resolve_devices(config, devices)`` GPUs, one thread each.
    ``on_batch(b, phase, engine)`` (phase 'start'/'end') is an optional
    instrumentation hook (bench.py records CUDA events through it; rank 0's
    engine only)."""
    config.validate()
    for mid in list(pincell.fuel_material_ids) + [pincell.moderator_material_id]:
        if mid < 0 or mid >= library.n_materials:
            raise ConfigurationError(f"geometry references material {mid} "
                                     f"but the library has {library.n_materials}")
    index = _union_for(config, library, index)

    world = current_world()
    if world.distributed:
        if devices is not None:
            raise ConfigurationError("devices= is for single-process runs; under "
                                     "torch.distributed each rank uses its own GPU")
        return _run_rank(config, library, pincell, world, on_batch, index=index)
    devs = resolve_devices(config, devices)
    if len(devs) == 1:
        return _run_rank(config, library, pincell, World(device=devs[0]), on_batch, index=index)
    return _run_threads(config, library, pincell, devs, on_batch, index)


def _union_for(config: RunConfig, library, index):
    """R:145-152: the union index the lookup backend needs (built when not
    given; merged channels materialized for "unionized"); None for binary."""
    if config.accel == "binary":
        return None
    if index is None:
        index = xslib.build_unionized_index(library)
    if config.accel == "unionized" and index.merged_channels is None:
        xslib.merge_channels(library, index)
    return index


def _run_threads(config, library, pincell, devs, on_batch, index=None) -> RunResult:
    import threading

    import torch
    torch.cuda.init()                           # once, before the device threads start
    group = ThreadGroup(len(devs))
    results: list = [None] * len(devs)
    errors: list = [None] * len(devs)
    seen: dict[int, int] = {}
    slots = []
    for d in devs:
        slots.append(seen.get(d, 0))
        seen[d] = seen.get(d, 0) + 1

    def body(r):
        try:
            torch.cuda.set_device(devs[r])
            w = World(rank=r, size=len(devs), device_backend=True, group=group, device=devs[r])
            results[r] = _run_rank(config, library, pincell, w, on_batch if r == 0 else None,
                                   slot=slots[r], index=index)
        except BaseException as e:  # noqa: BLE001
            errors[r] = e
            group.abort()

    threads = [threading.Thread(target=body, args=(r,), name=f"emc-rank{r}") for r in range(len(devs))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    real = [e for e in errors if e is not None and not isinstance(e, threading.BrokenBarrierError)]
    if real:
        raise real[0]
    if any(e is not None for e in errors):
        raise errors[0]
    return results[0]


def _run_rank(config: RunConfig, library, pincell, world: World, on_batch, slot: int = 0,
              index=None) -> RunResult:
    """One rank's share of run_replicated; the returned RunResult is complete
    on rank 0 (global k, tallies, counters, final bank)."""
    ppb = config.particles_per_batch
    if world.distributed and world.size > ppb:
        raise ConfigurationError("more ranks than particles per batch")
    g_lo, g_hi = block_of(world.rank, world.size, ppb)
    eng = engine_for(_local_device(world), library, pincell, slot)
    eng.set_accel(config.accel, index)
    eng.set_extensions(pincell, config)
    eng.configure(config, g_lo, g_hi - g_lo)
    fixed_source = config.run_mode == "fixed_source"
    mesh = _MeshAccumulator(world, eng, config) if config.mesh is not None else None

    layout = TallyLayout(pincell.n_axial)
    use_logs = config.reduction == "deterministic"
    weight = float(ppb)
    n_batches = config.n_batches
    batch_sums = np.zeros((n_batches, layout.n_bins))
    keff_values = np.zeros(n_batches)
    run_counters: dict[str, int] = {}
    timings = {"lookup": 0.0, "advance": 0.0, "collision": 0.0, "sort": 0.0,
               "reduce": 0.0, "merge": 0.0}
    inactive_wall = active_wall = 0.0
    k_run = 1.0
    last_local = last_counts = None
    launches = 0
    nuclide_lookups_active = 0
    act = dict(lookup_active_s=0.0, lookup_launches_active=0, h2d_bytes_active=0,
               d2h_bytes_active=0)

    for b in range(n_batches):
        active = b >= config.inactive_batches
        if on_batch is not None:
            on_batch(b, "start", eng)
        t_batch = time.perf_counter()
        out = eng.run_batch(b, k_run, batch0=(b == 0), score=active)
        launches += out.launches
        # ONE small all-gather per batch carries every per-rank scalar:
        # error, site count, iterations, the 24 counters, the 4 timings (as
        # bit patterns) and, in fast mode, the tally bins (bit patterns)
        t0 = time.perf_counter()
        fast = None if use_logs else eng.reduce_bins(None)
        pack = np.concatenate([np.array([out.error, out.error_gid, out.n_sites, out.iterations], np.int64),
                               np.asarray(out.counters, np.int64),
                               np.ascontiguousarray(out.timings, np.float64).view(np.int64)] +
                              ([np.ascontiguousarray(fast, np.float64).view(np.int64)] if fast is not None else []))
        allp = allgather_array(world, pack)
        nc = out.counters.shape[0]
        nt = out.timings.shape[0]
        per_rank = allp[:, 4:4 + nc]
        tim_rank = np.ascontiguousarray(allp[:, 4 + nc:4 + nc + nt]).view(np.float64)
        for code, gid in allp[:, :2]:
            if code:
                cls, msg = _ERRORS[int(code)]
                raise cls(f"{msg} (batch {b}, particle {int(gid)})")

        # fission bank: global canonical order = rank-ordered concatenation;
        # each rank receives only the window its next batch resamples from
        counts = allp[:, 2].copy()
        n_bank = int(counts.sum())
        local = None
        if world.distributed:
            local = [device_view(p, max(out.n_sites, 1), dt, eng.device)
                     for p, dt in zip(eng.bank_device_ptrs(), BANK_DTYPES)] \
                if world.device_backend else \
                [__import__("torch").as_tensor(c) for c in eng.bank_to_host()]

        # tallies + k
        if use_logs:
            sums = chained_fold(world, lambda init: eng.reduce_bins(init), layout.n_bins)
        else:
            bins_rank = np.ascontiguousarray(allp[:, 4 + nc + nt:]).view(np.float64)
            sums = np.zeros(layout.n_bins)
            for r in range(bins_rank.shape[0]):       # rank order (R:238-240)
                sums += bins_rank[r]
        timings["reduce"] += time.perf_counter() - t0
        batch_sums[b] = sums
        keff_values[b] = sums[layout.keff_bin] / weight

        if mesh is not None and active:
            mesh.add_batch()
        sourced = int(per_rank[:, 7].sum())
        deaths = int(per_rank[:, 5].sum() + per_rank[:, 6].sum() + per_rank[:, 22].sum())
        if sourced != ppb or deaths != ppb:
            raise EventMCError(f"neutron bookkeeping broken in batch {b}: {sourced} sourced, "
                               f"{deaths} absorbed or leaked, {ppb} expected")
        sums_spec = _COUNTER_SUMS + (_COUNTER_LEAKS if pincell.boundary == "vacuum" else ()) + \
            (_COUNTER_GUARD if config.box_guard else ())
        batch_counters = combine_counters(per_rank, sums_spec, _COUNTER_MAXES)
        for name, _ in sums_spec:
            run_counters[name] = run_counters.get(name, 0) + batch_counters[name]
        for name, _ in _COUNTER_MAXES:
            run_counters[name] = max(run_counters.get(name, 0), batch_counters[name])
        if active:
            nuclide_lookups_active += int(per_rank[:, 21].sum())
            act["lookup_active_s"] += float(tim_rank[:, 0].sum())
            act["lookup_launches_active"] += int(allp[:, 3].sum())
            # host<->device traffic of the batch: control block per iteration,
            # counters + tally bins at the end (engine.py / emc_engine.cu)
            act["h2d_bytes_active"] += 48 + 64
            act["d2h_bytes_active"] += 48 * (out.iterations + 2) + 24 * 8 + layout.n_bins * 8
        tim = tim_rank.sum(axis=0)
        for key, i in (("lookup", 0), ("advance", 1), ("collision", 2), ("sort", 3)):
            timings[key] += float(tim[i])

        # population control for the next batch (R:271-280); a fixed-source
        # run samples its source afresh every batch (extension)
        if b < n_batches - 1 and fixed_source:
            pass
        elif b < n_batches - 1:
            if n_bank == 0:
                raise PopulationCollapseError(f"no fission sites banked in batch {b}")
            u, _ = prng.next_uniform(prng.batch_stream(config.seed, b))
            if world.distributed:
                t0 = time.perf_counter()
                src, lo = exchange_bank(world, local[2:9], counts, ppb, u)
                if not world.device_backend:     # gloo (tests): stage the window on this GPU
                    src = _host_to_device_bank(eng, src)
                timings["merge"] += time.perf_counter() - t0
                eng.set_source_device([t.data_ptr() for t in src], n_bank, u, keep=src, lo=lo)
            else:
                eng.set_source_local(u)
            k_run = keff_values[b]
        else:
            last_local, last_counts = local, counts
        wall = time.perf_counter() - t_batch
        if on_batch is not None:
            on_batch(b, "end", eng)
        if active:
            active_wall += wall
        else:
            inactive_wall += wall

    # final canonical bank on rank 0's host: the run's only full-bank movement
    # (every batch before moved just the resampling windows)
    if world.distributed:
        g = gather_bank(world, last_local, last_counts)
        cols = [c.numpy() for c in g] if g is not None else \
            [np.empty(0, dt) for dt in BANK_DTYPES]
    else:
        cols = list(eng.bank_to_host())
    bank = FissionBank(*cols)
    act["d2h_bytes_final_bank"] = 68 * len(bank)      # after the loop: not inside the active wall
    act["ranks"] = world.size
    act["devices"] = world.size if (world.threads or world.device_backend) else 1

    keff = KeffSeries(keff_values, config.inactive_batches)
    k_mean = k_stderr = tally_mean = tally_stderr = None
    if config.active_batches >= 2:
        k_mean, k_stderr = keff.statistics()
        x = batch_sums[config.inactive_batches:, :layout.n_tally_bins] / weight
        tally_mean, tally_stderr = batch_statistics(x)
    inactive_rate = (config.inactive_batches * ppb / inactive_wall
                     if config.inactive_batches > 0 and inactive_wall > 0.0 else None)
    active_rate = (config.active_batches * ppb / active_wall
                   if config.active_batches > 0 and active_wall > 0.0 else None)
    if mesh is not None:
        mesh_mean, mesh_stderr = mesh.result(config.active_batches, weight)
    else:
        mesh_mean = mesh_stderr = None
    timings["gpu_launches"] = launches
    timings["nuclide_lookups_active"] = nuclide_lookups_active
    timings.update(act)
    return RunResult(keff=keff, k_mean=k_mean, k_stderr=k_stderr, tally_mean=tally_mean,
                     tally_stderr=tally_stderr, batch_sums=batch_sums, layout=layout, bank=bank,
                     timings=timings, inactive_wall=inactive_wall, active_wall=active_wall,
                     inactive_rate=inactive_rate, active_rate=active_rate,
                     counters=run_counters, config=config.echo(),
                     library_fingerprint=xslib.library_fingerprint(library),
                     geometry_fingerprint=pincell.fingerprint(),
                     mesh_mean=mesh_mean, mesh_stderr=mesh_stderr)


class _MeshAccumulator:
    """Per-batch mesh sums (device, float64) summed across ranks, then
    accumulated as sum and sum of squares over active batches on the device
    (torch as plumbing); mean / stderr per source particle at the end, like
    tally.batch_statistics for the dense bins."""

    def __init__(self, world: World, eng, config):
        import torch
        self.world, self.eng = world, eng
        self.shape = tuple(int(v) for v in config.mesh)[::-1] + (2,)
        ptr, n = eng.mesh_device()
        self.view = device_view(ptr, n, "float64", eng.device)
        self.sum = torch.zeros_like(self.view)
        self.sq = torch.zeros_like(self.view)

    def add_batch(self):
        import torch
        x = allreduce_tensor(self.world, self.view.clone())
        self.sum += x
        self.sq += x * x
        torch.cuda.synchronize(x.device)     # the next batch re-zeroes the buffer on the engine stream

    def result(self, n_active: int, weight: float):
        s = self.sum.cpu().numpy() / weight
        q = self.sq.cpu().numpy() / (weight * weight)
        mean = s / max(n_active, 1)
        if n_active >= 2:
            var = np.maximum(q / n_active - mean * mean, 0.0) * n_active / (n_active - 1)
            err = np.sqrt(var / n_active)
        else:
            err = np.full_like(mean, np.nan)
        return mean.reshape(self.shape), err.reshape(self.shape)


def _host_to_device_bank(eng, cols):
    """gloo runs (the multi-rank GPU parity test: several ranks sharing one
    GPU, where NCCL cannot run) exchange windows through host memory."""
    import torch
    return [c.to(torch.device("cuda", eng.device)).contiguous() for c in cols]


@dataclass
class ScalingRow:
    workers: int
    particles_per_worker: int
    inactive_rate: float
    active_rate: float
    efficiency: float


def weak_scaling_study(base_config: RunConfig, library, pincell, worker_list: list[int],
                       particles_per_worker: int, index=None) -> list[ScalingRow]:
    """particles_per_batch = W * particles_per_worker; efficiency =
    active_rate(W) / (W * active_rate(1)) (R:329-355).  Row W runs on W GPUs
    (one thread per device, run_replicated); a W larger than the visible GPU
    count would measure one GPU's throughput under a W-GPU label, so it is
    refused."""
    if not worker_list or worker_list[0] != 1 or sorted(worker_list) != list(worker_list):
        raise ConfigurationError("worker list must be ascending and start at 1")
    ndev = _device_count()
    if worker_list[-1] > ndev:
        raise ConfigurationError(f"scaling study over {worker_list[-1]} workers needs "
                                 f"{worker_list[-1]} GPUs; {ndev} visible")
    if base_config.active_batches < 1 or base_config.inactive_batches < 1:
        raise ConfigurationError("scaling study needs at least one batch in each phase")
    rows: list[ScalingRow] = []
    base_rate = None
    for w in worker_list:
        cfg = replace(base_config, workers=w, particles_per_batch=w * particles_per_worker)
        res = run_replicated(cfg, library, pincell, index=index)
        if base_rate is None:
            base_rate = res.active_rate
        rows.append(ScalingRow(w, particles_per_worker, res.inactive_rate, res.active_rate,
                               res.active_rate / (w * base_rate)))
    return rows


def warm_up() -> None:
    """Create the device context and run a miniature problem (loads the
    kernels so later timings exclude module load)."""
    from .presets import analytic_infinite_medium
    library, pincell = analytic_infinite_medium()
    for mode in ("history", "event"):
        cfg = RunConfig(particles_per_batch=8, inactive_batches=1, active_batches=2,
                        mode=mode, max_in_flight=4, accel="unionized")
        run_replicated(cfg, library, pincell)
