"""CPU ORACLE driver -- test infrastructure only (see oracle/emc_oracle.c).

Restates the reference's per-batch coordinator ``run_replicated``
(/root/reference/pkg/src/eventmc/replication.py:155-315, cited R:<line>) in
numpy around the C restatement of the kernels.  Used by tests/ as the parity
checker, by __graft_entry__.smoke() and by bench.py's ``cpu_baseline`` /
``--impl reference`` legs.  The product package never imports this module.

Inputs are plain arrays so the oracle does not depend on the product's
objects: ``lib`` is the 12-tuple of ``Library.arrays()`` (xslib.py:119-153)
and ``geom`` the 8-tuple of ``Pincell.as_tuple()`` (geometry.py:83-90).
"""

from __future__ import annotations

import ctypes as C
import hashlib
import os
import subprocess
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

N_COUNTERS = 24
CNT = dict(LOG_N=0, SITE_N=1, OVF=2, ERR=3, ERR_AUX=4, CAPTURES=5, FISSIONS=6,
           SOURCED=7, MAX_DRAWS=8, CLAMPS=9, INTERP_TRANSPORT=10,
           INTERP_SCORE=11, EV_LOOKUP=12, EV_ADVANCE=13, EV_COLLISION=14,
           INV_LOOKUP=15, INV_ADVANCE=16, INV_COLLISION=17, SORTS=18,
           MAX_INFLIGHT=19, MAX_HIST_LOG=20)
COUNTER_SUMS = (("captures", 5), ("fissions", 6), ("sourced", 7),
                ("energy_clamps", 9), ("interp_transport", 10),
                ("interp_score", 11), ("events_lookup", 12),
                ("events_advance", 13), ("events_collision", 14),
                ("invocations_lookup", 15), ("invocations_advance", 16),
                ("invocations_collision", 17), ("sorts", 18))
COUNTER_MAXES = (("max_draws_per_history", 8),
                 ("max_log_entries_per_history", 20),
                 ("max_in_flight_observed", 19))
ERRORS = {1: ("GeometryError", "no boundary intersection"),
          2: ("GeometryError", "particle outside the cell box"),
          3: ("StreamOverlapError", "history consumed a full RNG stride"),
          4: ("RunawayHistoryError", "history exceeded the contribution-log cap"),
          5: ("EventMCError", "event queue invariant violated"),
          6: ("PhysicsError", "sigma_t <= 0 (void materials unsupported)")}

P = C.c_void_p


class OLib(C.Structure):
    _fields_ = [("grid_off", P), ("grids", P), ("ch_t", P), ("ch_s", P),
                ("ch_c", P), ("ch_f", P), ("nu", P), ("mat_off", P),
                ("mat_nuc", P), ("mat_den", P), ("emin", C.c_double),
                ("emax", C.c_double)]


class OGeom(C.Structure):
    _fields_ = [("radius", C.c_double), ("r2", C.c_double), ("hp", C.c_double),
                ("height", C.c_double), ("n_axial", C.c_int64),
                ("zplanes", P), ("fuel_mats", P), ("mod_mat", C.c_int64),
                # extensions: slab, vacuum, mesh
                ("slab", C.c_int32), ("vacuum", C.c_int32), ("mesh", P),
                ("mnx", C.c_int32), ("mny", C.c_int32), ("mnz", C.c_int32), ("mpad", C.c_int32),
                ("mx0", C.c_double), ("my0", C.c_double), ("mz0", C.c_double),
                ("mdx", C.c_double), ("mdy", C.c_double), ("mdz", C.c_double),
                ("lat_n", C.c_int32), ("n_pins", C.c_int32), ("pitch", C.c_double),
                ("pin_map", P), ("pin_xy", P),
                # box guard extension (RunConfig.box_guard; include/emc.h)
                ("guard", C.c_int32), ("gpad", C.c_int32)]


class OSlots(C.Structure):
    _fields_ = [(n, P) for n in ("px", "py", "pz", "dx", "dy", "dz", "en", "wt",
                                 "rng", "draws", "gid", "ordctr", "histlog",
                                 "kind", "axial", "mat", "cm_t", "cm_s", "cm_c",
                                 "cm_f", "cm_nsf", "part_t")] + \
        [("nslots", C.c_int64), ("part_cols", C.c_int64)]


class OLog(C.Structure):
    _fields_ = [("gid", P), ("ord", P), ("bin", P), ("val", P), ("cap", C.c_int64)]


class OSites(C.Structure):
    _fields_ = [(n, P) for n in ("parent", "ord", "x", "y", "z", "dx", "dy",
                                 "dz", "E")] + [("cap", C.c_int64)]


class OSrc(C.Structure):
    _fields_ = [(n, P) for n in ("x", "y", "z", "dx", "dy", "dz", "E")]


class OParams(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("batch", C.c_int64), ("pmax", C.c_int64),
                ("alpha", C.c_double), ("fission_t", C.c_double),
                ("k_run", C.c_double), ("fused", C.c_int32),
                ("score", C.c_int32), ("use_logs", C.c_int32),
                ("sort_enabled", C.c_int32), ("sort_every", C.c_int32),
                ("batch0", C.c_int32), ("history", C.c_int32),
                ("perturb_gid", C.c_int64),
                ("fixed_source", C.c_int32), ("pad", C.c_int32), ("src_energy", C.c_double)]


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc, no FMA contraction, glibc libm)."""
    src = os.path.join(HERE, "emc_oracle.c")
    if force or not os.path.exists(LIB_PATH) or \
            os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math",
                        "-fPIC", "-shared", src, "-o", LIB_PATH, "-lm"],
                       check=True)
    return LIB_PATH


_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        build()
        L = C.CDLL(LIB_PATH)
        L.oracle_run_batch.restype = None
        L.oracle_lcg_skip.restype = C.c_uint64
        L.oracle_lcg_skip.argtypes = [C.c_uint64, C.c_uint64]
        L.oracle_boundary_distance.restype = C.c_double
        L.oracle_boundary_distance.argtypes = [C.c_double] * 6 + [
            C.c_int64, C.c_int64, P, P]
        L.oracle_locate.argtypes = [C.c_double] * 3 + [P, P]
        L.oracle_isotropic.argtypes = [C.c_double, C.c_double, P]
        L.oracle_macro_lookup.argtypes = [P, C.c_int64, C.c_double, P, P]
        L.oracle_replay_into_bins.argtypes = [P, P, P, C.c_int64]
        L.oracle_sort_queue.argtypes = [P, C.c_int64, P, P]
        _LIB = L
    return _LIB


def _p(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


class OracleLibrary:
    """Keeps the numpy arrays alive behind the OLib struct."""

    def __init__(self, arrays):
        (grid_off, grids, ch_t, ch_s, ch_c, ch_f, nu, mat_off, mat_nuc,
         mat_den, emin, emax) = arrays
        self.keep = [np.ascontiguousarray(grid_off, np.int64),
                     np.ascontiguousarray(grids, np.float64),
                     np.ascontiguousarray(ch_t, np.float64),
                     np.ascontiguousarray(ch_s, np.float64),
                     np.ascontiguousarray(ch_c, np.float64),
                     np.ascontiguousarray(ch_f, np.float64),
                     np.ascontiguousarray(nu, np.float64),
                     np.ascontiguousarray(mat_off, np.int64),
                     np.ascontiguousarray(mat_nuc, np.int32),
                     np.ascontiguousarray(mat_den, np.float64)]
        self.s = OLib(*[_p(a) for a in self.keep], float(emin), float(emax))
        mo = self.keep[7]
        self.n_materials = mo.shape[0] - 1
        self.max_comp = int(np.max(np.diff(mo))) if mo.shape[0] > 1 else 0


class OracleGeometry:
    """``geom`` = Pincell.as_tuple(); ``slab``/``vacuum`` and ``mesh``
    (nx, ny, nz) are the extensions of SURVEY 8f row 1 (off by default).
    With a mesh, ``self.mesh`` is this geometry's accumulator (one per worker:
    see OracleGeometry.for_worker)."""

    def __init__(self, geom, slab=False, vacuum=False, mesh=None, lattice=None, guard=False):
        radius, r2, hp, height, n_axial, zplanes, fuel_mats, mod_mat = geom
        self.args = (geom, slab, vacuum, mesh, lattice, guard)
        self.keep = [np.ascontiguousarray(zplanes, np.float64),
                     np.ascontiguousarray(fuel_mats, np.int32)]
        self.n_axial = int(n_axial)
        hp, height = float(hp), float(height)
        if mesh is not None:
            nx, ny, nz = (int(v) for v in mesh)
            self.mesh = np.zeros(2 * nx * ny * nz)
            mptr, dims = _p(self.mesh), (nx, ny, nz, 0)
            box = (-hp, -hp, 0.0, (2.0 * hp) / nx, (2.0 * hp) / ny, height / nz)
        else:
            self.mesh, mptr, dims, box = None, None, (0, 0, 0, 0), (0.0,) * 6
        lat = (1, 0, 0.0, None, None)
        if lattice is not None and int(lattice[0]) > 1:     # (n, pitch, pin_map)
            n, pitch, pmap = int(lattice[0]), float(lattice[1]), np.asarray(lattice[2], np.int32)
            xy = [(-hp + (i + 0.5) * pitch, -hp + (j + 0.5) * pitch)
                  for j in range(n) for i in range(n) if pmap[j * n + i]]
            self.keep += [np.ascontiguousarray((pmap != 0).astype(np.int32)),
                          np.ascontiguousarray(np.array(xy, np.float64).ravel())]
            lat = (n, len(xy), pitch, _p(self.keep[2]), _p(self.keep[3]))
        self.s = OGeom(float(radius), float(r2), hp, height,
                       int(n_axial), _p(self.keep[0]), _p(self.keep[1]),
                       int(mod_mat), int(bool(slab)), int(bool(vacuum)), mptr, *dims, *box, *lat,
                       int(bool(guard)), 0)

    def for_worker(self):
        return OracleGeometry(*self.args) if self.mesh is not None else self


# ---- single-op wrappers (parity checks of the device ops) -------------------

def lcg_skip(state: int, n: int) -> int:
    return int(lib().oracle_lcg_skip(state, n))


def macro_lookup(olib: OracleLibrary, m: int, energy: float):
    sums = np.zeros(5)
    parts = np.zeros((max(olib.max_comp, 1), 4))
    lib().oracle_macro_lookup(C.byref(olib.s), m, energy, _p(sums), _p(parts))
    return sums, parts


def locate(ogeom: OracleGeometry, x, y, z):
    out = np.zeros(3, np.int64)
    lib().oracle_locate(x, y, z, C.byref(ogeom.s), _p(out))
    return tuple(int(v) for v in out)


def boundary_distance(ogeom: OracleGeometry, pos, d, kind, axial):
    surf = np.zeros(1, np.int64)
    dist = lib().oracle_boundary_distance(*map(float, pos), *map(float, d),
                                          int(kind), int(axial),
                                          C.byref(ogeom.s), _p(surf))
    return dist, int(surf[0])


def isotropic(u1, u2):
    out = np.zeros(3)
    lib().oracle_isotropic(u1, u2, _p(out))
    return tuple(out)


def sort_queue(q, mats, ens):
    q = np.array(q, np.int32, copy=True)
    lib().oracle_sort_queue(_p(q), q.shape[0],
                            _p(np.ascontiguousarray(mats, np.int32)),
                            _p(np.ascontiguousarray(ens, np.float64)))
    return q


# ---- worker state (R:62-111) ------------------------------------------------

class _Worker:
    def __init__(self, assigned, cfg, max_comp, n_bins):
        n_assigned = assigned.shape[0]
        nslots = max(1, min(cfg["max_in_flight"], n_assigned)) \
            if cfg["mode"] == "event" else 1
        self.assigned = np.ascontiguousarray(assigned, np.int64)
        part_cols = max(max_comp if cfg["tally_mode"] == "fused" else 1, 1)
        f64 = lambda: np.zeros(nslots)  # noqa: E731
        self.arr = dict(px=f64(), py=f64(), pz=f64(), dx=f64(), dy=f64(),
                        dz=f64(), en=f64(), wt=np.ones(nslots),
                        rng=np.zeros(nslots, np.uint64),
                        draws=np.zeros(nslots, np.int64),
                        gid=np.zeros(nslots, np.int64),
                        ordctr=np.zeros(nslots, np.int32),
                        histlog=np.zeros(nslots, np.int32),
                        kind=np.zeros(nslots, np.int8),
                        axial=np.zeros(nslots, np.int32),
                        mat=np.zeros(nslots, np.int32),
                        cm_t=f64(), cm_s=f64(), cm_c=f64(), cm_f=f64(),
                        cm_nsf=f64(),
                        part_t=np.zeros((nslots, part_cols)))
        self.slots = OSlots(*[_p(self.arr[f[0]]) for f in OSlots._fields_[:22]],
                            nslots, part_cols)
        self._alloc_logs(n_assigned * 96 + 4096)
        self._alloc_sites(n_assigned * 6 + 1024)
        self.wbins = np.zeros(n_bins)
        self.counters = np.zeros(N_COUNTERS, np.int64)
        self.timings = np.zeros(4)

    def _alloc_logs(self, cap):
        self.logs = (np.zeros(cap, np.int64), np.zeros(cap, np.int32),
                     np.zeros(cap, np.int32), np.zeros(cap))
        self.log_s = OLog(*[_p(a) for a in self.logs], cap)

    def _alloc_sites(self, cap):
        self.sites = tuple(np.zeros(cap, dt) for dt in
                           (np.int64, np.int32) + (np.float64,) * 7)
        self.site_s = OSites(*[_p(a) for a in self.sites], cap)

    def grow_for(self, ovf):
        if ovf == 1:
            self._alloc_logs(2 * self.logs[0].shape[0])
        else:
            self._alloc_sites(2 * self.sites[0].shape[0])


def _run_worker(w: _Worker, olib, ogeom, src_s, params: OParams, n_bins):
    while True:  # R:122-142 grow-and-rerun on overflow
        w.counters[:] = 0
        w.timings[:] = 0.0
        w.wbins[:] = 0.0
        if ogeom.mesh is not None:
            ogeom.mesh[:] = 0.0
        lib().oracle_run_batch(_p(w.assigned), C.c_int64(w.assigned.shape[0]),
                               C.byref(w.slots), C.byref(olib.s),
                               C.byref(ogeom.s), C.byref(src_s),
                               C.byref(w.log_s), C.byref(w.site_s),
                               _p(w.wbins), C.c_int32(n_bins),
                               _p(w.counters), _p(w.timings), C.byref(params))
        ovf = int(w.counters[CNT["OVF"]])
        if ovf == 0:
            return
        w.grow_for(ovf)


# ---- prng helpers (prng.py:37-87) ---------------------------------------------

MASK63 = (1 << 63) - 1
MULT = 2806196910506780709


def next_uniform(state: int):
    s = (MULT * state + 1) & MASK63
    u = s * 2.0 ** -63
    if u >= 1.0:
        u = 1.0 - 2.0 ** -53
    return u, s


def batch_stream(seed: int, b: int) -> int:
    return lcg_skip(seed & MASK63, (1 << 62) + b * 152917)


def systematic_resample_indices(n_bank, target, u):  # transport.py:188-200
    if n_bank >= target:
        idx = np.floor((np.arange(target, dtype=np.float64) + u)
                       * n_bank / target).astype(np.int64)
        np.clip(idx, 0, n_bank - 1, out=idx)
    else:
        idx = np.arange(target, dtype=np.int64) % n_bank
    return idx


class OracleError(Exception):
    def __init__(self, kind, msg):
        super().__init__(msg)
        self.kind = kind


DEFAULTS = dict(max_in_flight=10000, tally_mode="fused", reduction="deterministic",
                sort_enabled=True, sort_every_n=1, workers=1, seed=42, alpha_scatter=0.5,
                fission_temperature=1.3e6, perturb_particle=-1, mode="event")


def run(cfg: dict, lib_arrays, geom, workers: int | None = None,
        batches: range | None = None) -> dict:
    """Restatement of run_replicated (R:155-315).  ``cfg`` holds the RunConfig
    fields by name (missing ones take RunConfig's defaults, T:30-45).
    Returns keff values, batch sums, final bank, counters, timings and the
    active/inactive rates."""
    cfg = dict(DEFAULTS, **cfg)
    olib = OracleLibrary(lib_arrays)
    mesh = cfg.get("mesh")
    ogeom = OracleGeometry(geom, slab=cfg.get("slab", False), vacuum=cfg.get("vacuum", False),
                           mesh=mesh, lattice=cfg.get("lattice"), guard=cfg.get("box_guard", False))
    fixed = cfg.get("run_mode", "eigenvalue") == "fixed_source"
    ppb = int(cfg["particles_per_batch"])
    n_axial = ogeom.n_axial
    n_tally = (n_axial + 1) * 5
    n_bins = n_tally + 1
    use_logs = cfg.get("reduction", "deterministic") == "deterministic"
    weight = float(ppb)
    nw = int(workers if workers is not None else cfg.get("workers", 1))
    ws = [_Worker(np.arange(w, ppb, nw, dtype=np.int64), cfg, olib.max_comp,
                  n_bins) for w in range(nw)]
    wgeom = [ogeom.for_worker() for _ in ws]
    mesh_sum = mesh_sq = None
    if mesh is not None:
        mesh_sum, mesh_sq = np.zeros_like(ogeom.mesh), np.zeros_like(ogeom.mesh)
    n_batches = int(cfg["inactive_batches"]) + int(cfg["active_batches"])
    n_inactive = int(cfg["inactive_batches"])
    batch_sums = np.zeros((n_batches, n_bins))
    keff = np.zeros(n_batches)
    run_counters: dict = {}
    timings = dict(lookup=0.0, advance=0.0, collision=0.0, sort=0.0,
                   reduce=0.0, merge=0.0)
    inactive_wall = active_wall = 0.0
    k_run = 1.0
    src_arrays = [np.zeros(1) for _ in range(7)]
    bank = None
    pool = ThreadPoolExecutor(max_workers=nw) if nw > 1 else None
    seed = int(cfg.get("seed", 42))
    try:
        for b in (batches if batches is not None else range(n_batches)):
            active = b >= n_inactive
            t_batch = time.perf_counter()
            src_s = OSrc(*[_p(a) for a in src_arrays])
            params = OParams(seed & MASK63, b, ppb,
                             float(cfg.get("alpha_scatter", 0.5)),
                             float(cfg.get("fission_temperature", 1.3e6)),
                             k_run,
                             int(cfg.get("tally_mode", "fused") == "fused"),
                             int(active), int(use_logs),
                             int(cfg.get("sort_enabled", True)),
                             int(cfg.get("sort_every_n", 1)), int(b == 0),
                             int(cfg["mode"] == "history"),
                             int(cfg.get("perturb_particle", -1)),
                             int(fixed), 0, float(cfg.get("source_energy", 0.0)))
            if pool is not None:
                futs = [pool.submit(_run_worker, w, olib, g, src_s, params,
                                    n_bins) for w, g in zip(ws, wgeom)]
                for f in futs:
                    f.result()
            else:
                _run_worker(ws[0], olib, wgeom[0], src_s, params, n_bins)
            if mesh is not None and active:
                mb = np.zeros_like(mesh_sum)
                for g in wgeom:
                    mb += g.mesh
                mesh_sum += mb
                mesh_sq += mb * mb
            for w in ws:
                err = int(w.counters[CNT["ERR"]])
                if err:
                    kind, msg = ERRORS[err]
                    raise OracleError(kind, f"{msg} (batch {b}, particle "
                                      f"{int(w.counters[CNT['ERR_AUX']])})")
            t0 = time.perf_counter()
            ns = [int(w.counters[CNT["SITE_N"]]) for w in ws]
            cat = [np.concatenate([w.sites[k][:n] for w, n in zip(ws, ns)])
                   for k in range(9)]
            perm = np.lexsort((cat[1], cat[0]))
            bank = [a[perm] for a in cat]
            timings["merge"] += time.perf_counter() - t0
            t0 = time.perf_counter()
            sums = np.zeros(n_bins)
            if use_logs:
                n_l = [int(w.counters[CNT["LOG_N"]]) for w in ws]
                gid = np.concatenate([w.logs[0][:n] for w, n in zip(ws, n_l)])
                binidx = np.concatenate([w.logs[2][:n] for w, n in zip(ws, n_l)])
                vals = np.concatenate([w.logs[3][:n] for w, n in zip(ws, n_l)])
                if gid.shape[0]:
                    perm = np.argsort(gid, kind="stable")
                    bi = np.ascontiguousarray(binidx[perm])
                    vv = np.ascontiguousarray(vals[perm])
                    lib().oracle_replay_into_bins(_p(sums), _p(bi), _p(vv),
                                                  bi.shape[0])
            else:
                for w in ws:
                    sums += w.wbins
            timings["reduce"] += time.perf_counter() - t0
            batch_sums[b] = sums
            keff[b] = sums[n_tally] / weight
            sourced = sum(int(w.counters[CNT["SOURCED"]]) for w in ws)
            deaths = sum(int(w.counters[5]) + int(w.counters[6]) + int(w.counters[22]) for w in ws)
            if sourced != ppb or deaths != ppb:
                raise OracleError("EventMCError", "neutron bookkeeping broken")
            for name, idx in COUNTER_SUMS + ((("leaks", 22),) if cfg.get("vacuum") else ()) + \
                    ((("box_guard", 23),) if cfg.get("box_guard") else ()):
                run_counters[name] = run_counters.get(name, 0) + sum(
                    int(w.counters[idx]) for w in ws)
            for name, idx in COUNTER_MAXES:
                run_counters[name] = max(run_counters.get(name, 0),
                                         max(int(w.counters[idx]) for w in ws))
            for key, ti in (("lookup", 0), ("advance", 1), ("collision", 2),
                            ("sort", 3)):
                timings[key] += sum(float(w.timings[ti]) for w in ws)
            if b < n_batches - 1 and fixed:
                pass                                # fixed source: sampled afresh every batch
            elif b < n_batches - 1:
                if bank[0].shape[0] == 0:
                    raise OracleError("PopulationCollapseError",
                                      f"no fission sites banked in batch {b}")
                u, _ = next_uniform(batch_stream(seed, b))
                idx = systematic_resample_indices(bank[0].shape[0], ppb, u)
                src_arrays = [np.ascontiguousarray(bank[k][idx])
                              for k in range(2, 9)]
                k_run = keff[b]
            wall = time.perf_counter() - t_batch
            if active:
                active_wall += wall
            else:
                inactive_wall += wall
    finally:
        if pool is not None:
            pool.shutdown(wait=False)
    n_active = n_batches - n_inactive
    mesh_out = {}
    if mesh is not None:
        nx, ny, nz = (int(v) for v in mesh)
        mean = mesh_sum / weight / max(n_active, 1)
        mesh_out = dict(mesh_mean=mean.reshape(nz, ny, nx, 2),
                        mesh_sum=mesh_sum.reshape(nz, ny, nx, 2),
                        mesh_sq=mesh_sq.reshape(nz, ny, nx, 2))
    return dict(keff=keff, batch_sums=batch_sums, bank=bank, **mesh_out,
                counters=run_counters, timings=timings,
                inactive_wall=inactive_wall, active_wall=active_wall,
                active_rate=(n_active * ppb / active_wall
                             if n_active and active_wall > 0 else None),
                inactive_rate=(n_inactive * ppb / inactive_wall
                               if n_inactive and inactive_wall > 0 else None))


def fingerprint(res: dict) -> str:
    """RunResult.physics_fingerprint (transport.py:147-153)."""
    h = hashlib.sha256()
    h.update(res["keff"].tobytes())
    h.update(res["batch_sums"].tobytes())
    h.update(b"".join(a.tobytes() for a in res["bank"]))
    return h.hexdigest()
