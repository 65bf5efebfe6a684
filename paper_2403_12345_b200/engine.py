"""Python handle on one libemc device context (one GPU).

``DeviceEngine`` owns an ``emc_ctx``: it uploads a Library/Pincell, is
configured for a run (this rank's contiguous particle block), runs batches
and exposes results.  ``api_engine()`` is the per-process context used by the
single-operation API wrappers (macro_lookup, locate, ...); it re-uploads
only when a different Library / Pincell object is passed.
"""

from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import NativeUnavailableError


@dataclass
class BatchOutcome:
    counters: np.ndarray        # int64[24], kernels.py:81-103 layout
    timings: np.ndarray         # seconds: lookup, advance(+crossing), collision, sort
    n_sites: int
    n_logs: int
    iterations: int
    launches: int
    error: int
    error_gid: int
    reruns: int


class DeviceEngine:
    def __init__(self, device: int = 0, stream: int | None = None):
        self.lib = N.load_library_file()
        if N.device_count() < 1:
            raise NativeUnavailableError("no CUDA device visible to libemc (no CPU fallback)")
        h = C.c_void_p()
        N.check(self.lib.emc_create(device, C.byref(h)), "emc_create")
        self._h = h
        self.device = device
        self._keep = []
        self._src_keep = None
        self.library_obj = None
        self.pincell_obj = None
        self.union_obj = None            # UnionizedIndex on the device (set_accel)
        self.union_merged = False
        self.n_bins = 0
        self.max_comp = 0
        self.n_materials = 0
        if stream is not None:
            self.set_stream(stream)

    def close(self):
        if getattr(self, "_h", None):
            self.lib.emc_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    def set_stream(self, stream: int):
        N.check(self.lib.emc_set_stream(self._h, C.c_void_p(stream)), "emc_set_stream")

    @property
    def launch_count(self) -> int:
        return int(self.lib.emc_launch_count(self._h))

    # ------------------------------------------------------------- inputs
    def upload_library(self, library) -> None:
        (grid_off, grids, ch_t, ch_s, ch_c, ch_f, nu, mat_off, mat_nuc, mat_den,
         emin, emax) = library.arrays()
        arrs = [np.ascontiguousarray(grid_off, np.int64), np.ascontiguousarray(grids, np.float64),
                np.ascontiguousarray(ch_t, np.float64), np.ascontiguousarray(ch_s, np.float64),
                np.ascontiguousarray(ch_c, np.float64), np.ascontiguousarray(ch_f, np.float64),
                np.ascontiguousarray(nu, np.float64), np.ascontiguousarray(mat_off, np.int64),
                np.ascontiguousarray(mat_nuc, np.int32), np.ascontiguousarray(mat_den, np.float64)]
        desc = N.EmcLibrary(arrs[0].shape[0] - 1, arrs[1].shape[0], arrs[7].shape[0] - 1,
                            arrs[8].shape[0], *[N.ptr(a) for a in arrs], float(emin), float(emax))
        N.check(self.lib.emc_upload_library(self._h, C.byref(desc)), "emc_upload_library")
        self.library_obj = weakref.ref(library)
        self.union_obj = None            # the upload dropped the union index
        self.union_merged = False
        self.n_materials = arrs[7].shape[0] - 1
        self.max_comp = int(np.max(np.diff(arrs[7]))) if self.n_materials else 0

    def upload_geometry(self, pincell) -> None:
        radius, r2, hp, height, n_axial, zplanes, fuel_mats, mod_mat = pincell.as_tuple()
        zp = np.ascontiguousarray(zplanes, np.float64)
        fm = np.ascontiguousarray(fuel_mats, np.int32)
        desc = N.EmcGeometry(radius, r2, hp, height, int(n_axial), N.ptr(zp), N.ptr(fm),
                             int(mod_mat))
        N.check(self.lib.emc_upload_geometry(self._h, C.byref(desc)), "emc_upload_geometry")
        self._geometry_options(pincell)
        self.pincell_obj = weakref.ref(pincell)
        self.n_bins = (int(n_axial) + 1) * 5 + 1

    def configure(self, config, gid_lo: int, n_assigned: int) -> None:
        cfg = N.EmcRunConfig(config.particles_per_batch, gid_lo, n_assigned,
                             config.max_in_flight, int(config.mode == "history"),
                             int(config.tally_mode == "fused"),
                             int(config.reduction == "deterministic"),
                             int(bool(config.sort_enabled)), int(config.sort_every_n),
                             int(bool(getattr(config, "box_guard", False))),
                             config.seed & ((1 << 63) - 1), config.alpha_scatter,
                             config.fission_temperature, int(config.perturb_particle))
        N.check(self.lib.emc_configure(self._h, C.byref(cfg)), "emc_configure")

    def _geometry_options(self, pincell) -> None:
        """Slab / vacuum / lattice (extensions): part of
        the geometry, so every upload applies them (off for the reference's
        pincell)."""
        N.check(self.lib.emc_set_geometry_options(self._h, int(pincell.is_slab),
                                                  int(pincell.boundary == "vacuum")),
                "emc_set_geometry_options")
        n = int(getattr(pincell, "lattice", 1))
        pm = np.ascontiguousarray(pincell.pin_map if n > 1 else [1], np.int32)
        N.check(self.lib.emc_set_lattice(self._h, n, float(pincell.pitch), N.ptr(pm)), "emc_set_lattice")

    def set_extensions(self, pincell, config) -> None:
        """Geometry options, fixed source and mesh tally (extensions, SURVEY
        8f); applied on every run because engines are reused."""
        self._geometry_options(pincell)
        N.check(self.lib.emc_set_fixed_source(self._h, int(config.run_mode == "fixed_source"),
                                              float(config.source_energy)), "emc_set_fixed_source")
        nx, ny, nz = (int(v) for v in config.mesh) if config.mesh is not None else (0, 0, 0)
        N.check(self.lib.emc_set_mesh(self._h, nx, ny, nz), "emc_set_mesh")

    def mesh_device(self) -> tuple[int, int]:
        """(device pointer, length) of this batch's mesh sums (2 per cell)."""
        p, n = C.c_void_p(), C.c_int64()
        N.check(self.lib.emc_mesh_device(self._h, C.byref(p), C.byref(n)), "emc_mesh_device")
        return int(p.value or 0), int(n.value)

    # ------------------------------------------------------------ batches
    def set_source_local(self, u: float) -> None:
        N.check(self.lib.emc_set_source_local(self._h, u), "emc_set_source_local")
        self._src_keep = None

    def set_source_device(self, ptrs, n: int, u: float, keep=None, lo: int | None = None) -> None:
        """Resample the next batch from 7 device arrays (x..E): the whole
        global bank (lo None) or the window starting at global site `lo`."""
        arr = (C.c_void_p * 7)(*[C.c_void_p(int(p)) for p in ptrs])
        if lo is None:
            N.check(self.lib.emc_set_source_device(self._h, arr, n, u), "emc_set_source_device")
        else:
            N.check(self.lib.emc_set_source_window(self._h, arr, n, u, int(lo)), "emc_set_source_window")
        self._src_keep = keep

    def run_batch(self, batch: int, k_run: float, batch0: bool, score: bool) -> BatchOutcome:
        args = N.EmcBatchArgs(batch, k_run, int(batch0), int(score))
        res = N.EmcBatchResult()
        N.check(self.lib.emc_run_batch(self._h, C.byref(args), C.byref(res)), "emc_run_batch")
        return BatchOutcome(np.array(res.counters[:], np.int64), np.array(res.timings[:]),
                            res.n_sites, res.n_logs, res.iterations, res.launches, res.error,
                            res.error_gid, res.reruns)

    def reduce_bins(self, init: np.ndarray | None = None) -> np.ndarray:
        out = np.zeros(self.n_bins)
        ini = None if init is None else np.ascontiguousarray(init, np.float64)
        N.check(self.lib.emc_reduce_bins(self._h, N.ptr(ini), N.ptr(out), self.n_bins),
                "emc_reduce_bins")
        return out

    def bank_size(self) -> int:
        n = C.c_int64(0)
        N.check(self.lib.emc_bank_size(self._h, C.byref(n)), "emc_bank_size")
        return n.value

    def bank_device_ptrs(self) -> list[int]:
        arr = (C.c_void_p * 9)()
        N.check(self.lib.emc_bank_device(self._h, arr), "emc_bank_device")
        return [int(p or 0) for p in arr]

    def bank_to_host(self, start: int = 0, n: int | None = None) -> tuple:
        if n is None:
            n = self.bank_size() - start
        cols = [np.empty(n, np.int64), np.empty(n, np.int32)] + [np.empty(n) for _ in range(7)]
        N.check(self.lib.emc_bank_copy(self._h, start, n, *[N.ptr(c) for c in cols]),
                "emc_bank_copy")
        return tuple(cols)

    # ------------------------------------------------------- API operations
    def xs_lookup(self, mats: np.ndarray, ens: np.ndarray, partials: bool = True):
        n = mats.shape[0]
        sums = np.zeros((n, 5))
        mc = max(self.max_comp, 1)
        parts = np.zeros((n, mc, 4)) if partials else None
        N.check(self.lib.emc_xs_lookup(self._h, n, N.ptr(mats), N.ptr(ens), N.ptr(sums),
                                       N.ptr(parts), mc), "emc_xs_lookup")
        if parts is not None and self.max_comp == 0:
            parts = parts[:, :0]
        return sums, parts

    ACCEL_CODES = {"binary": 0, "double_index": 1, "unionized": 2}

    def set_accel(self, accel: str, index=None) -> None:
        """Lookup backend (kernels.py ACCEL_*): "binary" = the device's log-hash
        search; "double_index" / "unionized" = the union grid of `index`
        (uploaded once per index object), merged channels for "unionized"."""
        code = self.ACCEL_CODES[accel]
        if code and (self.union_obj is None or self.union_obj() is not index or
                     (code == 2 and not self.union_merged)):
            ug = np.ascontiguousarray(index.union_grid, np.float64)
            mp = np.ascontiguousarray(index.index_map, np.int32)
            mg = None
            if code == 2:
                mg = np.ascontiguousarray(index.merged_channels, np.float64)
            N.check(self.lib.emc_upload_union(self._h, N.ptr(ug), ug.shape[0], N.ptr(mp),
                                              N.ptr(mg) if mg is not None else None), "emc_upload_union")
            self.union_obj = weakref.ref(index)
            self.union_merged = mg is not None
        N.check(self.lib.emc_set_accel(self._h, code), "emc_set_accel")

    def grid_index(self, entries: np.ndarray, ens: np.ndarray) -> np.ndarray:
        """[n, 2] (clamp state, bracket index) of composition entries at E."""
        entries = np.ascontiguousarray(entries, np.int32)
        ens = np.ascontiguousarray(ens, np.float64)
        out = np.zeros((entries.shape[0], 2), np.int32)
        N.check(self.lib.emc_grid_index(self._h, entries.shape[0], N.ptr(entries), N.ptr(ens), N.ptr(out)),
                "emc_grid_index")
        return out

    def locate(self, pos: np.ndarray) -> np.ndarray:
        out = np.zeros((pos.shape[0], 3), np.int32)
        N.check(self.lib.emc_locate(self._h, pos.shape[0], N.ptr(pos), N.ptr(out)), "emc_locate")
        return out

    def distance(self, pos, dirs, cells):
        pos = np.ascontiguousarray(pos, np.float64)
        dirs = np.ascontiguousarray(dirs, np.float64)
        cells = np.ascontiguousarray(cells, np.int32)
        n = pos.shape[0]
        dist = np.zeros(n)
        surf = np.zeros(n, np.int32)
        N.check(self.lib.emc_distance(self._h, n, N.ptr(pos), N.ptr(dirs), N.ptr(cells),
                                      N.ptr(dist), N.ptr(surf)), "emc_distance")
        return dist, surf

    def particle_ops(self, states: np.ndarray, sigma_t: np.ndarray):
        states = np.ascontiguousarray(states, np.uint64)
        sigma_t = np.ascontiguousarray(sigma_t, np.float64)
        n = states.shape[0]
        iso = np.zeros((n, 3))
        dcol = np.zeros(n)
        s1 = np.zeros(n, np.uint64)
        s2 = np.zeros(n, np.uint64)
        N.check(self.lib.emc_particle_ops(self._h, n, N.ptr(states), N.ptr(sigma_t), N.ptr(iso),
                                          N.ptr(dcol), N.ptr(s1), N.ptr(s2)), "emc_particle_ops")
        return iso, dcol, s1, s2

    def sort_queue(self, q: np.ndarray, mats: np.ndarray, ens: np.ndarray) -> np.ndarray:
        q = np.ascontiguousarray(q, np.int32)
        mats = np.ascontiguousarray(mats, np.int32)
        ens = np.ascontiguousarray(ens, np.float64)
        out = np.zeros_like(q)
        N.check(self.lib.emc_sort_queue(self._h, q.shape[0], N.ptr(q), mats.shape[0], N.ptr(mats),
                                        N.ptr(ens), N.ptr(out)), "emc_sort_queue")
        return out

    def replay_bins(self, binidx: np.ndarray, vals: np.ndarray, n_bins: int) -> np.ndarray:
        out = np.zeros(n_bins)
        N.check(self.lib.emc_replay_bins(self._h, binidx.shape[0], N.ptr(binidx), N.ptr(vals),
                                         n_bins, N.ptr(out)), "emc_replay_bins")
        return out

    def lcg_skip(self, states: np.ndarray, ks: np.ndarray) -> np.ndarray:
        states = np.ascontiguousarray(states, np.uint64)
        ks = np.ascontiguousarray(ks, np.uint64)
        out = np.zeros_like(states)
        N.check(self.lib.emc_lcg_skip(self._h, states.shape[0], N.ptr(states), N.ptr(ks),
                                      N.ptr(out)), "emc_lcg_skip")
        return out

    def libm(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float64)
        out = np.zeros((x.shape[0], 3))
        N.check(self.lib.emc_libm_eval(self._h, x.shape[0], N.ptr(x), N.ptr(out)), "emc_libm_eval")
        return out

    def div(self, num: np.ndarray, den: np.ndarray) -> np.ndarray:
        """[n, 2]: staged-lookup division (precomputed reciprocal) and IEEE n/d."""
        num = np.ascontiguousarray(num, np.float64)
        den = np.ascontiguousarray(den, np.float64)
        out = np.zeros((num.shape[0], 2))
        N.check(self.lib.emc_div_eval(self._h, num.shape[0], N.ptr(num), N.ptr(den), N.ptr(out)), "emc_div_eval")
        return out


_API: DeviceEngine | None = None


def api_engine(library=None, pincell=None) -> DeviceEngine:
    """Process-wide context for the single-operation API wrappers."""
    global _API
    if _API is None:
        _API = DeviceEngine(0)
    if library is not None and (_API.library_obj is None or _API.library_obj() is not library):
        _API.upload_library(library)
    if pincell is not None and (_API.pincell_obj is None or _API.pincell_obj() is not pincell):
        _API.upload_geometry(pincell)
    return _API
