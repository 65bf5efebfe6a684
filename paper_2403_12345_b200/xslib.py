"""Cross-section library: data model, synthetic generator, file format and
the public lookups (device-evaluated).

Public names and behaviour follow eventmc/xslib.py (X:<line>):
  * ``NuclideXS`` / ``Material`` / ``MacroXS`` / ``UnionizedIndex`` /
    ``Library`` data model (X:55-157) with ``Library.arrays()`` giving the flat
    structure-of-arrays view (X:119-153) that the engine uploads;
  * ``generate_synthetic_library`` (X:243-271) -- bit-identical output: the
    generator draws the same LCG uniforms (vectorised here) and evaluates the
    same numpy expressions;
  * ``build_unionized_index`` / ``merge_channels`` (X:321-358) and the
    ``MCXSLIB1`` file format (X:366-431);
  * ``macro_lookup`` / ``micro_lookup`` (X:279-318) run on the GPU through
    libemc (emc_xs_lookup).  The device search is the log-hashed bracket
    search for every ``accel`` value; the reference's three backends are
    bit-equivalent by construction (X:9-19), so the requested backend only
    changes validation, never the numbers.
"""

from __future__ import annotations

import hashlib
import io
import math
import struct
from dataclasses import dataclass, field

import numpy as np

from .errors import ConfigurationError, InvalidEnergyError, UnknownMaterialError
from .prng import STRIDE, skip_ahead, uniform_sequence

EMIN = 1.0e-5
EMAX = 2.0e7

ACCEL_CODES = {"binary": 0, "double_index": 1, "unionized": 2}

_FILE_MAGIC = b"MCXSLIB1"
_FILE_VERSION = 1

_CONTROL_POINTS = 8          # channel curves are piecewise-linear in log E
_FISSILE_PROBABILITY = 0.2
_NU_FISSILE = 2.43
_NONFISSILE_CEILING = 1.0e-6


@dataclass
class NuclideXS:
    """Pointwise cross sections of one nuclide (barns vs eV)."""

    energy_grid: np.ndarray
    sigma_total: np.ndarray
    sigma_scatter: np.ndarray
    sigma_capture: np.ndarray
    sigma_fission: np.ndarray
    nu: float


@dataclass
class Material:
    """Composition: (nuclide id, atom density [atoms/(barn cm)]) pairs."""

    id: int
    composition: list[tuple[int, float]]


@dataclass
class MacroXS:
    """Macroscopic cross sections (1/cm)."""

    sigma_t: float
    sigma_s: float
    sigma_c: float
    sigma_f: float
    nu_sigma_f: float


@dataclass
class UnionizedIndex:
    """Union energy grid + per-nuclide bracket indices (+ optional merged
    bounding channel values (t0,t1,s0,s1,c0,c1,f0,f1))."""

    union_grid: np.ndarray
    index_map: np.ndarray
    merged_channels: np.ndarray | None = None


@dataclass
class Library:
    """Nuclides plus material compositions."""

    nuclides: list[NuclideXS]
    materials: list[Material]
    generation_seed: int | None = None
    _flat: tuple | None = field(default=None, repr=False, compare=False)

    @property
    def n_nuclides(self) -> int:
        return len(self.nuclides)

    @property
    def n_materials(self) -> int:
        return len(self.materials)

    @property
    def max_composition(self) -> int:
        return max((len(m.composition) for m in self.materials), default=0)

    def arrays(self) -> tuple:
        """(grid_off, grids, ch_t, ch_s, ch_c, ch_f, nu, mat_off, mat_nuc,
        mat_den, emin, emax) -- concatenated per-nuclide arrays with offsets."""
        if self._flat is None:
            lengths = np.array([n.energy_grid.shape[0] for n in self.nuclides],
                               dtype=np.int64)
            grid_off = np.concatenate(([0], np.cumsum(lengths))).astype(np.int64)

            def cat(attr):
                if not self.nuclides:
                    return np.empty(0, np.float64)
                return np.ascontiguousarray(np.concatenate(
                    [np.asarray(getattr(n, attr), np.float64) for n in self.nuclides]))

            grids, ch_t, ch_s = cat("energy_grid"), cat("sigma_total"), cat("sigma_scatter")
            ch_c, ch_f = cat("sigma_capture"), cat("sigma_fission")
            nu = np.array([n.nu for n in self.nuclides], dtype=np.float64)
            sizes = np.array([len(m.composition) for m in self.materials], np.int64)
            mat_off = np.concatenate(([0], np.cumsum(sizes))).astype(np.int64)
            mat_nuc = np.array([nid for m in self.materials for nid, _ in m.composition],
                               dtype=np.int32)
            mat_den = np.array([den for m in self.materials for _, den in m.composition],
                               dtype=np.float64)
            emin = min(float(n.energy_grid[0]) for n in self.nuclides)
            emax = max(float(n.energy_grid[-1]) for n in self.nuclides)
            self._flat = (grid_off, grids, ch_t, ch_s, ch_c, ch_f, nu, mat_off,
                          mat_nuc, mat_den, emin, emax)
        return self._flat


# ----------------------------------------------------------------- synthesis

def _channel_curve(loggrid, knots, uvals, lo, hi):
    values = lo + uvals * (hi - lo)
    return np.interp(loggrid, knots, values)


def _make_nuclide(state: int, gridpoints: int, scatter_range, capture_range,
                  fission_range, force_nonfissile: bool = False) -> NuclideXS:
    """One synthetic nuclide from its LCG stream (X:186-223 algorithm)."""
    n_jit = max(gridpoints - 2, 0)
    draws = uniform_sequence(state, n_jit + 3 * _CONTROL_POINTS + 1)
    log_lo, log_hi = math.log(EMIN), math.log(EMAX)
    if gridpoints == 1:
        grid = np.array([EMIN])
    else:
        logs = np.linspace(log_lo, log_hi, gridpoints)
        if n_jit:
            spacing = (log_hi - log_lo) / (gridpoints - 1)
            logs[1:-1] += (draws[:n_jit] - 0.5) * 0.8 * spacing
        grid = np.exp(logs)
        grid[0], grid[-1] = EMIN, EMAX
    loggrid = np.log(grid)
    knots = np.linspace(log_lo, log_hi, _CONTROL_POINTS)
    k = _CONTROL_POINTS
    scatter = _channel_curve(loggrid, knots, draws[n_jit:n_jit + k], *scatter_range)
    capture = _channel_curve(loggrid, knots, draws[n_jit + k:n_jit + 2 * k], *capture_range)
    fission = _channel_curve(loggrid, knots, draws[n_jit + 2 * k:n_jit + 3 * k], *fission_range)
    if not force_nonfissile and draws[n_jit + 3 * k] < _FISSILE_PROBABILITY:
        nu = _NU_FISSILE
    else:
        fission = fission * (_NONFISSILE_CEILING / fission.max())
        nu = 0.0
    return NuclideXS(grid, scatter + capture + fission, scatter, capture, fission, nu)


def _make_composition(state: int, n_nuclides: int, count: int, density_range,
                      id_offset: int = 0) -> list[tuple[int, float]]:
    """`count` distinct ids (partial Fisher-Yates, then ascending) with
    log-uniform densities (X:226-240 algorithm)."""
    draws = uniform_sequence(state, 2 * count)
    pool = np.arange(n_nuclides)
    for i in range(count):
        j = min(i + int(draws[i] * (n_nuclides - i)), n_nuclides - 1)
        pool[i], pool[j] = pool[j], pool[i]
    picked = np.sort(pool[:count])
    lo, hi = math.log(density_range[0]), math.log(density_range[1])
    return [(int(nid) + id_offset, math.exp(lo + draws[count + i] * (hi - lo)))
            for i, nid in enumerate(picked)]


def generate_synthetic_library(n_nuclides: int, gridpoints_per_nuclide: int,
                               n_materials: int, nuclides_per_material: int,
                               seed: int) -> Library:
    """Deterministic synthetic library (X:243-271)."""
    if min(n_nuclides, gridpoints_per_nuclide, n_materials, nuclides_per_material) < 1:
        raise ConfigurationError("library generation counts must all be >= 1")
    if nuclides_per_material > n_nuclides:
        raise ConfigurationError("nuclides_per_material cannot exceed n_nuclides")
    band = (0.1, 20.0)
    nuclides = [_make_nuclide(skip_ahead(seed, n * STRIDE), gridpoints_per_nuclide,
                              band, band, band) for n in range(n_nuclides)]
    materials = [Material(m, _make_composition(skip_ahead(seed, (n_nuclides + m) * STRIDE),
                                               n_nuclides, nuclides_per_material,
                                               (1e-4, 1e-1)))
                 for m in range(n_materials)]
    return Library(nuclides, materials, generation_seed=seed)


# --------------------------------------------------------- unionized index

def build_unionized_index(library: Library, merged: bool = False) -> UnionizedIndex:
    """Union grid + bracket map (X:321-339)."""
    if library.n_nuclides == 0:
        raise ConfigurationError("cannot unionize an empty library")
    grids = [n.energy_grid for n in library.nuclides]
    union = np.unique(np.concatenate(grids))
    index_map = np.empty((union.shape[0], len(grids)), np.int32)
    for col, g in enumerate(grids):
        idx = np.searchsorted(g, union, side="right") - 1
        index_map[:, col] = np.clip(idx, 0, max(g.shape[0] - 2, 0))
    index = UnionizedIndex(union, index_map)
    if merged:
        merge_channels(library, index)
    return index


def merge_channels(library: Library, index: UnionizedIndex) -> None:
    """Bounding channel values on the union grid (X:342-358)."""
    merged = np.empty((index.union_grid.shape[0], library.n_nuclides, 8))
    for col, nuc in enumerate(library.nuclides):
        lo = index.index_map[:, col].astype(np.int64)
        hi = np.minimum(lo + 1, nuc.energy_grid.shape[0] - 1)
        for slot, arr in enumerate((nuc.sigma_total, nuc.sigma_scatter,
                                    nuc.sigma_capture, nuc.sigma_fission)):
            merged[:, col, 2 * slot] = arr[lo]
            merged[:, col, 2 * slot + 1] = arr[hi]
    index.merged_channels = merged


def union_tuple(index: UnionizedIndex | None, accel: str) -> tuple:
    """Placeholder kept for API compatibility (X:160-172)."""
    if accel == "binary" or index is None:
        return (np.zeros(2), np.zeros((2, 1), np.int32), np.zeros((1, 1, 8)))
    merged = index.merged_channels
    if accel != "unionized" or merged is None:
        merged = np.zeros((1, 1, 8))
    return (index.union_grid, index.index_map, merged)


# ------------------------------------------------------------ file format

def _write(library: Library, fh) -> None:
    fh.write(_FILE_MAGIC)
    fh.write(struct.pack("<II", _FILE_VERSION, library.n_nuclides))
    for nuc in library.nuclides:
        fh.write(struct.pack("<Id", nuc.energy_grid.shape[0], nuc.nu))
        for arr in (nuc.energy_grid, nuc.sigma_total, nuc.sigma_scatter,
                    nuc.sigma_capture, nuc.sigma_fission):
            fh.write(np.asarray(arr).astype("<f8").tobytes())
    fh.write(struct.pack("<I", library.n_materials))
    for mat in library.materials:
        fh.write(struct.pack("<I", len(mat.composition)))
        for nid, den in mat.composition:
            fh.write(struct.pack("<Id", nid, den))


def library_bytes(library: Library) -> bytes:
    buf = io.BytesIO()
    _write(library, buf)
    return buf.getvalue()


def library_fingerprint(library: Library) -> str:
    return hashlib.sha256(library_bytes(library)).hexdigest()


def save_library(library: Library, path: str) -> None:
    with open(path, "wb") as fh:
        _write(library, fh)


def load_library(path: str) -> Library:
    with open(path, "rb") as fh:
        blob = fh.read()
    if blob[:8] != _FILE_MAGIC:
        raise ConfigurationError(f"{path}: not a library file (bad magic)")
    version, n_nuc = struct.unpack_from("<II", blob, 8)
    if version != _FILE_VERSION:
        raise ConfigurationError(f"{path}: unsupported library version {version}")
    pos = 16
    nuclides = []
    for _ in range(n_nuc):
        npts, nu = struct.unpack_from("<Id", blob, pos)
        pos += 12
        cols = []
        for _ in range(5):
            cols.append(np.frombuffer(blob, "<f8", npts, pos).astype(np.float64))
            pos += 8 * npts
        nuclides.append(NuclideXS(*cols, nu))
    (n_mat,) = struct.unpack_from("<I", blob, pos)
    pos += 4
    materials = []
    for m in range(n_mat):
        (count,) = struct.unpack_from("<I", blob, pos)
        pos += 4
        comp = []
        for _ in range(count):
            nid, den = struct.unpack_from("<Id", blob, pos)
            pos += 12
            comp.append((nid, den))
        materials.append(Material(m, comp))
    return Library(nuclides, materials, generation_seed=None)


# ------------------------------------------------------------------ lookups

def _check_energy(energy: float) -> None:
    if not math.isfinite(energy) or energy <= 0.0:
        raise InvalidEnergyError(f"invalid lookup energy {energy!r}")


def macro_lookup_batch(library: Library, material_ids, energies,
                       partials: bool = True, accel: str = "binary",
                       index: UnionizedIndex | None = None):
    """Vectorised macro_lookup on the GPU: returns (sums[n,5] =
    (t, s, c, f, nu_f), partials[n, max_comp, 4] or None).  `accel` selects
    the lookup backend (K:306-320); the union ones need `index`."""
    from .engine import api_engine
    mats = np.ascontiguousarray(material_ids, np.int32)
    ens = np.ascontiguousarray(energies, np.float64)
    if mats.shape != ens.shape or mats.ndim != 1:
        raise ConfigurationError("material_ids and energies must be 1-D and equal length")
    if mats.size and (mats.min() < 0 or mats.max() >= library.n_materials):
        raise UnknownMaterialError("material id not in library")
    if ens.size and not (np.all(np.isfinite(ens)) and np.all(ens > 0.0)):
        raise InvalidEnergyError("lookup energies must be finite and positive")
    if accel not in ACCEL_CODES:
        raise ConfigurationError(f"unknown lookup backend {accel!r}")
    if accel != "binary" and index is None:
        raise ConfigurationError(f"accel={accel!r} requires a UnionizedIndex")
    if accel == "unionized" and index.merged_channels is None:
        merge_channels(library, index)
    eng = api_engine(library=library)
    eng.set_accel(accel, index)
    try:
        return eng.xs_lookup(mats, ens, partials)
    finally:
        eng.set_accel("binary")


def macro_lookup(library: Library, material_id: int, energy: float,
                 accel: str = "binary",
                 index: UnionizedIndex | None = None) -> tuple[MacroXS, np.ndarray]:
    """Macroscopic cross sections of one material at one energy (X:292-318).
    Returns (MacroXS, partials[ncomp, 4]) with columns (t, s, c, f)."""
    _check_energy(energy)
    if material_id < 0 or material_id >= library.n_materials:
        raise UnknownMaterialError(f"material {material_id} not in library")
    if accel not in ACCEL_CODES:
        raise ConfigurationError(f"unknown lookup backend {accel!r}")
    if accel != "binary":
        if index is None:
            raise ConfigurationError(f"accel={accel!r} requires a UnionizedIndex")
        if accel == "unionized" and index.merged_channels is None:
            merge_channels(library, index)
    ncomp = len(library.materials[material_id].composition)
    sums, parts = macro_lookup_batch(library, [material_id], [energy], accel=accel, index=index)
    return MacroXS(*(float(v) for v in sums[0])), parts[0, :ncomp].copy()


def micro_lookup(nuclide: NuclideXS, energy: float) -> tuple[float, float, float, float]:
    """(total, scatter, capture, fission) of one nuclide at one energy
    (X:279-289): a unit-density single-nuclide material, whose partials are
    1.0 * sigma = sigma exactly."""
    _check_energy(energy)
    single = Library([nuclide], [Material(0, [(0, 1.0)])])
    _, parts = macro_lookup_batch(single, [0], [energy])
    t, s, c, f = (float(v) for v in parts[0, 0])
    return t, s, c, f
