"""Benchmark problems (eventmc/presets.py:34-99), generated bit-identically.

``depleted_pincell(n_fuel, n_mod, gridpoints, n_axial, seed)`` is the
depleted-fuel pin: every fuel material holds all fuel nuclides (burnup
style) with its own densities, one fuel material per axial segment, plus a
moderator material.  SURVEY.md section 8 maps the BASELINE configs onto it:
C1 = (12, 3, 100, 8), C3 (HM-small) = (34, 3, 11303, 100),
C4 (HM-large) = (272, 3, 11303, 100).  ``analytic_infinite_medium`` has
k_inf = nu*sigma_f/(sigma_c+sigma_f) = 1.215 in closed form.

``pwr_assembly`` is BASELINE config 2 (absent from the
reference): a 2D 17x17 lattice of depleted-fuel pins with 25 water holes
(guide and instrument tube positions), ~30 synthetic nuclides, reflective.

``shielding_slab`` is BASELINE config 5 (absent from the
reference): a vacuum-bounded slab of alternating non-fissile layers (a
light scatterer and two absorber mixes) driven by a surface source on z = 0,
for fixed-source runs with a 3D mesh flux tally.
"""

from __future__ import annotations

import numpy as np

from .geometry import Pincell
from .prng import STRIDE, skip_ahead
from .xslib import Library, Material, NuclideXS, _make_composition, _make_nuclide

# shielding slab (extension): per-material channel bands, densities
SLAB_BANDS = (((3.0, 8.0), (0.05, 0.3)),      # light scatterer (scatter, capture barns)
              ((2.0, 5.0), (0.2, 1.0)),       # absorber mix A
              ((1.0, 4.0), (0.5, 2.0)))       # absorber mix B
SLAB_DENSITY = (1.0e-3, 1.0e-2)

DEFAULT_FUEL_NUCLIDES = 251
DEFAULT_MODERATOR_NUCLIDES = 3
DEFAULT_GRIDPOINTS = 100
DEFAULT_N_AXIAL = 100

# channel magnitude bands (barns) and density bands (atoms/(barn cm))
FUEL_BANDS = ((2.0, 8.0), (0.3, 2.5), (1.5, 8.0))          # scatter, capture, fission
MODERATOR_BANDS = ((3.0, 8.0), (0.1, 0.5), (0.1, 0.5))
FUEL_DENSITY = (6.0e-4, 6.0e-3)
MODERATOR_DENSITY = (3.0e-2, 9.0e-2)

ANALYTIC_K_INF = 2.43 * 0.5 / (0.5 + 0.5)


def depleted_pincell(n_fuel_nuclides: int = DEFAULT_FUEL_NUCLIDES,
                     n_moderator_nuclides: int = DEFAULT_MODERATOR_NUCLIDES,
                     gridpoints: int = DEFAULT_GRIDPOINTS,
                     n_axial: int = DEFAULT_N_AXIAL,
                     seed: int = 1) -> tuple[Library, Pincell]:
    n_total = n_fuel_nuclides + n_moderator_nuclides
    nuclides = [_make_nuclide(skip_ahead(seed, i * STRIDE), gridpoints, *FUEL_BANDS)
                for i in range(n_fuel_nuclides)]
    nuclides += [_make_nuclide(skip_ahead(seed, (n_fuel_nuclides + i) * STRIDE),
                               gridpoints, *MODERATOR_BANDS, force_nonfissile=True)
                 for i in range(n_moderator_nuclides)]
    materials = [Material(m, _make_composition(skip_ahead(seed, (n_total + m) * STRIDE),
                                               n_fuel_nuclides, n_fuel_nuclides,
                                               FUEL_DENSITY))
                 for m in range(n_axial)]
    materials.append(Material(n_axial, _make_composition(
        skip_ahead(seed, (n_total + n_axial) * STRIDE), n_moderator_nuclides,
        n_moderator_nuclides, MODERATOR_DENSITY, id_offset=n_fuel_nuclides)))
    library = Library(nuclides, materials, generation_seed=seed)
    cell = Pincell(n_axial=n_axial, fuel_material_ids=list(range(n_axial)),
                   moderator_material_id=n_axial)
    return library, cell


def analytic_infinite_medium() -> tuple[Library, Pincell]:
    """One nuclide with constant sigma_s=2, sigma_c=0.5, sigma_f=0.5 b,
    nu=2.43, filling fuel and moderator (a uniform infinite medium)."""
    grid = np.array([1.0e-5, 2.0e7])
    nuc = NuclideXS(grid, np.array([3.0, 3.0]), np.array([2.0, 2.0]),
                    np.array([0.5, 0.5]), np.array([0.5, 0.5]), 2.43)
    library = Library([nuc], [Material(0, [(0, 1.0)])])
    return library, Pincell(n_axial=1, fuel_material_ids=[0], moderator_material_id=0)


def shielding_slab(nuclides_per_material: int = 8, gridpoints: int = 2000, n_layers: int = 12,
                   width: float = 60.0, thickness: float = 60.0,
                   seed: int = 7) -> tuple[Library, Pincell]:
    """Fixed-source shielding benchmark (BASELINE config 5): three synthetic
    non-fissile materials (scatterer, two absorber mixes), ``n_layers`` layers
    of equal thickness along z cycling scatterer/A/scatterer/B, a
    ``width`` x ``width`` x ``thickness`` cm box with vacuum boundaries.
    Run it with ``RunConfig(run_mode="fixed_source", mesh=(nx, ny, nz))``."""
    nuclides, materials = [], []
    for m, (sb, cb) in enumerate(SLAB_BANDS):
        for i in range(nuclides_per_material):
            k = m * nuclides_per_material + i
            nuclides.append(_make_nuclide(skip_ahead(seed, k * STRIDE), gridpoints, sb, cb, (0.1, 0.2),
                                          force_nonfissile=True))
    n_total = len(nuclides)
    for m in range(len(SLAB_BANDS)):
        materials.append(Material(m, _make_composition(skip_ahead(seed, (n_total + m) * STRIDE),
                                                       nuclides_per_material, nuclides_per_material,
                                                       SLAB_DENSITY, id_offset=m * nuclides_per_material)))
    library = Library(nuclides, materials, generation_seed=seed)
    layers = [(0, 1, 0, 2)[j % 4] for j in range(n_layers)]
    cell = Pincell(fuel_radius=0.0, pitch=width, height=thickness, n_axial=n_layers,
                   fuel_material_ids=layers, moderator_material_id=0, boundary="vacuum")
    return library, cell


# 17x17 PWR assembly: guide-tube and central instrument-tube positions (row, column)
PWR_17_WATER_HOLES = ((2, 5), (2, 8), (2, 11), (3, 3), (3, 13), (5, 2), (5, 5), (5, 8), (5, 11), (5, 14),
                      (8, 2), (8, 5), (8, 8), (8, 11), (8, 14), (11, 2), (11, 5), (11, 8), (11, 11),
                      (11, 14), (13, 3), (13, 13), (14, 5), (14, 8), (14, 11))


def pwr_assembly(n_fuel_nuclides: int = 27, n_moderator_nuclides: int = 3, gridpoints: int = 11303,
                 n_axial: int = 1, seed: int = 1) -> tuple[Library, Pincell]:
    """BASELINE config 2: 17x17 fuel assembly (264 pins + 25 water holes) of
    the depleted_pincell materials (same generator and seeds), reflective
    outer planes; n_axial = 1 makes it 2D (reflective z planes)."""
    library, pin = depleted_pincell(n_fuel_nuclides, n_moderator_nuclides, gridpoints, n_axial, seed)
    pin_map = [1] * (17 * 17)
    for r, c in PWR_17_WATER_HOLES:
        pin_map[r * 17 + c] = 0
    cell = Pincell(fuel_radius=pin.fuel_radius, pitch=pin.pitch, height=pin.height, n_axial=n_axial,
                   fuel_material_ids=list(pin.fuel_material_ids),
                   moderator_material_id=pin.moderator_material_id, lattice=17, pin_map=pin_map)
    return library, cell


# Hoogenboom-Martin core map: 241 fuel assemblies in a 17 x 17 assembly grid
# (row lengths, centred; the 48 corner positions are water)
HM_CORE_ROWS = (7, 11, 13, 15, 15, 17, 17, 17, 17, 17, 17, 17, 15, 15, 13, 11, 7)


def hm_assembly_map(core_rows=HM_CORE_ROWS, reflector: int = 1) -> list[list[int]]:
    """Assembly grid of the core plus `reflector` rings of water assemblies:
    1 = fuel assembly, 0 = water."""
    n = len(core_rows)
    m = n + 2 * reflector
    grid = [[0] * m for _ in range(m)]
    for r, k in enumerate(core_rows):
        lo = (n - k) // 2
        for c in range(lo, lo + k):
            grid[reflector + r][reflector + c] = 1
    return grid


def hm_core(n_fuel_nuclides: int = 272, n_moderator_nuclides: int = 3, gridpoints: int = 11303,
            n_axial: int = 100, seed: int = 1, core_rows=HM_CORE_ROWS, reflector: int = 1,
            height: float = 366.0) -> tuple[Library, Pincell]:
    """Hoogenboom-Martin-style full core (BASELINE configs 3 and 4; SURVEY 8f
    row 2): 241 17x17 fuel assemblies (264 fuel pins + 25 guide/instrument
    tubes each, pitch 1.26 cm) in a 17 x 17 assembly grid with water corners,
    one ring of water-reflector assemblies, 366 cm tall with `n_axial` axial
    fuel zones (one depleted-fuel material each, the depleted_pincell
    generator and seeds), reflective outer planes.  The assembly pitch is
    exactly 17 pin pitches, so the two-level lattice (core -> assembly -> pin)
    is one global pin lattice of (17 + 2 * reflector) * 17 cells per side whose
    pin map is the assembly map expanded by the assembly's own pin map: the
    device's lattice tracking (one integer cell index per axis) serves it
    unchanged."""
    library, pin = depleted_pincell(n_fuel_nuclides, n_moderator_nuclides, gridpoints, n_axial, seed)
    amap = hm_assembly_map(core_rows, reflector)
    na = len(amap)
    n = na * 17
    apin = [1] * (17 * 17)
    for r, c in PWR_17_WATER_HOLES:
        apin[r * 17 + c] = 0
    pin_map = [0] * (n * n)
    for ar in range(na):
        for ac in range(na):
            if not amap[ar][ac]:
                continue
            for r in range(17):
                row = (ar * 17 + r) * n + ac * 17
                pin_map[row:row + 17] = apin[r * 17:(r + 1) * 17]
    cell = Pincell(fuel_radius=pin.fuel_radius, pitch=pin.pitch, height=height, n_axial=n_axial,
                   fuel_material_ids=list(pin.fuel_material_ids),
                   moderator_material_id=pin.moderator_material_id, lattice=n, pin_map=pin_map)
    return library, cell
