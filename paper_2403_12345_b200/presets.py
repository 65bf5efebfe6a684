"""Benchmark problems (eventmc/presets.py:34-99), generated bit-identically.

``depleted_pincell(n_fuel, n_mod, gridpoints, n_axial, seed)`` is the
depleted-fuel pin: every fuel material holds all fuel nuclides (burnup
style) with its own densities, one fuel material per axial segment, plus a
moderator material.  SURVEY.md section 8 maps the BASELINE configs onto it:
C1 = (12, 3, 100, 8), C3 (HM-small) = (34, 3, 11303, 100),
C4 (HM-large) = (272, 3, 11303, 100).  ``analytic_infinite_medium`` has
k_inf = nu*sigma_f/(sigma_c+sigma_f) = 1.215 in closed form.
"""

from __future__ import annotations

import numpy as np

from .geometry import Pincell
from .prng import STRIDE, skip_ahead
from .xslib import Library, Material, NuclideXS, _make_composition, _make_nuclide

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
