"""CPU oracle for the SURVEY 8f row-1 extension (fixed-source shielding slab,
vacuum boundaries, 3D track-length mesh tallies).  The reference has no such
features, so parity for them is pinned against this restatement (GPU side:
tests/test_gpu_extensions.py) plus size-independent properties checked here:
neutron balance with leakage, mesh totals equal to the region totals, and an
eigenvalue run with a mesh switched on still reproducing the reference's
fingerprint (scoring a mesh consumes no random numbers)."""

import os

import numpy as np
import pytest

from conftest import GOLDEN, golden_geom, golden_lib_arrays
from oracle import driver

P = pytest.importorskip("paper_2403_12345_b200")


def _slab_run(mode="event", n=1500, mesh=(3, 5, 12), **kw):
    lib, cell = P.shielding_slab(gridpoints=150)
    cfg = dict(particles_per_batch=n, inactive_batches=0, active_batches=2, mode=mode,
               run_mode="fixed_source", mesh=mesh, slab=True, vacuum=True, reduction="deterministic",
               max_in_flight=400, **kw)
    return driver.run(cfg, lib.arrays(), cell.as_tuple()), cell


@pytest.mark.parametrize("mode", ["event", "history"])
def test_slab_balance_and_mesh_totals(mode):
    res, cell = _slab_run(mode)
    c = res["counters"]
    assert c["sourced"] == 2 * 1500
    assert c["captures"] + c["fissions"] + c["leaks"] == c["sourced"]
    assert c["leaks"] > 0 and c["fissions"] == 0
    # every flight segment is scored once by its region and once across the mesh
    region_flux = res["batch_sums"][:, 0:5 * cell.n_axial:5].sum()
    region_tot = res["batch_sums"][:, 1:5 * cell.n_axial:5].sum()
    assert np.isclose(res["mesh_sum"][..., 0].sum(), region_flux, rtol=1e-12, atol=0)
    assert np.isclose(res["mesh_sum"][..., 1].sum(), region_tot, rtol=1e-12, atol=0)
    # attenuation: flux falls through the slab
    prof = res["mesh_mean"][..., 0].sum(axis=(1, 2))
    assert prof[0] > prof[len(prof) // 2] > prof[-1] >= 0.0


def test_slab_history_equals_event():
    a, _ = _slab_run("event")
    b, _ = _slab_run("history")
    assert driver.fingerprint(a) == driver.fingerprint(b)
    assert np.allclose(a["mesh_sum"], b["mesh_sum"], rtol=1e-12, atol=1e-300)


def test_slab_fixed_energy_source():
    res, _ = _slab_run(source_energy=2.0e6, n=500)
    assert res["counters"]["energy_clamps"] == 0
    assert res["counters"]["sourced"] == 1000


def test_mesh_does_not_perturb_eigenvalue_histories(golden):
    """C1 golden run with a mesh tally on: same fingerprint as the reference."""
    run = golden["runs"]["c1_event"]
    pm = golden["problems"]["c1"]
    cfg = dict(run["config"], mesh=(4, 4, 8))
    res = driver.run(cfg, golden_lib_arrays("c1"), golden_geom(pm))
    assert driver.fingerprint(res) == run["fingerprint"]
    act = run["config"]["inactive_batches"]
    region_flux = res["batch_sums"][act:, 0:5 * (pm["n_axial"] + 1):5].sum()
    assert np.isclose(res["mesh_sum"][..., 0].sum(), region_flux, rtol=1e-11, atol=0)


def test_vacuum_pincell_leaks_and_balances(golden):
    pm = golden["problems"]["small"]
    cfg = dict(particles_per_batch=3000, inactive_batches=1, active_batches=2, mode="event",
               vacuum=True, reduction="deterministic")
    res = driver.run(cfg, golden_lib_arrays("small"), golden_geom(pm))
    c = res["counters"]
    assert c["leaks"] > 0
    assert c["captures"] + c["fissions"] + c["leaks"] == c["sourced"]


# ---- lattice extension (BASELINE config 2) -------------------

def _lattice_cfg(cell, **kw):
    return dict(kw, lattice=(cell.lattice, cell.pitch, cell.pin_map))


def test_full_lattice_equals_infinite_pincell_statistically():
    """An all-pin reflective lattice is the same infinite medium as one
    reflective pincell: k agrees within statistics (the histories differ)."""
    lib, pin = P.depleted_pincell(12, 3, 100, 1, seed=1)
    lat = P.Pincell(fuel_radius=pin.fuel_radius, pitch=pin.pitch, height=pin.height, n_axial=1,
                    fuel_material_ids=pin.fuel_material_ids,
                    moderator_material_id=pin.moderator_material_id, lattice=5)
    base = dict(particles_per_batch=20000, inactive_batches=3, active_batches=10, mode="event",
                reduction="fast", workers=8)
    a = driver.run(dict(base), lib.arrays(), pin.as_tuple())
    b = driver.run(_lattice_cfg(lat, **base), lib.arrays(), lat.as_tuple())
    ka, kb = a["keff"][3:], b["keff"][3:]
    se = np.sqrt(ka.var(ddof=1) / ka.size + kb.var(ddof=1) / kb.size)
    assert abs(ka.mean() - kb.mean()) < 4.0 * se, (ka.mean(), kb.mean(), se)


def test_assembly_mesh_is_pinwise_and_balanced():
    lib, cell = P.pwr_assembly(gridpoints=200)
    cfg = _lattice_cfg(cell, particles_per_batch=4000, inactive_batches=1, active_batches=2,
                       mode="history", mesh=(17, 17, 1), reduction="deterministic")
    res = driver.run(cfg, lib.arrays(), cell.as_tuple())
    c = res["counters"]
    assert c["captures"] + c["fissions"] == c["sourced"]
    flux = res["batch_sums"][1:, 0:10:5].sum()
    assert np.isclose(res["mesh_sum"][..., 0].sum(), flux, rtol=1e-12, atol=0)
    ev = driver.run(dict(cfg, mode="event"), lib.arrays(), cell.as_tuple())
    assert driver.fingerprint(ev) == driver.fingerprint(res)       # executor-invariant


def test_hm_core_layout():
    """presets.hm_core: 241 fuel assemblies of the 17x17 pin map in a 17x17
    assembly grid with water corners, a one-assembly water reflector, one
    global pin lattice; a one-assembly core without reflector is exactly
    the pwr_assembly lattice."""
    import paper_2403_12345_b200 as P
    lib, cell = P.hm_core(12, 3, 100, 4)
    assert cell.lattice == 19 * 17
    assert sum(cell.pin_map) == 241 * 264
    assert abs(cell.half_width - 19 * 17 * 1.26 / 2) < 1e-12
    amap = P.presets.hm_assembly_map()
    assert sum(map(sum, amap)) == 241 and amap[0] == [0] * 19
    pm = np.asarray(cell.pin_map).reshape(cell.lattice, cell.lattice)
    assert (pm == pm[::-1]).all() and (pm == pm[:, ::-1]).all() and (pm == pm.T).all()
    _, one = P.hm_core(12, 3, 100, 1, core_rows=(1,), reflector=0)
    _, asm = P.pwr_assembly(12, 3, 100, 1)
    assert one.lattice == 17 and list(one.pin_map) == list(asm.pin_map)


def test_hm_core_oracle_runs_balanced():
    """The oracle transports a small HM core (lattice restatement) with exact
    neutron balance (checked per batch inside driver.run)."""
    import paper_2403_12345_b200 as P
    lib, cell = P.hm_core(12, 3, 100, 4, core_rows=(1, 3, 1), height=40.0)
    cfg = dict(particles_per_batch=500, inactive_batches=1, active_batches=1, mode="history",
               seed=3, lattice=(cell.lattice, cell.pitch, cell.pin_map))
    res = driver.run(cfg, lib.arrays(), cell.as_tuple())
    assert res["counters"]["sourced"] == 1000
    assert 0.0 < res["keff"][1] < 2.0
