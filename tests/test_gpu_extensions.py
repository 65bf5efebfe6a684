"""GPU parity for the SURVEY 8f row-1 extension (fixed-source shielding slab,
vacuum boundaries, 3D track-length mesh tallies) against the oracle's
restatement of the same extension (the reference has none of these:
parity is pinned to oracle/, see tests/test_oracle_extensions.py)."""

import numpy as np
import pytest

from conftest import golden_library
from oracle import driver

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2403_12345_b200")


def _oracle(cfg, lib, cell):
    return driver.run(dict(cfg.__dict__, slab=cell.is_slab, vacuum=cell.boundary == "vacuum"),
                      lib.arrays(), cell.as_tuple())


@pytest.mark.parametrize("mode,energy", [("event", 0.0), ("history", 0.0), ("event", 2.0e6)])
def test_slab_fixed_source_matches_oracle(mode, energy):
    lib, cell = P.shielding_slab(gridpoints=150)
    cfg = P.RunConfig(particles_per_batch=1500, inactive_batches=0, active_batches=3, mode=mode,
                      run_mode="fixed_source", source_energy=energy, mesh=(3, 5, 12),
                      reduction="deterministic", max_in_flight=400)
    res = P.run_replicated(cfg, lib, cell)
    ores = _oracle(cfg, lib, cell)
    assert res.physics_fingerprint() == driver.fingerprint(ores)
    for k in ("sourced", "captures", "fissions", "leaks", "events_lookup", "events_collision",
              "max_draws_per_history", "interp_transport"):
        assert res.counters[k] == ores["counters"][k], k
    # atomics only reorder the per-cell sums of bit-identical segment scores
    assert np.allclose(res.mesh_mean, ores["mesh_mean"], rtol=1e-12, atol=0)
    assert res.mesh_stderr.shape == res.mesh_mean.shape


def test_slab_large_population_fast_reduction():
    lib, cell = P.shielding_slab()
    cfg = P.RunConfig(particles_per_batch=200_000, inactive_batches=0, active_batches=2,
                      run_mode="fixed_source", mesh=(20, 20, 60), reduction="fast",
                      max_in_flight=200_000)
    res = P.run_replicated(cfg, lib, cell)
    ores = _oracle(cfg, lib, cell)
    for k in ("sourced", "captures", "leaks", "events_lookup", "events_collision"):
        assert res.counters[k] == ores["counters"][k], k
    assert np.allclose(res.batch_sums, ores["batch_sums"], rtol=1e-10, atol=0)
    assert np.allclose(res.mesh_mean, ores["mesh_mean"], rtol=1e-10, atol=1e-300)
    flux = res.batch_sums[:, 0:5 * cell.n_axial:5].sum() / cfg.particles_per_batch / 2
    assert np.isclose(res.mesh_mean[..., 0].sum(), flux, rtol=1e-10)


def test_mesh_on_eigenvalue_run_keeps_reference_fingerprint(golden):
    run = golden["runs"]["c1_event"]
    pm = golden["problems"]["c1"]
    cell = P.Pincell(n_axial=pm["n_axial"], fuel_material_ids=pm["fuel_material_ids"],
                     moderator_material_id=pm["moderator_material_id"])
    cfg = P.RunConfig(**dict(run["config"], mesh=(4, 4, 8)))
    res = P.run_replicated(cfg, golden_library("c1"), cell)
    assert res.physics_fingerprint() == run["fingerprint"]
    act = cfg.inactive_batches
    flux = res.batch_sums[act:, 0:5 * (pm["n_axial"] + 1):5].sum() / cfg.particles_per_batch
    assert np.isclose(res.mesh_mean[..., 0].sum() * cfg.active_batches, flux, rtol=1e-11)


def test_vacuum_pincell_eigenvalue_matches_oracle(golden):
    pm = golden["problems"]["small"]
    cell = P.Pincell(n_axial=pm["n_axial"], fuel_material_ids=pm["fuel_material_ids"],
                     moderator_material_id=pm["moderator_material_id"], boundary="vacuum")
    lib = golden_library("small")
    cfg = P.RunConfig(particles_per_batch=3000, inactive_batches=1, active_batches=2, mode="event",
                      reduction="deterministic", max_in_flight=700)
    res = P.run_replicated(cfg, lib, cell)
    ores = _oracle(cfg, lib, cell)
    assert res.physics_fingerprint() == driver.fingerprint(ores)
    assert res.counters["leaks"] == ores["counters"]["leaks"] > 0


@pytest.mark.parametrize("mode", ["event", "history"])
def test_pwr_assembly_lattice_matches_oracle(mode):
    """BASELINE config 2 geometry (17x17 lattice with water holes, SURVEY 8f
    row 2) at parity scale: histories bit-identical to the oracle."""
    lib, cell = P.pwr_assembly(gridpoints=300)
    cfg = P.RunConfig(particles_per_batch=4000, inactive_batches=1, active_batches=2, mode=mode,
                      reduction="deterministic", max_in_flight=1500, mesh=(17, 17, 1))
    res = P.run_replicated(cfg, lib, cell)
    ores = driver.run(dict(cfg.__dict__, lattice=(cell.lattice, cell.pitch, cell.pin_map)),
                      lib.arrays(), cell.as_tuple())
    assert res.physics_fingerprint() == driver.fingerprint(ores)
    for k in ("sourced", "captures", "fissions", "events_lookup", "events_collision", "interp_transport"):
        assert res.counters[k] == ores["counters"][k], k
    assert np.allclose(res.mesh_mean, ores["mesh_mean"], rtol=1e-12, atol=0)


@pytest.mark.parametrize("mode", ["event", "history"])
def test_hm_core_small_matches_oracle(mode):
    """Hoogenboom-Martin-style core (presets.hm_core: assemblies of the 17x17
    pin map in a core map with water corners and a water reflector ring) on a
    5-assembly core, 10 axial zones: histories bit-identical to the oracle."""
    lib, cell = P.hm_core(20, 3, 400, 10, core_rows=(1, 3, 1), reflector=1, height=60.0)
    cfg = P.RunConfig(particles_per_batch=4000, inactive_batches=1, active_batches=2, mode=mode,
                      reduction="deterministic", max_in_flight=1500)
    res = P.run_replicated(cfg, lib, cell)
    ores = driver.run(dict(cfg.__dict__, lattice=(cell.lattice, cell.pitch, cell.pin_map)),
                      lib.arrays(), cell.as_tuple())
    assert res.physics_fingerprint() == driver.fingerprint(ores)
    for k in ("sourced", "captures", "fissions", "events_lookup", "events_collision", "interp_transport"):
        assert res.counters[k] == ores["counters"][k], k


@pytest.mark.parametrize("nfuel", [34, 272])
def test_hm_core_full_size_matches_oracle(nfuel):
    """The full HM core (241 assemblies, 323 x 323 pin cells, 366 cm, 100 axial
    zones) with the C3 / C4 libraries (34 / 272 fuel nuclides, 11,303-point
    grids) at 200k particles in flight: the production path (sorted sweeps
    through the pipelined staged lookup, then the tail kernels) against the
    oracle, bit for bit."""
    import os
    lib, cell = P.hm_core(nfuel, 3, 11303, 100)
    cfg = P.RunConfig(particles_per_batch=200_000, inactive_batches=1, active_batches=1, mode="event",
                      reduction="deterministic", max_in_flight=200_000, seed=42)
    res = P.run_replicated(cfg, lib, cell)
    ores = driver.run(dict(cfg.__dict__, mode="history", lattice=(cell.lattice, cell.pitch, cell.pin_map)),
                      lib.arrays(), cell.as_tuple(), workers=os.cpu_count() or 1)
    assert res.physics_fingerprint() == driver.fingerprint(ores)
    for k in ("events_lookup", "events_advance", "events_collision", "fissions", "captures"):
        assert res.counters[k] == ores["counters"][k], k


def test_pwr_assembly_c2_scale_staged_equals_plain():
    """C2 at 1M particles: the staged lookup and the plain kernel agree bit
    for bit on the lattice problem (27-nuclide fuel group: staged path)."""
    import os
    lib, cell = P.pwr_assembly()
    cfg = P.RunConfig(particles_per_batch=1_000_000, inactive_batches=1, active_batches=1,
                      reduction="deterministic", max_in_flight=1_000_000)
    out = {}
    for kern in ("staged", "plain"):
        os.environ["EMC_LOOKUP"] = kern
        try:
            out[kern] = P.run_replicated(cfg, lib, cell).physics_fingerprint()
        finally:
            os.environ.pop("EMC_LOOKUP", None)
    assert out["staged"] == out["plain"]


def _edge_library():
    """A 20-nuclide fuel group that drives every path of the staged lookup:
    a 1-point nuclide (point window), a 2-point nuclide, a nuclide whose grid
    leaves the guard-free division range (IEEE-division fallback for the whole
    nuclide), exact duplicate energies across nuclides, and long/short grids
    (staged windows and over-wide windows that fall back to the global path)."""
    rng = np.random.default_rng(5)
    nucs = []

    def nuc(grid, fiss):
        g = np.asarray(grid, np.float64)
        n = g.shape[0]
        s = rng.uniform(2.0, 8.0, n)
        c = rng.uniform(0.3, 2.5, n)
        f = rng.uniform(1.5, 8.0, n) if fiss else np.full(n, 1e-7)
        return P.NuclideXS(g, s + c + f, s, c, f, 2.43 if fiss else 0.0)

    nucs.append(nuc([1.0e-5], True))                                  # glen 1
    nucs.append(nuc([1.0e-5, 2.0e7], False))                          # glen 2
    nucs.append(nuc([1.0e-70, 1.0e-69, 1.0, 2.0e7], False))           # outside the safe range
    shared = np.exp(np.linspace(np.log(1e-5), np.log(2e7), 400))
    for k in range(17):
        if k % 5 == 0:
            g = shared.copy()                                          # identical grids
        else:
            npts = int(rng.integers(20, 3000))
            g = np.sort(np.exp(rng.uniform(np.log(1e-5), np.log(2e7), npts)))
            g[0], g[-1] = 1e-5, 2e7
            g = np.unique(g)
        nucs.append(nuc(g, k % 3 == 0))
    mod = [nuc(np.exp(np.linspace(np.log(1e-5), np.log(2e7), 100)), False) for _ in range(3)]
    nucs += mod
    dens = rng.uniform(6e-4, 6e-3, 20)
    mats = [P.Material(m, [(i, float(dens[i] * (1 + 0.1 * m))) for i in range(20)]) for m in range(2)]
    mats.append(P.Material(2, [(20 + i, 0.05) for i in range(3)]))
    lib = P.Library(nucs, mats)
    cell = P.Pincell(n_axial=2, fuel_material_ids=[0, 1], moderator_material_id=2)
    return lib, cell


@pytest.mark.parametrize("cap,tail_n", [(3000, 0), (3000, None), (256, 0), (256, None), (3000, "finish")])
def test_edge_library_staged_paths_match_oracle(cap, tail_n, engine_env):
    """tail_n=0 disables tail mode and the finish, so every sweep is sorted and
    goes through the staged kernels (with cap = ppb the default thresholds
    would hand the whole run to the finish / tail kernels); "finish" runs every
    batch through k_finish_warp."""
    if tail_n == "finish":
        engine_env(EMC_FINISH_N=100_000_000)
    elif tail_n is not None:
        engine_env(EMC_TAIL_N=tail_n, EMC_FINISH_N=0)
    lib, cell = _edge_library()
    cfg = P.RunConfig(particles_per_batch=3000, inactive_batches=2, active_batches=2, mode="event",
                      reduction="deterministic", max_in_flight=cap)
    res = P.run_replicated(cfg, lib, cell)
    ores = driver.run(dict(cfg.__dict__), lib.arrays(), cell.as_tuple())
    assert res.physics_fingerprint() == driver.fingerprint(ores)
    assert res.counters["interp_transport"] == ores["counters"]["interp_transport"]


@pytest.mark.parametrize("which", ["lattice", "slab", "pincell_vacuum"])
def test_extension_geometry_ops_match_oracle(which):
    """Cell search and distance-to-boundary of the extension geometries on the
    device (public API) against the oracle, bit for bit, on random points and
    directions, including points near lattice planes and pin surfaces."""
    from paper_2403_12345_b200.engine import api_engine
    if which == "lattice":
        _, cell = P.pwr_assembly(gridpoints=50)
        og = driver.OracleGeometry(cell.as_tuple(), lattice=(cell.lattice, cell.pitch, cell.pin_map))
    elif which == "slab":
        _, cell = P.shielding_slab(gridpoints=50)
        og = driver.OracleGeometry(cell.as_tuple(), slab=True, vacuum=True)
    else:
        cell = P.Pincell(n_axial=4, fuel_material_ids=[0, 0, 0, 0], moderator_material_id=0, boundary="vacuum")
        og = driver.OracleGeometry(cell.as_tuple(), vacuum=True)
    rng = np.random.default_rng(17)
    n = 6000
    hp, h = cell.half_width, cell.height
    pts = np.stack([rng.uniform(-hp, hp, n), rng.uniform(-hp, hp, n), rng.uniform(0, h, n)], 1)
    if which == "lattice":      # cluster a third of the points on cell planes and pin surfaces
        k = n // 3
        i = rng.integers(0, cell.lattice, k)
        pts[:k, 0] = -hp + i * cell.pitch + rng.normal(0, 1e-9, k)
        ang = rng.uniform(0, 2 * np.pi, k)
        pts[k:2 * k, 0] = -hp + (rng.integers(0, 17, k) + 0.5) * cell.pitch + cell.fuel_radius * np.cos(ang)
        pts[k:2 * k, 1] = -hp + (rng.integers(0, 17, k) + 0.5) * cell.pitch + cell.fuel_radius * np.sin(ang)
    mu = rng.uniform(-1, 1, n)
    phi = rng.uniform(0, 2 * np.pi, n)
    dirs = np.stack([np.sqrt(1 - mu * mu) * np.cos(phi), np.sqrt(1 - mu * mu) * np.sin(phi), mu], 1)
    loc = P.geometry.locate_batch(cell, pts)
    want = np.array([driver.locate(og, *p) for p in pts])
    assert np.array_equal(loc, want)
    inside = loc[:, 0] >= 0
    cells = loc[inside][:, :2].astype(np.int32)
    dist, surf = api_engine(pincell=cell).distance(pts[inside], dirs[inside], cells)
    for j, (p, d, c) in enumerate(zip(pts[inside], dirs[inside], cells)):
        od, osf = driver.boundary_distance(og, p, d, int(c[0]), int(c[1]))
        assert (dist[j], surf[j]) == (od, osf), (j, p, d, c)
