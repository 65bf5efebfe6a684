"""The CPU oracle (oracle/) pinned against outputs of the reference itself.

tests/golden/* were produced by running the reference (eventmc, numba) in the
build container (tests/golden/make_golden.py).  The oracle -- a C restatement
of kernels.py plus a numpy restatement of run_replicated -- must reproduce
them bit-for-bit: fingerprints, per-batch k, raw batch sums, final bank and
the schedule-invariant counters.  Only then is it trusted as the checker for
the GPU engine on inputs the goldens do not cover.
"""

import math
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden_geom, golden_lib_arrays
from oracle import driver

FAST_RUNS = ["small_history", "small_event_cap16", "small_event_naive", "small_perturb17",
             "small_seed6", "small_inact0", "small_hotsrc", "small_fast", "analytic_event_w2",
             "c1_event"]

INVARIANT = ("sourced", "captures", "fissions", "energy_clamps", "events_lookup",
             "events_advance", "events_collision", "max_draws_per_history",
             "interp_transport", "interp_score", "max_log_entries_per_history")


def _cfg(run):
    cfg = dict(max_in_flight=10000, tally_mode="fused", reduction="deterministic",
               sort_enabled=True, sort_every_n=1, workers=1, seed=42)
    cfg.update(run["config"])
    return cfg


@pytest.mark.parametrize("name", FAST_RUNS)
def test_oracle_reproduces_reference_run(golden, name):
    run = golden["runs"][name]
    res = driver.run(_cfg(run), golden_lib_arrays(run["problem"]),
                     golden_geom(golden["problems"][run["problem"]]))
    z = np.load(os.path.join(GOLDEN, f"run_{name}.npz"))
    assert np.array_equal(res["keff"], z["keff"])
    assert np.array_equal(res["batch_sums"], z["batch_sums"])
    assert driver.fingerprint(res) == run["fingerprint"]
    for k in INVARIANT:
        assert res["counters"][k] == run["counters"][k], k


def test_oracle_worker_count_invariance(golden):
    run = golden["runs"]["small_event_cap16"]
    ref = run["fingerprint"]
    for w in (2, 3, 8):
        res = driver.run(_cfg(run), golden_lib_arrays("small"), golden_geom(golden["problems"]["small"]),
                         workers=w)
        assert driver.fingerprint(res) == ref


def test_oracle_macro_lookup_matches_reference():
    z = np.load(os.path.join(GOLDEN, "lookup_small.npz"))
    olib = driver.OracleLibrary(golden_lib_arrays("small"))
    for q in range(z["mats"].shape[0]):
        sums, parts = driver.macro_lookup(olib, int(z["mats"][q]), float(z["energies"][q]))
        assert np.array_equal(sums, z["sums"][q])
        n = parts.shape[0]
        assert np.array_equal(parts, z["partials"][q][:n])


def test_oracle_geometry_matches_reference(golden):
    z = np.load(os.path.join(GOLDEN, "geometry_c1.npz"))
    og = driver.OracleGeometry(golden_geom(golden["problems"]["c1"]))
    for i in range(0, z["pts"].shape[0], 7):
        kd, ax, mat = driver.locate(og, *z["pts"][i])
        assert (kd, ax, mat) == (z["kind"][i], z["axial"][i], z["mat"][i])
        if kd >= 0:
            d, s = driver.boundary_distance(og, z["pts"][i], z["dirs"][i], kd, ax)
            assert s == z["surf"][i]
            assert d == z["dist"][i]


def test_oracle_isotropic_matches_reference():
    z = np.load(os.path.join(GOLDEN, "particle_ops.npz"))
    for i, s in enumerate(z["states"][:500]):
        u1, s1 = driver.next_uniform(int(s))
        u2, _ = driver.next_uniform(s1)
        assert driver.isotropic(u1, u2) == tuple(z["iso"][i])


def test_oracle_lcg_skip_kats():
    # reference KATs: test_prng.py:15-49, test_acceptance.py:151-161
    mult = 2806196910506780709
    assert driver.lcg_skip(0, 1) == 1
    assert driver.lcg_skip(1, 1) == (mult + 1) % (1 << 63)
    for n in (0, 1, 2, 7, 1000, 152917):
        s = seq = 42
        for _ in range(n):
            _, seq = driver.next_uniform(seq)
        assert driver.lcg_skip(s, n) == seq


def test_oracle_sort_queue_stable():
    rng = np.random.RandomState(20240811)
    n = 5000
    mats = rng.randint(0, 7, n).astype(np.int32)
    ens = rng.choice([0.5, 1.0, 2.0, 4.0], n)
    q = rng.permutation(n).astype(np.int32)
    expected = sorted(range(n), key=lambda i: (mats[q[i]], ens[q[i]], i))
    assert np.array_equal(driver.sort_queue(q, mats, ens), q[np.array(expected)])


def test_oracle_error_codes(golden):
    grid = np.array([1.0e-5, 2.0e7])
    arrays = (np.array([0, 2], np.int64), grid, np.full(2, 5.0 + 2e-13), np.full(2, 5.0),
              np.full(2, 1e-13), np.full(2, 1e-13), np.zeros(1), np.array([0, 1], np.int64),
              np.array([0], np.int32), np.array([1.0]), 1.0e-5, 2.0e7)
    geom = golden_geom(dict(n_axial=1, fuel_material_ids=[0], moderator_material_id=0))
    with pytest.raises(driver.OracleError) as e:
        driver.run(dict(particles_per_batch=1, inactive_batches=1, active_batches=0, mode="history",
                        seed=1), arrays, geom)
    assert e.value.kind == golden["errors"]["pure_scatter_history"]
    with pytest.raises(driver.OracleError) as e:
        driver.run(dict(particles_per_batch=1, inactive_batches=0, active_batches=1, mode="history",
                        seed=1), arrays, geom)
    assert e.value.kind == golden["errors"]["runaway_log"]


def test_preset251_library_fixture_matches_reference(golden):
    from conftest import golden_library
    import paper_2403_12345_b200 as P
    lib = golden_library("preset251")
    assert P.xslib.library_fingerprint(lib) == golden["problems"]["preset251"]["library_fingerprint"]
