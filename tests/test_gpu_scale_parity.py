"""Bit-exact parity at the benchmark's scale (BASELINE configs 3 and 4).

* grid indices: the device's log-hash + forward scan against the reference's
  `E <= lo / E >= hi / searchsorted(grid, E, 'right') - 1` (kernels.py:600-621)
  on every grid point, both neighbours of every grid point and the midpoints of
  every C4 nuclide (north_star: "grid indices ... match the reference
  bit-exactly");
* the reference's criterion-4 oracle (tests/test_acceptance.py:122-148):
  10^5 random (material, E) queries, E log-uniform on [1e-6, 3e7] (beyond both
  grid ends), sums and partials bit-identical with the oracle on the C4
  library;
* whole runs on the C3 and C4 libraries at >= 300k particles in flight, the
  production lookup (k_lookup_piped over multi-chunk sorted queues, 2 CTAs per
  SM on every SM) serving the sweeps, against the C oracle's fingerprint.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2403_12345_b200")


@pytest.fixture(scope="module")
def c4():
    return P.depleted_pincell(272, 3, 11303, 100, seed=1)


@pytest.fixture(scope="module")
def c3():
    return P.depleted_pincell(34, 3, 11303, 100, seed=1)


def _first_entry_per_nuclide(arrays):
    mat_nuc = arrays[8]
    first = {}
    for k, nid in enumerate(mat_nuc):
        first.setdefault(int(nid), k)
    return first


def _reference_bracket(grid, E):
    """(state, index) of kernels.py:600-621: clamp low, clamp high, else the
    binary search's grids[i] <= E < grids[i+1]."""
    st = np.zeros(E.shape[0], np.int32)
    idx = np.searchsorted(grid, E, side="right").astype(np.int64) - 1
    lo, hi = E <= grid[0], E >= grid[-1]
    st[lo], idx[lo] = 1, 0
    st[hi], idx[hi] = 2, grid.shape[0] - 1
    return st, idx.astype(np.int32)


def test_grid_indices_every_c4_nuclide(c4):
    from paper_2403_12345_b200.engine import api_engine
    lib, _ = c4
    arrays = lib.arrays()
    grid_off, grids = arrays[0], arrays[1]
    eng = api_engine(library=lib)
    first = _first_entry_per_nuclide(arrays)
    assert len(first) == grid_off.shape[0] - 1          # every nuclide is in some material
    checked = 0
    for nid, k in sorted(first.items()):
        g = grids[grid_off[nid]:grid_off[nid + 1]]
        mids = 0.5 * (g[:-1] + g[1:])
        E = np.concatenate([g, np.nextafter(g, 0.0), np.nextafter(g, np.inf), mids,
                            [1e-300, 1e-6, g[0] * 0.5, g[-1] * 2.0, 3e7, 1e300]])
        got = eng.grid_index(np.full(E.shape[0], k, np.int32), E)
        st, idx = _reference_bracket(g, E)
        bad = np.flatnonzero((got[:, 0] != st) | (got[:, 1] != idx))
        assert bad.size == 0, (nid, E[bad[:5]], got[bad[:5]], st[bad[:5]], idx[bad[:5]])
        checked += E.shape[0]
    assert checked > 4 * 11303 * 275


def test_criterion4_random_queries_c4_vs_oracle(c4):
    """kernels.macro_lookup_full through the public API vs the oracle's
    restatement, 10^5 queries as the reference's acceptance test draws them."""
    from oracle import driver
    lib, _ = c4
    rng = np.random.RandomState(4)
    n = 10**5
    E = np.exp(rng.uniform(np.log(1e-6), np.log(3e7), n))
    E[:16] = [lib.arrays()[10], lib.arrays()[11], 1e-6, 3e7] * 4    # emin, emax, beyond both ends
    mats = rng.randint(0, lib.n_materials, n).astype(np.int64)
    sums, parts = P.xslib.macro_lookup_batch(lib, mats, E)
    olib = driver.OracleLibrary(lib.arrays())
    for q in range(n):
        s, p = driver.macro_lookup(olib, int(mats[q]), float(E[q]))
        assert np.array_equal(sums[q], s), q
        ncomp = len(lib.materials[int(mats[q])].composition)
        assert np.array_equal(parts[q, :ncomp], p[:ncomp]), q


def _oracle_fingerprint(lib, cell, cfg):
    import os
    from oracle import driver
    ores = driver.run(dict(cfg.__dict__, mode="history"), lib.arrays(), cell.as_tuple(),
                      workers=os.cpu_count() or 1)
    return driver.fingerprint(ores), ores


_ORACLE = {}


@pytest.mark.parametrize("problem", ["c3", "c4"])
@pytest.mark.parametrize("tail_n", [None, "4096", "finish"])
def test_scale_run_matches_oracle(problem, tail_n, c3, c4, engine_env):
    """300k particles per batch, all in flight (1 inactive + 2 active batches,
    deterministic reduction): sorted sweeps of >= 262k particles go through the
    pipelined staged lookup; with EMC_TAIL_N=4096 (finish off) every sweep down
    to 4096 particles does; "finish" hands every whole batch to the
    warp-cooperative finish kernel (k_finish_warp) right after sourcing.
    Fingerprint (k series, tallies, banks, event counts) must equal the
    oracle's."""
    lib, cell = c3 if problem == "c3" else c4
    cfg = P.RunConfig(particles_per_batch=300_000, inactive_batches=1, active_batches=2,
                      mode="event", seed=42, max_in_flight=300_000, reduction="deterministic")
    if problem not in _ORACLE:
        _ORACLE[problem] = _oracle_fingerprint(lib, cell, cfg)
    want, ores = _ORACLE[problem]
    if tail_n == "finish":
        engine_env(EMC_FINISH_N=100_000_000)
    elif tail_n is not None:
        engine_env(EMC_TAIL_N=tail_n, EMC_FINISH_N=0)
    res = P.run_replicated(cfg, lib, cell)
    assert res.physics_fingerprint() == want
    for k in ("events_lookup", "events_advance", "events_collision", "fissions", "captures"):
        assert res.counters[k] == ores["counters"][k], k


@pytest.fixture(scope="module")
def c3_index(c3):
    lib, _ = c3
    return P.build_unionized_index(lib, merged=True)


def test_union_backends_criterion4_c3(c3, c3_index):
    """The reference's criterion 4 (tests/test_acceptance.py:122-148) on the
    device: 10^5 random (material, E) queries give bit-identical sums and
    partials through the three lookup backends (log-hash for "binary", union
    grid + bracket map for "double_index", + merged channels for "unionized")."""
    lib, _ = c3
    rng = np.random.RandomState(11)
    n = 10**5
    E = np.exp(rng.uniform(np.log(1e-6), np.log(3e7), n))
    E[:4] = [c3_index.union_grid[0], c3_index.union_grid[-1], c3_index.union_grid[1], c3_index.union_grid[-2]]
    mats = rng.randint(0, lib.n_materials, n)
    ref = P.xslib.macro_lookup_batch(lib, mats, E)
    for accel in ("double_index", "unionized"):
        got = P.xslib.macro_lookup_batch(lib, mats, E, accel=accel, index=c3_index)
        assert np.array_equal(got[0], ref[0]), accel
        assert np.array_equal(got[1], ref[1]), accel


@pytest.mark.parametrize("accel", ["double_index", "unionized"])
def test_union_backend_run_matches_oracle(accel, c3, c3_index):
    """Transport with the union-grid lookup kernels (k_lookup_union) on the C3
    library, 300k in flight: the oracle's (binary-search) fingerprint."""
    lib, cell = c3
    cfg = P.RunConfig(particles_per_batch=300_000, inactive_batches=1, active_batches=2,
                      mode="event", seed=42, max_in_flight=300_000, reduction="deterministic")
    if "c3" not in _ORACLE:
        _ORACLE["c3"] = _oracle_fingerprint(lib, cell, cfg)
    want, _ = _ORACLE["c3"]
    res = P.run_replicated(P.RunConfig(**dict(cfg.__dict__, accel=accel)), lib, cell, index=c3_index)
    assert res.physics_fingerprint() == want


def test_fast_tally_bins_match_deterministic():
    """The fast reduction's warp-aggregated scoring (reduce-scatter butterfly
    per region, up to three regions per warp, per-lane atomics beyond) against
    the deterministic log fold, bin by bin, on the HM core -- 100 axial fuel
    regions + moderator, so warps mix regions and every scoring branch runs.
    Batch 0 only (k_run = 1 in both modes: the same histories); atomics only
    reorder the sums: 1e-11 relative per bin."""
    lib, cell = P.hm_core(34, 3, 11303, 100, seed=1)
    res = {}
    for red in ("fast", "deterministic"):
        cfg = P.RunConfig(particles_per_batch=300_000, inactive_batches=0, active_batches=1, mode="event",
                          seed=42, max_in_flight=300_000, reduction=red)
        res[red] = P.run_replicated(cfg, lib, cell)
    a, b = np.asarray(res["fast"].batch_sums[0]), np.asarray(res["deterministic"].batch_sums[0])
    assert a.shape == b.shape and np.count_nonzero(b) > 300
    assert np.allclose(a, b, rtol=1e-11, atol=0)
    for k in ("events_lookup", "events_advance", "events_collision", "fissions", "captures"):
        assert res["fast"].counters[k] == res["deterministic"].counters[k], k


@pytest.mark.slow
def test_deterministic_log_above_int32(engine_env):
    """the deterministic contribution log passes 2^31 entries
    around 13-14M histories per rank (~160 entries per history on this
    library).  One scored 14M-particle batch: the log holds > 2^31 entries,
    is sorted with 64-bit item counts and folded; its bins equal the fast
    (atomic) sums of the same batch to 1e-9 relative (same histories: k_run =
    1 in batch 0; only the summation order differs)."""
    from paper_2403_12345_b200.engine import DeviceEngine
    lib, cell = P.depleted_pincell(12, 3, 100, 8, seed=1)
    ppb = 14_000_000
    out = {}
    for red in ("deterministic", "fast"):
        eng = DeviceEngine(0)
        try:
            eng.upload_library(lib)
            eng.upload_geometry(cell)
            cfg = P.RunConfig(particles_per_batch=ppb, inactive_batches=0, active_batches=1, mode="event",
                              seed=42, max_in_flight=ppb, reduction=red)
            eng.set_extensions(cell, cfg)
            eng.configure(cfg, 0, ppb)
            res = eng.run_batch(0, 1.0, batch0=True, score=True)
            assert res.error == 0
            out[red] = (res, eng.reduce_bins(None))
        finally:
            eng.close()
    det, fast = out["deterministic"], out["fast"]
    assert det[0].n_logs > 2**31
    assert det[0].n_sites == fast[0].n_sites
    assert np.allclose(det[1], fast[1], rtol=1e-9, atol=0)
    assert det[1][-1] > 0.0


@pytest.mark.slow
def test_hm_core_10m_batch_matches_oracle():
    """One 10M-history batch of the benchmark problem (C4 library on the HM
    core, batch 0, deterministic reduction: ~1.6e9 log entries) against the
    oracle's restatement run on all host cores: k, tallies, fission bank and
    event counts bit for bit -- the full production path (sorted pipelined
    sweeps at 10M in flight, same-material chains, tail, warp finish)."""
    import os
    from oracle import driver
    lib, cell = P.hm_core(272, 3, 11303, 100, seed=1)
    cfg = P.RunConfig(particles_per_batch=10_000_000, inactive_batches=1, active_batches=0, mode="event",
                      seed=42, max_in_flight=10_000_000, reduction="deterministic")
    res = P.run_replicated(cfg, lib, cell)
    ores = driver.run(dict(cfg.__dict__, mode="history", lattice=(cell.lattice, cell.pitch, cell.pin_map)),
                      lib.arrays(), cell.as_tuple(), workers=os.cpu_count() or 1)
    assert res.physics_fingerprint() == driver.fingerprint(ores)
    for k in ("events_lookup", "events_advance", "events_collision", "fissions", "captures", "interp_transport"):
        assert res.counters[k] == ores["counters"][k], k


@pytest.mark.slow
def test_full_size_schedule_invariance_and_bank_order():
    """Schedule invariance (the reference's acceptance criterion 1) at the
    benchmark's full size: batch 0 of C4 on the HM core at 40M particles (k_run
    = 1, so histories depend only on (seed, gid)) run with all particles in
    flight and sorted lookups, and with a 10M in-flight cap, refills and
    unsorted lookups: identical canonical fission banks and event counts; the
    bank is in canonical (parent, ordinal) order."""
    lib, cell = P.hm_core(272, 3, 11303, 100, seed=1)
    out = []
    for cap, srt in ((40_000_000, True), (10_000_000, False)):
        cfg = P.RunConfig(particles_per_batch=40_000_000, inactive_batches=1, active_batches=0, mode="event",
                          seed=42, max_in_flight=cap, sort_enabled=srt, reduction="fast")
        out.append(P.run_replicated(cfg, lib, cell))
    a, b = out
    assert a.bank.tobytes() == b.bank.tobytes()
    for k in ("events_lookup", "events_advance", "events_collision", "fissions", "captures", "interp_transport",
              "sourced", "max_draws_per_history"):
        assert a.counters[k] == b.counters[k], k
    parent, ordinal = a.bank.parent, a.bank.ordinal
    key = parent.astype(np.int64) * 64 + ordinal
    assert np.all(np.diff(key) > 0)
    assert abs(a.keff.values[0] - b.keff.values[0]) <= 1e-12 * a.keff.values[0]
