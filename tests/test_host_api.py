"""Host-side API: data model, generator, file format, PRNG contracts, config
validation, statistics, resampling (reference test strategy)."""

import math

import numpy as np
import pytest

import paper_2403_12345_b200 as P
from paper_2403_12345_b200 import prng, xslib
from paper_2403_12345_b200.tally import batch_statistics, finalize

MOD = 1 << 63


# ---- library generator: bit-identical to the reference (golden fingerprints)
@pytest.mark.parametrize("name,factory", [
    ("analytic", lambda: P.analytic_infinite_medium()),
    ("small", lambda: P.depleted_pincell(12, 3, 40, 8)),
    ("c1", lambda: P.depleted_pincell(12, 3, 100, 8)),
    ("preset251", lambda: P.depleted_pincell()),
])
def test_presets_match_reference_fingerprints(golden, name, factory):
    lib, cell = factory()
    assert P.library_fingerprint(lib) == golden["problems"][name]["library_fingerprint"]
    assert cell.fingerprint() == golden["problems"][name]["geometry_fingerprint"]


def test_arrays_match_golden():
    from conftest import golden_lib_arrays
    lib, _ = P.depleted_pincell(12, 3, 40, 8)
    for a, b in zip(lib.arrays(), golden_lib_arrays("small")):
        assert np.array_equal(np.asarray(a), np.asarray(b))


def test_generation_deterministic_and_invariants():
    a = P.generate_synthetic_library(5, 30, 2, 3, seed=11)
    b = P.generate_synthetic_library(5, 30, 2, 3, seed=11)
    c = P.generate_synthetic_library(5, 30, 2, 3, seed=12)
    assert xslib.library_bytes(a) == xslib.library_bytes(b) != xslib.library_bytes(c)
    lib = P.generate_synthetic_library(10, 50, 4, 6, seed=77)
    for n in lib.nuclides:
        assert np.all(np.diff(n.energy_grid) > 0)
        assert np.array_equal(n.sigma_total, n.sigma_scatter + n.sigma_capture + n.sigma_fission)
        assert n.nu in (0.0, 2.43)
    for m in lib.materials:
        ids = [nid for nid, _ in m.composition]
        assert len(set(ids)) == 6 and ids == sorted(ids)
        assert all(1e-4 <= den <= 0.1 for _, den in m.composition)
    with pytest.raises(P.ConfigurationError):
        P.generate_synthetic_library(0, 10, 1, 1, seed=1)
    with pytest.raises(P.ConfigurationError):
        P.generate_synthetic_library(5, 10, 1, 6, seed=1)


def test_file_round_trip(tmp_path):
    lib = P.generate_synthetic_library(6, 20, 3, 4, seed=5)
    path = str(tmp_path / "lib.bin")
    P.save_library(lib, path)
    back = P.load_library(path)
    assert xslib.library_bytes(back) == xslib.library_bytes(lib)
    (tmp_path / "junk").write_bytes(b"NOTALIB!" + b"\0" * 32)
    with pytest.raises(P.ConfigurationError):
        P.load_library(str(tmp_path / "junk"))


def test_union_index_bounding_property():
    lib = P.generate_synthetic_library(6, 40, 2, 4, seed=3)
    idx = P.build_unionized_index(lib, merged=True)
    for n, nuc in enumerate(lib.nuclides):
        g = nuc.energy_grid
        for j, e in enumerate(idx.union_grid):
            i = idx.index_map[j, n]
            assert 0 <= i <= g.shape[0] - 2
            if g[0] <= e < g[-1]:
                assert g[i] <= e < g[i + 1]
    assert idx.merged_channels.shape == (idx.union_grid.shape[0], 6, 8)


# ---- PRNG contracts (reference test_prng.py)
def test_prng_kats():
    u, s = prng.next_uniform(0)
    assert s == 1 and u == 1.0 / MOD
    assert prng.next_uniform(1)[1] == (prng.MULTIPLIER + 1) % MOD
    for n in (0, 1, 2, 7, 1000, 152917):
        seq = 987654321
        for _ in range(n):
            _, seq = prng.next_uniform(seq)
        assert prng.skip_ahead(987654321, n) == seq
    rng = np.random.RandomState(3)
    for _ in range(100):
        s0 = int(rng.randint(0, 2**62))
        a, b = int(rng.randint(0, 2**40)), int(rng.randint(0, 2**40))
        assert prng.skip_ahead(prng.skip_ahead(s0, a), b) == prng.skip_ahead(s0, a + b)


def test_stream_layout():
    assert prng.seed_stream(42, 0, 1, 10) == prng.skip_ahead(prng.seed_stream(42, 0, 0, 10), prng.STRIDE)
    assert prng.seed_stream(42, 1, 0, 10) == prng.skip_ahead(42, 10 * prng.STRIDE)
    assert prng.batch_stream(42, 0) == prng.skip_ahead(42, prng.AUX_STREAM_OFFSET)


def test_uniform_sequence_matches_sequential():
    s = 2**62 + 12345
    seq = []
    for _ in range(3000):
        u, s = prng.next_uniform(s)
        seq.append(u)
    assert np.array_equal(prng.uniform_sequence(2**62 + 12345, 3000), np.array(seq))


# ---- configuration / layout / statistics
def test_config_validation():
    for kw in (dict(particles_per_batch=0), dict(mode="warp"), dict(workers=5, particles_per_batch=4),
               dict(alpha_scatter=1.5), dict(max_in_flight=0), dict(sort_every_n=0),
               dict(tally_mode="x"), dict(accel="x"), dict(reduction="x"),
               dict(fission_temperature=0.0), dict(inactive_batches=0, active_batches=0)):
        with pytest.raises(P.ConfigurationError):
            P.RunConfig(**kw).validate()
    P.RunConfig().validate()
    with pytest.raises(P.ConfigurationError):
        P.run_history(P.RunConfig(mode="event"), *P.analytic_infinite_medium())
    with pytest.raises(P.ConfigurationError):
        P.run_event(P.RunConfig(mode="history"), *P.analytic_infinite_medium())


def test_layout_and_statistics():
    lay = P.TallyLayout(n_axial=4)
    assert (lay.n_regions, lay.n_tally_bins, lay.keff_bin, lay.n_bins) == (5, 25, 25, 26)
    assert lay.region_label(4) == ("moderator", None)
    mean, err = batch_statistics(np.array([[1.0], [3.0]]))
    assert mean[0] == 2.0 and err[0] == 1.0
    x = np.random.RandomState(1).uniform(0.5, 1.5, (20, 4))
    m2, e2 = finalize(x.sum(0), (x * x).sum(0), 20)
    m1, e1 = batch_statistics(x)
    assert np.allclose(m1, m2, rtol=1e-14) and np.allclose(e1, e2, rtol=1e-9)
    with pytest.raises(P.StatisticsError):
        batch_statistics(np.ones((1, 2)))


def test_resample_formula():
    from paper_2403_12345_b200.transport import systematic_resample_indices as sri
    assert np.array_equal(sri(8, 8, 0.37), np.arange(8))
    assert np.array_equal(sri(16, 8, 0.0), np.arange(0, 16, 2))
    for u in (0.0, 0.123, 0.5, 0.99):
        assert list(sri(7, 3, u)) == [math.floor((i + u) * 7 / 3) for i in range(3)]
    assert list(sri(3, 8, 0.7)) == [0, 1, 2, 0, 1, 2, 0, 1]
    n = 10
    bank = P.FissionBank(np.arange(n, dtype=np.int64), np.zeros(n, np.int32), *[np.zeros(n)] * 6,
                         np.full(n, 1e6))
    out, st = P.resample_fission_bank(bank, 4, 123)
    assert len(out) == 4 and st == prng.skip_ahead(123, 1)
    with pytest.raises(P.PopulationCollapseError):
        P.resample_fission_bank(P.FissionBank(*[np.zeros(0)] * 9), 4, 1)


def test_geometry_host_parts():
    with pytest.raises(P.ConfigurationError):
        P.Pincell(fuel_radius=0.7, pitch=1.26)
    with pytest.raises(P.ConfigurationError):
        P.Pincell(n_axial=0)
    assert P.apply_boundary((0.6, 0.8, 0.0), "x_max") == (-0.6, 0.8, 0.0)
    with pytest.raises(ValueError):
        P.apply_boundary((1.0, 0.0, 0.0), "cylinder")
    cell = P.Pincell(n_axial=10)
    assert cell.as_tuple()[5][6] == (6 * 10.0) / 10
