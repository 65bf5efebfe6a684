"""Generate the golden fixtures by running the REFERENCE (eventmc) in this container.

This script is the provenance of everything under tests/golden/.  It imports
the reference package from /root/reference/pkg/src (read-only; numba cache
redirected to /tmp) and records, for a set of small parity configurations:

  * the library fingerprint and the flat library arrays (npz, small libs only),
  * per-batch k values, raw batch sums, the final canonical fission bank,
    the run counters and RunResult.physics_fingerprint(),
  * macro_lookup results (sums + partials) on seeded random queries,
  * boundary_distance / locate results on seeded random rays,
  * a few transcendental-dependent particle ops (sample_isotropic,
    sample_collision_distance) on seeded states.

Nothing in tests/, bench.py or the package reads /root/reference at run time;
only the committed outputs of this script are used.

Run:  NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
from dataclasses import replace

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")

import eventmc  # noqa: E402
from eventmc import geometry, presets, transport, xslib  # noqa: E402
from eventmc.replication import run_replicated  # noqa: E402
from eventmc.transport import RunConfig  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def _hex(x: float) -> str:
    return float(x).hex()


def lib_arrays(lib) -> dict:
    (grid_off, grids, ch_t, ch_s, ch_c, ch_f, nu, mat_off, mat_nuc, mat_den,
     emin, emax) = lib.arrays()
    return dict(grid_off=grid_off, grids=grids, ch_t=ch_t, ch_s=ch_s,
                ch_c=ch_c, ch_f=ch_f, nu=nu, mat_off=mat_off,
                mat_nuc=mat_nuc, mat_den=mat_den,
                emin=np.float64(emin), emax=np.float64(emax))


PROBLEMS = {
    "analytic": lambda: presets.analytic_infinite_medium(),
    "small": lambda: presets.depleted_pincell(12, 3, 40, 8),
    "c1": lambda: presets.depleted_pincell(12, 3, 100, 8),
    "preset251": lambda: presets.depleted_pincell(),
}

# (name, problem, RunConfig kwargs, save bank rows)
RUNS = [
    ("analytic_event_w2", "analytic",
     dict(particles_per_batch=20000, inactive_batches=5, active_batches=20,
          mode="event", seed=42, workers=2)),
    ("small_history", "small",
     dict(particles_per_batch=400, inactive_batches=2, active_batches=3,
          mode="history", seed=5)),
    ("small_event_cap16", "small",
     dict(particles_per_batch=400, inactive_batches=2, active_batches=3,
          mode="event", seed=5, max_in_flight=16)),
    ("small_event_naive", "small",
     dict(particles_per_batch=400, inactive_batches=2, active_batches=3,
          mode="event", seed=5, max_in_flight=64, tally_mode="naive")),
    ("small_perturb17", "small",
     dict(particles_per_batch=400, inactive_batches=2, active_batches=3,
          mode="history", seed=5, perturb_particle=17)),
    ("small_seed6", "small",
     dict(particles_per_batch=400, inactive_batches=2, active_batches=3,
          mode="history", seed=6)),
    ("small_inact0", "small",
     dict(particles_per_batch=400, inactive_batches=0, active_batches=6,
          mode="history", seed=5)),
    ("small_fast", "small",
     dict(particles_per_batch=400, inactive_batches=2, active_batches=3,
          mode="event", seed=5, reduction="fast")),
    ("small_hotsrc", "small",
     dict(particles_per_batch=300, inactive_batches=1, active_batches=2,
          mode="event", seed=2, fission_temperature=1.0e8)),
    ("c1_event", "c1",
     dict(particles_per_batch=10000, inactive_batches=10, active_batches=10,
          mode="event", seed=42)),
    ("preset251_event_w2", "preset251",
     dict(particles_per_batch=10000, inactive_batches=5, active_batches=5,
          mode="event", seed=42, workers=2)),
]


def run_one(name, prob, kwargs, problems):
    lib, cell = problems[prob]
    cfg = RunConfig(**kwargs)
    res = run_replicated(cfg, lib, cell)
    bank = res.bank
    rec = {
        "problem": prob,
        "config": kwargs,
        "fingerprint": res.physics_fingerprint(),
        "keff": [_hex(v) for v in res.keff.values],
        "k_mean": None if res.k_mean is None else _hex(res.k_mean),
        "k_stderr": None if res.k_stderr is None else _hex(res.k_stderr),
        "counters": {k: int(v) for k, v in res.counters.items()},
        "bank_len": len(bank),
        "bank_sha256": hashlib.sha256(bank.tobytes()).hexdigest(),
        "batch_sums_sha256": hashlib.sha256(res.batch_sums.tobytes()).hexdigest(),
        "library_fingerprint": res.library_fingerprint,
        "geometry_fingerprint": res.geometry_fingerprint,
    }
    np.savez_compressed(
        os.path.join(OUT, f"run_{name}.npz"),
        keff=res.keff.values, batch_sums=res.batch_sums,
        bank_parent=bank.parent, bank_ordinal=bank.ordinal,
        bank_x=bank.x, bank_y=bank.y, bank_z=bank.z,
        bank_dx=bank.dx, bank_dy=bank.dy, bank_dz=bank.dz,
        bank_energy=bank.energy)
    return rec


def main():
    eventmc.warm_up()
    problems = {k: f() for k, f in PROBLEMS.items()}
    meta = {"generator": "tests/golden/make_golden.py",
            "reference": "eventmc 0.1.0 (/root/reference/pkg)",
            "numpy": np.__version__,
            "problems": {}, "runs": {}, "errors": {}}
    import numba
    meta["numba"] = numba.__version__
    for k, (lib, cell) in problems.items():
        meta["problems"][k] = {
            "library_fingerprint": xslib.library_fingerprint(lib),
            "geometry_fingerprint": cell.fingerprint(),
            "n_axial": cell.n_axial,
            "fuel_material_ids": list(map(int, cell.fuel_material_ids)),
            "moderator_material_id": int(cell.moderator_material_id),
        }
        if k != "preset251":
            np.savez_compressed(os.path.join(OUT, f"lib_{k}.npz"),
                                **lib_arrays(lib))
    for name, prob, kwargs in RUNS:
        print("run", name, flush=True)
        meta["runs"][name] = run_one(name, prob, kwargs, problems)
        print("   ", meta["runs"][name]["fingerprint"], flush=True)

    # error-path goldens (exception class names)
    def uniform_medium(ss, sc, sf, nu):
        grid = np.array([1.0e-5, 2.0e7])
        nuc = xslib.NuclideXS(grid, np.full(2, ss + sc + sf), np.full(2, ss),
                              np.full(2, sc), np.full(2, sf), nu)
        return xslib.Library([nuc], [xslib.Material(0, [(0, 1.0)])])
    cell = presets.analytic_infinite_medium()[1]
    for name, lib, cfg in [
        ("pure_scatter_history",
         uniform_medium(5.0, 1e-13, 1e-13, 0.0),
         RunConfig(particles_per_batch=1, inactive_batches=1, active_batches=0,
                   mode="history", seed=1)),
        ("runaway_log",
         uniform_medium(5.0, 1e-13, 1e-13, 0.0),
         RunConfig(particles_per_batch=1, inactive_batches=0, active_batches=1,
                   mode="history", seed=1)),
    ]:
        try:
            run_replicated(cfg, lib, cell)
            meta["errors"][name] = None
        except Exception as e:  # noqa: BLE001
            meta["errors"][name] = type(e).__name__

    # macro lookups on the small library
    rng = np.random.RandomState(20240811)
    lib, cell = problems["small"]
    n = 2000
    energies = np.exp(rng.uniform(np.log(1e-6), np.log(3e7), n))
    mats = rng.randint(0, lib.n_materials, n)
    sums = np.zeros((n, 5))
    parts = np.zeros((n, lib.max_composition, 4))
    for q in range(n):
        mx, p = xslib.macro_lookup(lib, int(mats[q]), float(energies[q]))
        sums[q] = (mx.sigma_t, mx.sigma_s, mx.sigma_c, mx.sigma_f, mx.nu_sigma_f)
        parts[q, :p.shape[0]] = p
    np.savez_compressed(os.path.join(OUT, "lookup_small.npz"), mats=mats,
                        energies=energies, sums=sums, partials=parts)

    # geometry: random rays in the C1 pincell
    lib, cell = problems["c1"]
    m = 5000
    hp = cell.pitch / 2
    pts = np.stack([rng.uniform(-hp, hp, m), rng.uniform(-hp, hp, m),
                    rng.uniform(0, cell.height, m)], axis=1)
    mu = rng.uniform(-1, 1, m)
    phi = rng.uniform(0, 2 * np.pi, m)
    s = np.sqrt(1 - mu * mu)
    dirs = np.stack([s * np.cos(phi), s * np.sin(phi), mu], axis=1)
    from eventmc import kernels
    geom = cell.as_tuple()
    kind = np.zeros(m, np.int64)
    ax = np.zeros(m, np.int64)
    mat = np.zeros(m, np.int64)
    dist = np.zeros(m)
    surf = np.zeros(m, np.int64)
    for i in range(m):
        kd, a, mi = kernels.locate_point(*pts[i], geom)
        kind[i], ax[i], mat[i] = kd, a, mi
        d, sf = kernels.boundary_distance(*pts[i], *dirs[i], kd, a, geom)
        dist[i], surf[i] = d, sf
    np.savez_compressed(os.path.join(OUT, "geometry_c1.npz"), pts=pts, dirs=dirs,
                        kind=kind, axial=ax, mat=mat, dist=dist, surf=surf)

    # particle ops that go through glibc transcendentals
    states = [int(x) for x in rng.randint(0, 2**62, 2000, dtype=np.int64)]
    iso = np.array([transport.sample_isotropic(s)[0] for s in states])
    dcol = np.array([transport.sample_collision_distance(1.7, s)[0]
                     for s in states])
    np.savez_compressed(os.path.join(OUT, "particle_ops.npz"),
                        states=np.array(states, np.uint64), iso=iso, dcol=dcol)

    with open(os.path.join(OUT, "golden.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print("done")


if __name__ == "__main__":
    main()
