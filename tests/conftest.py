import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libemc.so")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN, "golden.json")) as fh:
        return json.load(fh)


def golden_lib_arrays(name):
    z = np.load(os.path.join(GOLDEN, f"lib_{name}.npz"))
    return tuple(z[k] for k in ("grid_off", "grids", "ch_t", "ch_s", "ch_c", "ch_f", "nu",
                                "mat_off", "mat_nuc", "mat_den")) + (float(z["emin"]), float(z["emax"]))


def golden_geom(pm, radius=0.4096, pitch=1.26, height=10.0):
    n = pm["n_axial"]
    return (radius, radius * radius, pitch / 2.0, height, np.int64(n),
            np.array([(j * height) / n for j in range(n + 1)]),
            np.asarray(pm["fuel_material_ids"], np.int32), np.int64(pm["moderator_material_id"]))


def golden_library(name):
    """Rebuild a Library object from the committed golden arrays (so GPU
    parity never depends on the host's numpy SIMD paths)."""
    from paper_2403_12345_b200.xslib import Library, Material, NuclideXS
    (grid_off, grids, ch_t, ch_s, ch_c, ch_f, nu, mat_off, mat_nuc, mat_den,
     _, _) = golden_lib_arrays(name)
    nucs = []
    for i in range(grid_off.shape[0] - 1):
        a, b = grid_off[i], grid_off[i + 1]
        nucs.append(NuclideXS(grids[a:b].copy(), ch_t[a:b].copy(), ch_s[a:b].copy(),
                              ch_c[a:b].copy(), ch_f[a:b].copy(), float(nu[i])))
    mats = []
    for m in range(mat_off.shape[0] - 1):
        a, b = mat_off[m], mat_off[m + 1]
        mats.append(Material(m, [(int(mat_nuc[k]), float(mat_den[k])) for k in range(a, b)]))
    return Library(nucs, mats)


def gpu_available():
    try:
        from paper_2403_12345_b200 import _native
        return _native.device_count() > 0
    except Exception:  # noqa: BLE001
        return False


@pytest.fixture
def engine_env(monkeypatch):
    """Set EMC_* tuning variables for one test: the engine reads them when it
    is created, so the cached per-device engines are dropped before and after."""
    def _drop():
        from paper_2403_12345_b200 import replication
        for eng in list(replication._ENGINES.values()):
            eng.close()
        replication._ENGINES.clear()

    def _set(**env):
        for k, v in env.items():
            monkeypatch.setenv(k, str(v))
        _drop()

    yield _set
    monkeypatch.undo()
    _drop()
