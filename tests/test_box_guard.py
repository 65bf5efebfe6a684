"""Box guard (RunConfig.box_guard, include/emc.h) in the CPU oracle.

The C4 escape fixture (tests/golden/c4_escape.json, made by
tests/golden/make_escape_fixture.py from the GPU run traced by
tools/c4_escape_replay.py): one history of batch 21 of the driver's C4 bench
(seed 42, 40M particles per batch) whose nudge across an axial plane carries
it out of the fuel cylinder while its cell stays fuel; fuel cells never test
the box planes, so it flies past x = +hp and banks three fission sites
outside the box, which stops batch 22 with 'particle outside the cell box'.
"""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden_geom, golden_lib_arrays

D = pytest.importorskip("oracle.driver")


@pytest.fixture(scope="module")
def escape():
    with open(os.path.join(GOLDEN, "c4_escape.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="module")
def c4():
    import paper_2403_12345_b200 as P
    return P.depleted_pincell(272, 3, 11303, 100, seed=1)


def _replay(escape, c4, guard):
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(GOLDEN), "..", "tools"))
    from c4_escape_replay import replay_history
    lib, cell = c4
    site = [float.fromhex(h) for h in escape["source_site_hex"]]
    cnt, sites = replay_history(lib.arrays(), cell.as_tuple(), seed=42, batch=escape["batch"],
                                ppb=escape["ppb"], gid=escape["gid"], site=site,
                                k_run=float.fromhex(escape["k_run_hex"]), box_guard=guard)
    return cnt, [[float(sites[k][j]).hex() for k in range(2, 9)] for j in range(sites[0].shape[0])]


def test_oracle_reproduces_gpu_escape(escape, c4):
    """Guard off: the oracle (the reference's kernels restated, pinned to the
    reference's goldens) banks the same three sites as the B200 run did, bit for
    bit, and they lie outside the box -- the stop is the reference's own."""
    cnt, sites = _replay(escape, c4, 0)
    assert sites == escape["gpu_sites_hex"] == escape["guard0"]["sites_hex"]
    hp, height = c4[1].as_tuple()[2], c4[1].as_tuple()[3]
    for s in sites:
        x, y, z = (float.fromhex(v) for v in s[:3])
        assert abs(x) > hp or abs(y) > hp or not (0.0 <= z <= height)
    assert int(cnt[23]) == 0


def test_oracle_guard_keeps_sites_inside(escape, c4):
    cnt, sites = _replay(escape, c4, 1)
    assert sites == escape["guard1"]["sites_hex"]
    assert int(cnt[23]) == escape["guard1"]["counters"]["box_guard"] >= 1
    hp, height = c4[1].as_tuple()[2], c4[1].as_tuple()[3]
    for s in sites:
        x, y, z = (float.fromhex(v) for v in s[:3])
        assert abs(x) <= hp and abs(y) <= hp and 0.0 <= z <= height


@pytest.mark.parametrize("name", ["c1_event", "small_history", "preset251_event_w2"])
def test_guard_leaves_reference_runs_unchanged(golden, name):
    """Histories that stay inside the box are untouched: golden runs keep the
    reference's fingerprint with the guard on."""
    run = golden["runs"][name]
    pm = golden["problems"][run["problem"]]
    cfg = dict(run["config"], box_guard=True)
    res = D.run(cfg, golden_lib_arrays(run["problem"]), golden_geom(pm))
    assert D.fingerprint(res) == run["fingerprint"]
    assert res["counters"]["box_guard"] == 0

