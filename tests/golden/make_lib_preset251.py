"""Commit the preset-251 library arrays (depleted_pincell() defaults) as a
fixture, so GPU parity on the 251-nuclide golden run never depends on the GPU
host's numpy SIMD paths.  The arrays come from this package's generator and
are accepted only if their library fingerprint equals the one the reference
recorded in golden.json (make_golden.py ran the reference itself).

    python tests/golden/make_lib_preset251.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import paper_2403_12345_b200 as P  # noqa: E402

lib, cell = P.depleted_pincell()
want = json.load(open(os.path.join(HERE, "golden.json")))["problems"]["preset251"]["library_fingerprint"]
got = P.xslib.library_fingerprint(lib)
if got != want:
    raise SystemExit(f"library fingerprint {got} != reference {want}")
(grid_off, grids, ch_t, ch_s, ch_c, ch_f, nu, mat_off, mat_nuc, mat_den, emin, emax) = lib.arrays()
np.savez_compressed(os.path.join(HERE, "lib_preset251.npz"), grid_off=grid_off, grids=grids, ch_t=ch_t,
                    ch_s=ch_s, ch_c=ch_c, ch_f=ch_f, nu=nu, mat_off=mat_off, mat_nuc=mat_nuc,
                    mat_den=mat_den, emin=np.float64(emin), emax=np.float64(emax))
print("ok", got)
