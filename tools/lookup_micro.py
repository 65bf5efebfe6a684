"""XS-lookup microbenchmark (k_lookup_bench) on the C4 library with a
realistic in-flight population: 70% fuel (materials 0..99), 30% moderator;
energies = fission spectrum slowed down by k ~ Poisson(2.6) scatters
(E' = E*(0.5+0.5u)).  Sorted by (material, E) like the lookup queue.

    python tools/lookup_micro.py [n] [variants...]
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_12345_b200 as P  # noqa: E402
from paper_2403_12345_b200 import _native as N  # noqa: E402
from paper_2403_12345_b200.engine import DeviceEngine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8_000_000
variants = [int(v) for v in sys.argv[2:]] or [0, 1, 2, 3]
lib, cell = P.depleted_pincell(272, 3, 11303, 100, seed=1)
eng = DeviceEngine(0)
eng.upload_library(lib)
if 9 in variants:      # the pipelined kernel needs the configured sort-key layout
    eng.upload_geometry(cell)
    eng.configure(P.RunConfig(particles_per_batch=1000, max_in_flight=1000), 0, 1000)
rng = np.random.default_rng(1)
mats = np.where(rng.random(n) < 0.7, rng.integers(0, 100, n), 100).astype(np.int32)
E = -1.3e6 * np.log(1 - rng.random(n))
k = rng.poisson(2.6, n)
for j in range(k.max()):
    E = np.where(k > j, E * (0.5 + 0.5 * rng.random(n)), E)
E = np.clip(E, 1e-5, 2e7)
# material-major (plain kernels) and (group, E, material) order (staged kernels:
# 8 = k_lookup_staged, 9 = k_lookup_piped on the production sort key)
order_m = np.lexsort((E, mats))
ebin = np.floor(np.log2(E) * 512).astype(np.int64)     # ~ the production sort's log-hash bin
order_e = np.lexsort((mats, ebin, mats == 100))
ncomp = np.where(mats < 100, 272, 3)
nl = int(ncomp.sum())
for v in variants:
    o = order_e if v in (8, 9) else order_m     # variant 9 re-sorts by the production key
    mo, Eo = np.ascontiguousarray(mats[o]), np.ascontiguousarray(E[o])
    ms, cs = C.c_double(), C.c_double()
    N.check(eng.lib.emc_bench_lookup(eng._h, n, N.ptr(mo), N.ptr(Eo), v, 5, C.byref(ms), C.byref(cs)), "bench")
    print(f"variant {v}: {ms.value:8.3f} ms  {nl / ms.value / 1e6:7.1f} G nuclide-lookups/s  "
          f"{64 * nl / ms.value / 1e6:7.1f} GB/s algorithmic", flush=True)
