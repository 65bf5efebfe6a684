"""Is the C3 GeometryError (batch 5) reference behaviour?  Runs the oracle (the
C restatement pinned to the reference) on the bench's C3 run configuration
(inactive 3, active 3, 10M particles/batch, seed 42) on all host cores and
reports the first error; then the GPU engine on the same configuration."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2403_12345_b200 as P
from oracle import driver
lib, cell = P.depleted_pincell(34, 3, 11303, 100, seed=1)
nb = int(os.environ.get("NB", "6"))
cfg = dict(particles_per_batch=10_000_000, inactive_batches=3, active_batches=nb - 3, mode="event",
           max_in_flight=10_000_000, tally_mode="fused", reduction="fast", sort_enabled=True,
           sort_every_n=1, seed=42)
try:
    res = P.run_event(P.RunConfig(workers=1, **cfg), lib, cell)
    print("gpu ok keff", list(res.keff))
except Exception as e:  # noqa: BLE001
    print("gpu error:", type(e).__name__, e)
th = os.cpu_count()
t0 = time.time()
try:
    r = driver.run(dict(cfg, workers=th), lib.arrays(), cell.as_tuple(), workers=th)
    print("oracle ok keff", list(r["keff"]), time.time() - t0)
except Exception as e:  # noqa: BLE001
    print("oracle error:", type(e).__name__, e, time.time() - t0)
