"""Fingerprint of a C4 / C3 run at 300k particles in flight (1 + 2 batches,
deterministic): printed for comparing lookup configurations run in separate
processes (EMC_LK_PCFG=...)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_12345_b200 as P  # noqa: E402

for name, args in (("c4", (272, 3, 11303, 100)), ("c3", (34, 3, 11303, 100))):
    lib, cell = P.depleted_pincell(*args, seed=1)
    cfg = P.RunConfig(particles_per_batch=300_000, inactive_batches=1, active_batches=2, mode="event",
                      seed=42, max_in_flight=300_000, reduction="deterministic")
    res = P.run_replicated(cfg, lib, cell)
    print("FP", name, os.environ.get("EMC_LK_PCFG", "default"), res.physics_fingerprint(), flush=True)
