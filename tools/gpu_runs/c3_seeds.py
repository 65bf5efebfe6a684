"""Which seeds run the C3 configuration for NB batches without the reference's
boundary GeometryError (GPU only)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2403_12345_b200 as P
lib, cell = P.depleted_pincell(34, 3, 11303, 100, seed=1)
nb = int(os.environ.get("NB", "12"))
for seed in (7, 1, 3, 11):
    cfg = P.RunConfig(particles_per_batch=10_000_000, inactive_batches=3, active_batches=nb - 3, mode="event",
                      max_in_flight=10_000_000, tally_mode="fused", reduction="fast", seed=seed, workers=1)
    try:
        r = P.run_event(cfg, lib, cell)
        print("seed", seed, "ok", r.k_mean if hasattr(r, "k_mean") else list(r.keff)[-1])
    except Exception as e:  # noqa: BLE001
        print("seed", seed, "error", e)
