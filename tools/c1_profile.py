"""C1 (10k particles/batch, 12-nuclide pincell, deterministic reduction):
per-batch wall time split for the event and history executors on the GPU.
    python tools/c1_profile.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_12345_b200 as P  # noqa: E402

lib, cell = P.depleted_pincell(12, 3, 100, 8, seed=1)
for mode in ("event", "history", "event"):
    cfg = P.RunConfig(particles_per_batch=10_000, inactive_batches=5, active_batches=20, mode=mode,
                      max_in_flight=10_000, reduction="deterministic", seed=42)
    t0 = time.perf_counter()
    res = P.run_replicated(cfg, lib, cell)
    wall = time.perf_counter() - t0
    t = res.timings
    print(mode, f"active_rate {res.active_rate / 1e6:.3f} M/s  wall {wall:.3f}s  per-active-batch "
          f"{res.active_wall / 20 * 1e3:.2f} ms; kernel s: lookup {t['lookup']:.4f} adv {t['advance']:.4f} "
          f"coll {t['collision']:.4f} sort {t['sort']:.4f} reduce {t['reduce']:.4f} merge {t['merge']:.4f} "
          f"launches {t['gpu_launches']} fp {res.physics_fingerprint()[:12]}", flush=True)
