"""Host-side profile of the C5 workload (fixed-source slab + mesh)."""
import cProfile, pstats, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2403_12345_b200 as P
lib, cell = P.shielding_slab()
cfg = P.RunConfig(particles_per_batch=10_000_000, inactive_batches=1, active_batches=4, mode="event",
                  sort_enabled=True, max_in_flight=10_000_000, tally_mode="fused", reduction="fast",
                  seed=42, workers=1, run_mode="fixed_source", mesh=(100, 100, 120))
P.run_event(cfg, lib, cell)
t = []
def on_batch(b, phase, e):
    torch.cuda.synchronize(); t.append((b, phase, time.perf_counter()))
pr = cProfile.Profile(); pr.enable()
t0 = time.perf_counter(); res = P.run_event(cfg, lib, cell, on_batch=on_batch); t1 = time.perf_counter()
pr.disable()
print("wall per batch ms", (t1 - t0) / 5 * 1e3, {k: round(v, 4) for k, v in res.timings.items() if isinstance(v, float)})
d = [(t[i + 1][2] - t[i][2]) * 1e3 for i in range(0, len(t) - 1, 2)]
g = [(t[i + 1][2] - t[i][2]) * 1e3 for i in range(1, len(t) - 1, 2)]
print("in-batch ms", [round(x, 2) for x in d], "between ms", [round(x, 2) for x in g])
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
