"""One active batch of a bench.py workload (default C4: the HM core) at reduced population, for ncu captures: the first
launch of every kernel sees the full in-flight population.

    ncu --set full -k regex:k_lookup -c 1 -o gpurun_out/prof python tools/profile_step.py
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2403_12345_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--particles", type=int, default=4_000_000)
ap.add_argument("--batches", type=int, default=1)
ap.add_argument("--reduction", default="fast")
ap.add_argument("--workload", default="c4", help="bench.py workload whose problem is profiled")
args = ap.parse_args()
import bench  # noqa: E402
lib, cell = bench.problem(args)
cfg = P.RunConfig(particles_per_batch=args.particles, inactive_batches=0,
                  active_batches=args.batches, mode="event", max_in_flight=args.particles,
                  reduction=args.reduction, seed=42)
res = P.run_event(cfg, lib, cell)
print("k", res.keff.values, "timings", {k: v for k, v in res.timings.items()})
