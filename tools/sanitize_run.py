"""Small runs for compute-sanitizer (memcheck / racecheck / synccheck): the
staged pipelined lookup forced on small sorted queues (EMC_TAIL_N=0), the
tail / warp-finish path, both reductions, the history executor and the
fixed-source slab with mesh tallies.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_12345_b200 as P  # noqa: E402


def main():
    lib, cell = P.hm_core(34, 3, 11303, 100, seed=1)
    for red in ("fast", "deterministic"):
        cfg = P.RunConfig(particles_per_batch=20_000, inactive_batches=1, active_batches=1, mode="event",
                          seed=42, max_in_flight=20_000, reduction=red)
        r = P.run_replicated(cfg, lib, cell)
        print(red, "k", r.keff.values, flush=True)
    cfg = P.RunConfig(particles_per_batch=4_000, inactive_batches=1, active_batches=1, mode="history", seed=7)
    print("history k", P.run_replicated(cfg, lib, cell).keff.values, flush=True)
    slib, slab = P.shielding_slab()
    cfg = P.RunConfig(particles_per_batch=20_000, inactive_batches=0, active_batches=1, mode="event", seed=3,
                      run_mode="fixed_source", mesh=(10, 10, 20), reduction="fast")
    print("slab", P.run_replicated(cfg, slib, slab).counters["leaks"], flush=True)


if __name__ == "__main__":
    main()
