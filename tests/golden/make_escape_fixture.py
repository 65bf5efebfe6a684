"""Golden fixture of the C4 box escape (tests/golden/c4_escape.json).

Input: gpurun_out/c4_escape.json written on the GPU box by
tools/c4_escape_replay.py (the driver's C4 bench configuration without the box
guard stopped in batch 22; the script traced the offending source site to the
history that banked it).  This script replays that single history in the CPU
oracle with the box guard off and on and records the sites each banks, so the
tests can pin (a) the oracle/reference behaviour -- sites banked outside the
box -- and (b) the guarded behaviour, on the CPU and on the GPU.

    python tests/golden/make_escape_fixture.py
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def main():
    import paper_2403_12345_b200 as P
    from c4_escape_replay import replay_history
    r = json.load(open(os.path.join(ROOT, "gpurun_out", "c4_escape.json")))
    lib, cell = P.depleted_pincell(272, 3, 11303, 100, seed=1)
    site = [float.fromhex(h) for h in r["parent_source"]["site_hex"]]
    out = dict(problem="depleted_pincell(272,3,11303,100,seed=1)", seed=42, ppb=40_000_000,
               batch=21, gid=r["escaped_site"]["parent"], source_site_hex=r["parent_source"]["site_hex"],
               k_run_hex=float(r["parent_source"]["k_run"]).hex(),
               gpu_error=r["gpu"]["error"],
               gpu_sites_hex=[[v.hex() for v in s] for s in r["gpu_parent_sites"]])
    for guard in (0, 1):
        cnt, sites = replay_history(lib.arrays(), cell.as_tuple(), seed=42, batch=21, ppb=40_000_000,
                                    gid=out["gid"], site=site, k_run=float(r["parent_source"]["k_run"]),
                                    box_guard=guard)
        out[f"guard{guard}"] = dict(
            sites_hex=[[float(sites[k][j]).hex() for k in range(2, 9)] for j in range(sites[0].shape[0])],
            counters={"captures": int(cnt[5]), "fissions": int(cnt[6]), "events_lookup": int(cnt[12]),
                      "events_advance": int(cnt[13]), "events_collision": int(cnt[14]),
                      "draws": int(cnt[8]), "box_guard": int(cnt[23])})
    with open(os.path.join(HERE, "c4_escape.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
