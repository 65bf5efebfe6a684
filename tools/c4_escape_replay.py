"""Reproduce and explain the C4 'particle outside the cell box' stop.

BENCH_r01 died in batch 22 of the driver's 5 + 20 batch C4 run with
GeometryError 'particle outside the cell box (batch 22, particle 9583593)'.
This script (GPU box) runs the same C4 problem through the public API with the
same RunConfig as bench.py, keeps the canonical banks of the two latest
batches on the host, and when the run stops it traces the offending source
site back to its parent history:

  particle g of batch B resamples site idx = floor((g+u_B)*n/ppb) of bank B-1
  (transport.py:188-200, u_B = batch_stream(seed, B-1));
  that site's parent p started batch B-1 from site idx' of bank B-2.

It then replays the single history p of batch B-1 in the CPU oracle (the C
restatement of the reference kernels) from that source site with the k_run the
GPU used, and compares the sites it banks with the GPU's, bit for bit.  The
oracle is the checker here (tools/, test infrastructure), never the product.

    python tools/c4_escape_replay.py [--batches 25] [--warmup 5] [--seed 42]
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def replay_history(lib_arrays, geom, *, seed, batch, ppb, gid, site, k_run, box_guard=0):
    """One history (gid) of batch `batch` from source `site` (x,y,z,dx,dy,dz,E)
    through the oracle's history executor; returns (counters, banked sites)."""
    from oracle import driver as D
    olib = D.OracleLibrary(lib_arrays)
    ogeom = D.OracleGeometry(geom, guard=bool(box_guard))
    cfg = dict(D.DEFAULTS, mode="history", particles_per_batch=ppb)
    w = D._Worker(np.array([gid], np.int64), cfg, olib.max_comp, (ogeom.n_axial + 1) * 5 + 1)
    src = [np.array([v], np.float64) for v in site]
    # the kernels index the source by gid: point each column gid elements before its value
    src_s = D.OSrc(*[C.c_void_p(a.ctypes.data - 8 * gid) for a in src])
    params = D.OParams(seed & D.MASK63, batch, ppb, 0.5, 1.3e6, float(k_run), 1, 1, 0, 1, 1,
                       int(batch == 0), 1, -1, 0, 0, 0.0)
    D._run_worker(w, olib, ogeom, src_s, params, (ogeom.n_axial + 1) * 5 + 1)
    n = int(w.counters[D.CNT["SITE_N"]])
    return w.counters.copy(), [a[:n].copy() for a in w.sites]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", type=int, default=25)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--ppb", type=int, default=40_000_000)
    ap.add_argument("--box-guard", action="store_true")
    ap.add_argument("--out", default="gpurun_out/c4_escape.json")
    args = ap.parse_args()

    import paper_2403_12345_b200 as P
    from paper_2403_12345_b200 import engine as E
    from paper_2403_12345_b200 import prng

    lib, cell = P.depleted_pincell(272, 3, 11303, 100, seed=1)
    cfg = P.RunConfig(particles_per_batch=args.ppb, inactive_batches=args.warmup,
                      active_batches=args.batches - args.warmup, mode="event", sort_enabled=True,
                      max_in_flight=args.ppb, tally_mode="fused", reduction="fast", seed=args.seed,
                      **({"box_guard": True} if args.box_guard else {}))
    banks: dict[int, tuple] = {}
    k_runs: dict[int, float] = {}
    orig = E.DeviceEngine.run_batch

    def run_batch(self, batch, k_run, batch0, score):
        out = orig(self, batch, k_run, batch0, score)
        k_runs[batch] = k_run
        if out.error == 0:
            banks[batch] = self.bank_to_host()
            banks.pop(batch - 2, None)
        return out

    E.DeviceEngine.run_batch = run_batch
    t0 = time.time()
    report = dict(config=dict(ppb=args.ppb, batches=args.batches, warmup=args.warmup, seed=args.seed,
                              box_guard=args.box_guard))
    try:
        res = P.run_event(cfg, lib, cell)
        report["gpu"] = dict(completed=True, k_mean=res.k_mean, k_stderr=res.k_stderr,
                             counters=res.counters, wall_s=time.time() - t0)
        print(json.dumps(report))
        _write(args.out, report)
        return
    except P.GeometryError as exc:
        msg = str(exc)
        report["gpu"] = dict(completed=False, error=msg, wall_s=time.time() - t0)
    print(msg, flush=True)
    B = int(msg.split("batch ")[1].split(",")[0])
    g = int(msg.rsplit("particle ", 1)[1].rstrip(")"))
    radius, r2, hp, height = cell.as_tuple()[:4]

    def resample(bank, b_next, gg):
        n = bank[0].shape[0]
        u, _ = prng.next_uniform(prng.batch_stream(args.seed, b_next - 1))
        if n >= args.ppb:
            i = int(np.floor((gg + u) * n / args.ppb))
            return min(max(i, 0), n - 1)
        return gg % n

    bank1, bank2 = banks[B - 1], banks[B - 2]
    i1 = resample(bank1, B, g)
    site = [bank1[k][i1] for k in range(9)]
    parent, ordinal = int(site[0]), int(site[1])
    i2 = resample(bank2, B - 1, parent)
    psrc = [float(bank2[k][i2]) for k in range(2, 9)]
    x, y, z = (float(v) for v in site[2:5])
    report["escaped_site"] = dict(bank_batch=B - 1, index=i1, parent=parent, ordinal=ordinal,
                                  xyz=[x, y, z], xyz_hex=[v.hex() for v in (x, y, z)],
                                  hp=hp, height=height,
                                  outside=dict(x=abs(x) > hp, y=abs(y) > hp, z=(z < 0 or z > height)))
    report["parent_source"] = dict(bank_batch=B - 2, index=i2, site=psrc,
                                   site_hex=[v.hex() for v in psrc], k_run=k_runs[B - 1])
    # the parent's banked sites on the GPU (contiguous in the canonical bank)
    sel = np.nonzero(bank1[0] == parent)[0]
    gpu_sites = [[float(bank1[k][j]) for k in range(2, 9)] for j in sel]
    cnt, osites = replay_history(lib.arrays(), cell.as_tuple(), seed=args.seed, batch=B - 1, ppb=args.ppb,
                                 gid=parent, site=psrc, k_run=k_runs[B - 1])
    ora_sites = [[float(osites[k][j]) for k in range(2, 9)] for j in range(osites[0].shape[0])]
    report["oracle_replay"] = dict(error=int(cnt[3]), sites=ora_sites,
                                   captures=int(cnt[5]), fissions=int(cnt[6]),
                                   events=[int(cnt[12]), int(cnt[13]), int(cnt[14])],
                                   draws=int(cnt[8]))
    report["gpu_parent_sites"] = gpu_sites
    report["bit_identical"] = [[a.hex() for a in s] for s in gpu_sites] == \
        [[a.hex() for a in s] for s in ora_sites]
    print(json.dumps(report, indent=1))
    _write(args.out, report)


def _write(path, obj):
    os.makedirs(os.path.dirname(path) or ".", exist_ok=True)
    with open(path, "w") as fh:
        json.dump(obj, fh, indent=1)


if __name__ == "__main__":
    main()
