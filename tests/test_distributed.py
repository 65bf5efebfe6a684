"""Multi-rank coordinator logic over torch.distributed (gloo, world size 2,
CPU): rank partitioning, counter combination, rank-ordered fast reduction,
the chained deterministic fold (must equal a single-rank left fold bit for
bit) and the bank all-gather (rank-ordered concatenation)."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_2403_12345_b200 import distributed as D  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = D.current_world()
        assert (w.rank, w.size, w.device_backend) == (rank, world, False)
        rng = np.random.RandomState(7)
        n_bins = 11
        # per-rank contribution logs already in canonical (bin, gid, ord) order
        vals = [rng.uniform(0.1, 2.0, 40) for _ in range(world)]
        bins = [rng.randint(0, n_bins, 40) for _ in range(world)]

        def fold_local(init):
            out = np.zeros(n_bins) if init is None else init.copy()
            for b, v in zip(bins[rank], vals[rank]):
                out[b] += v
            return out
        chained = D.chained_fold(w, fold_local, n_bins)
        ref = np.zeros(n_bins)
        for r in range(world):
            for b, v in zip(bins[r], vals[r]):
                ref[b] += v
        ok_chain = np.array_equal(chained, ref)

        local = np.full(n_bins, float(rank + 1))
        fast = D.fast_bins(w, local)
        ok_fast = np.array_equal(fast, sum(np.full(n_bins, float(r + 1)) for r in range(world)))

        counts = np.array([3, 5][:world], np.int64)
        n = counts[rank]
        lo = int(counts[:rank].sum())
        cols = [torch.arange(lo, lo + n, dtype=torch.int64), torch.zeros(n, dtype=torch.int32)] + \
            [torch.full((n,), float(rank)) for _ in range(7)]
        g = D.gather_bank(w, cols, counts)
        ok_bank = (g[0].tolist() == list(range(int(counts.sum()))) and
                   g[2].tolist() == [0.0] * 3 + [1.0] * 5) if rank == 0 else g is None

        per_rank = D.allgather_array(w, np.array([rank + 1, 10 * (rank + 1)], np.int64))
        comb = D.combine_counters(per_rank, (("s", 0),), (("m", 1),))
        ok_cnt = comb == {"s": 3, "m": 20}
        q.put((rank, ok_chain, ok_fast, ok_bank, ok_cnt))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_collectives():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(2))
    for rank, *oks in res:
        assert all(oks), (rank, oks)


def test_block_partition_covers_batch():
    for ppb in (1, 7, 100, 40_000_003):
        for w in (1, 2, 3, 8):
            if w > ppb:
                continue
            blocks = [D.block_of(r, w, ppb) for r in range(w)]
            assert blocks[0][0] == 0 and blocks[-1][1] == ppb
            assert all(a[1] == b[0] for a, b in zip(blocks, blocks[1:]))


def _xchg_worker(rank, world, port, q, counts, ppb, u):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = D.current_world()
        counts = np.asarray(counts, np.int64)
        n = int(counts.sum())
        lo = int(counts[:rank].sum())
        glob = torch.arange(n, dtype=torch.float64) * 1.5 + 0.25
        mine = [glob[lo:lo + int(counts[rank])].clone(), -glob[lo:lo + int(counts[rank])].clone()]
        win, wlo = D.exchange_bank(w, mine, counts, ppb, u)
        g_lo, g_hi = D.block_of(rank, world, ppb)
        ok = True
        for g in range(g_lo, g_hi):
            i = D.resample_index(g, n, ppb, u)
            j = (i - wlo) % n
            ok &= j < win[0].shape[0] and float(win[0][j]) == float(glob[i]) and float(win[1][j]) == -float(glob[i])
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("counts,ppb,u", [
    ([30, 25, 41], 90, 0.37),      # bank larger than a batch: monotone windows
    ([10, 0, 17], 60, 0.9),        # bank smaller than a batch: g mod n windows that wrap
    ([5, 3, 2], 3, 0.01),          # tiny batch
    ([0, 0, 7], 12, 0.5),          # all sites on one rank
])
def test_gloo_world3_bank_window_exchange(counts, ppb, u):
    """Every rank receives exactly the bank window its particles resample
    from (the device reads element (i - lo) mod n for global site i)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_xchg_worker, args=(r, 3, port, q, counts, ppb, u)) for r in range(3)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(3))
    assert all(ok for _, ok in res), res


def test_needed_window_covers_resample_indices():
    rng = np.random.default_rng(1)
    for _ in range(2000):
        ppb = int(rng.integers(1, 200))
        w = min(int(rng.integers(1, 9)), ppb)
        n = int(rng.integers(1, 400))
        u = float(rng.random())
        for r in range(w):
            lo, hi = D.block_of(r, w, ppb)
            a, ln = D.needed_window(lo, hi, n, ppb, u)
            need = {D.resample_index(g, n, ppb, u) for g in range(lo, hi)}
            win = {(a + j) % n for j in range(ln)}
            assert need <= win and len(win) == ln <= n
            # tight: ~(block size) x n/ppb sites, i.e. ~1/W of the bank
            bound = (hi - lo) * n // ppb + 2 if n >= ppb else min(n, hi - lo)
            assert ln <= bound


def _xchg_worker_vec(rank, world, port, q, counts, ppb, u):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = D.current_world()
        counts = np.asarray(counts, np.int64)
        n = int(counts.sum())
        lo = int(counts[:rank].sum())
        glob = np.arange(n, dtype=np.float64) * 1.5 + 0.25
        mine = [torch.from_numpy(glob[lo:lo + int(counts[rank])].copy())]
        win, wlo = D.exchange_bank(w, mine, counts, ppb, u)
        g_lo, g_hi = D.block_of(rank, world, ppb)
        g = np.arange(g_lo, g_hi, dtype=np.float64)
        i = np.clip(np.floor(((g + u) * float(n)) / float(ppb)), 0, n - 1).astype(np.int64) \
            if n >= ppb else (g % n).astype(np.int64)
        j = (i - wlo) % n
        ok = bool((j < win[0].shape[0]).all()) and np.array_equal(win[0].numpy()[j], glob[i])
        q.put((rank, ok, int(win[0].shape[0])))
    finally:
        dist.destroy_process_group()


def test_gloo_world8_exchange_c4_like():
    """Eight gloo ranks at C4's shape scaled down 100x (400k particles per
    rank, ~1 site per particle, uneven counts): every rank's window holds the
    sites it resamples, and each moves ~1/8 of the bank, not all of it."""
    rng = np.random.default_rng(8)
    counts = rng.integers(380_000, 420_000, 8).tolist()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_xchg_worker_vec, args=(r, 8, port, q, counts, 8 * 400_000, 0.618))
             for r in range(8)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(8))
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert all(ok for _, ok, _ in res), res
    assert max(ln for _, _, ln in res) < sum(counts) // 8 + 2
