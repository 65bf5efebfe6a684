"""Single-process multi-device collectives (distributed.ThreadGroup): the
collectives run_replicated uses when one process drives several GPUs, one
host thread per device.  Here on CPU tensors, worlds of 2, 3 and 8 threads;
the same code moves device tensors with peer copies on a GPU box
(tests/test_gpu_multirank.py::test_thread_ranks_*)."""

import threading

import numpy as np
import pytest

from paper_2403_12345_b200 import distributed as D

torch = pytest.importorskip("torch")


def _run_world(size, fn):
    g = D.ThreadGroup(size)
    out = [None] * size
    errs = []

    def body(r):
        try:
            out[r] = fn(D.World(rank=r, size=size, group=g))
        except BaseException as e:  # noqa: BLE001
            errs.append(e)
            g.abort()

    ts = [threading.Thread(target=body, args=(r,)) for r in range(size)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(60)
    if errs:
        raise errs[0]
    return out


@pytest.mark.parametrize("size", [2, 3, 8])
def test_thread_collectives(size):
    n_bins = 11
    rng = np.random.default_rng(size)
    bins = [rng.integers(0, n_bins, 50) for _ in range(size)]
    vals = [rng.random(50) for _ in range(size)]
    counts = np.arange(1, size + 1, dtype=np.int64) * 3

    def fn(w):
        r = w.rank

        def fold_local(init):
            out = np.zeros(n_bins) if init is None else init.copy()
            for b, v in zip(bins[r], vals[r]):
                out[b] += v
            return out
        chained = D.chained_fold(w, fold_local, n_bins)
        fast = D.fast_bins(w, np.full(n_bins, float(r + 1)))
        per_rank = D.allgather_array(w, np.array([r + 1, 10 * (r + 1)], np.int64))
        lo = int(counts[:r].sum())
        cols = [torch.arange(lo, lo + int(counts[r]), dtype=torch.int64)] + \
            [torch.full((int(counts[r]),), float(r)) for _ in range(2)]
        bank = D.gather_bank(w, cols, counts)
        red = D.allreduce_tensor(w, torch.full((4,), float(r + 1)))
        return chained, fast, per_rank, bank, red

    res = _run_world(size, fn)
    ref = np.zeros(n_bins)
    for r in range(size):
        for b, v in zip(bins[r], vals[r]):
            ref[b] += v
    for r, (chained, fast, per_rank, bank, red) in enumerate(res):
        assert np.array_equal(chained, ref)            # bit-identical to one sequential fold
        assert np.array_equal(fast, np.full(n_bins, float(sum(range(1, size + 1)))))
        assert per_rank[:, 0].tolist() == list(range(1, size + 1))
        assert red.tolist() == [float(sum(range(1, size + 1)))] * 4
        if r == 0:
            assert bank[0].tolist() == list(range(int(counts.sum())))
            assert bank[1].tolist() == sum(([float(q)] * int(counts[q]) for q in range(size)), [])
        else:
            assert bank is None


def _check_windows(size, counts, ppb, u):
    counts = np.asarray(counts, np.int64)
    n = int(counts.sum())
    glob = torch.arange(n, dtype=torch.float64) * 1.5 + 0.25

    def fn(w):
        lo = int(counts[:w.rank].sum())
        mine = [glob[lo:lo + int(counts[w.rank])].clone(), -glob[lo:lo + int(counts[w.rank])].clone()]
        return D.exchange_bank(w, mine, counts, ppb, u)

    for r, (win, wlo) in enumerate(_run_world(size, fn)):
        g_lo, g_hi = D.block_of(r, size, ppb)
        g = np.arange(g_lo, g_hi, dtype=np.float64)
        if n >= ppb:
            i = np.clip(np.floor(((g + u) * float(n)) / float(ppb)), 0, n - 1).astype(np.int64)
        else:
            i = (g % n).astype(np.int64)
        j = (i - wlo) % n
        assert (j < win[0].shape[0]).all()
        assert np.array_equal(win[0].numpy()[j], glob.numpy()[i])
        assert np.array_equal(win[1].numpy()[j], -glob.numpy()[i])


@pytest.mark.parametrize("counts,ppb,u", [
    ([30, 25, 41], 90, 0.37),
    ([10, 0, 17], 60, 0.9),
    ([5, 3, 2], 3, 0.01),
    ([0, 0, 7], 12, 0.5),
])
def test_thread_bank_window_exchange(counts, ppb, u):
    _check_windows(3, counts, ppb, u)


def test_thread_world8_exchange_c4_like():
    """8 ranks at C4's shape scaled down 100x: 400k particles per rank,
    ~1 site per particle, uneven per-rank counts."""
    rng = np.random.default_rng(8)
    counts = rng.integers(380_000, 420_000, 8)
    _check_windows(8, counts, 8 * 400_000, 0.6180339887)


def test_thread_error_aborts_peers():
    """A rank that fails aborts the barrier: its peers stop waiting."""
    def fn(w):
        if w.rank == 1:
            raise ValueError("rank 1 failed")
        D.allgather_array(w, np.zeros(2))
        return True
    with pytest.raises((ValueError, threading.BrokenBarrierError)):
        _run_world(3, fn)
