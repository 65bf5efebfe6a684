"""Per-batch collectives of domain replication over torch.distributed.

One process per GPU.  Rank r owns the contiguous particle block
``[r*P//W, (r+1)*P//W)`` (the reference uses gid mod W, replication.py:178;
physics is assignment-invariant, acceptance criterion 2, and contiguous
blocks make the canonical bank the rank-ordered concatenation of the
rank-local canonical banks).  Per batch:

  * fission bank: all-gather of per-rank site counts; every rank then needs
    only the window of the global canonical bank its own particles resample
    from (a contiguous, possibly wrapped range of ~1/W of the bank, computed
    identically on every rank from the counts and the batch uniform), so the
    sites move with one variable-size all-to-all (NCCL over NVLink on GPU,
    gloo on CPU tests) instead of an all-gather of the whole bank;
  * tallies, deterministic: the canonical per-bin fold is chained through the
    ranks in order (rank r folds its log starting from rank r-1's partial
    sums), which is bit-identical to a single-rank fold -- then broadcast;
  * tallies, fast: all-gather of per-rank bin sums, summed in rank order
    (the reference's `sums += w.wbins` in worker order, R:238-240);
  * counters: all-gather, sums and maxima on the host.

The same collectives also run between threads of ONE process driving several
GPUs (``ThreadGroup``: the reference's single-process API, where
``RunConfig.workers`` is a worker-thread count, R:155-190): each thread owns
one device and one particle block, small arrays are exchanged through shared
host memory behind a barrier, and bank windows move device to device with
peer copies (NVLink) -- no NCCL communicator needed.

Everything here is plumbing on torch tensors; the transport arithmetic stays
in libemc.  The functions take/return plain numpy or torch tensors so the
host logic is testable with the gloo backend on CPU (tests/test_distributed.py).
"""

from __future__ import annotations

import threading
from dataclasses import dataclass

import numpy as np


class ThreadGroup:
    """Collectives between the threads of one process (one thread per GPU).

    Every collective is a rendezvous on one barrier; a thread that fails
    aborts the barrier so its peers raise BrokenBarrierError instead of
    waiting forever (run_replicated re-raises the original error)."""

    def __init__(self, size: int):
        self.size = size
        self.barrier = threading.Barrier(size)
        self.slots: list = [None] * size
        self.shared = None

    def wait(self) -> None:
        self.barrier.wait()

    def abort(self) -> None:
        self.barrier.abort()

    def allgather(self, rank: int, obj) -> list:
        self.slots[rank] = obj
        self.wait()
        out = list(self.slots)
        self.wait()                 # nobody overwrites a slot before all have read it
        return out


@dataclass(frozen=True)
class World:
    rank: int = 0
    size: int = 1
    device_backend: bool = False        # True: collectives on CUDA tensors (NCCL, or peer copies)

    forced: bool = False                # EMC_FORCE_COLLECTIVES=1: collectives even at size 1
    group: ThreadGroup | None = None    # set: threads of one process, not torch.distributed
    device: int = 0                     # this rank's GPU (thread worlds)

    @property
    def distributed(self) -> bool:
        return self.size > 1 or self.forced

    @property
    def threads(self) -> bool:
        return self.group is not None


def current_world() -> World:
    try:
        import torch.distributed as dist
    except Exception:  # noqa: BLE001
        return World()
    if not (dist.is_available() and dist.is_initialized()):
        return World()
    import os
    return World(dist.get_rank(), dist.get_world_size(), dist.get_backend() == "nccl",
                 os.environ.get("EMC_FORCE_COLLECTIVES") == "1")


def block_of(rank: int, size: int, ppb: int) -> tuple[int, int]:
    """[lo, hi) particle indices owned by `rank`."""
    return rank * ppb // size, (rank + 1) * ppb // size


def _tensor_device(world: World):
    import torch
    if world.threads:
        return torch.device("cuda", world.device) if world.device_backend else torch.device("cpu")
    return torch.device("cuda", torch.cuda.current_device()) if world.device_backend \
        else torch.device("cpu")


def allgather_array(world: World, arr: np.ndarray) -> np.ndarray:
    """Stack a small same-shape numpy array from every rank: [W, ...]."""
    if not world.distributed:
        return arr[None, ...].copy()
    if world.threads:
        return np.stack(world.group.allgather(world.rank, np.array(arr, copy=True)))
    import torch
    import torch.distributed as dist
    t = torch.as_tensor(np.ascontiguousarray(arr)).to(_tensor_device(world))
    parts = [torch.empty_like(t) for _ in range(world.size)]
    dist.all_gather(parts, t)
    return torch.stack(parts).cpu().numpy()


def combine_counters(per_rank: np.ndarray, sums, maxes) -> dict:
    """Counters of all ranks -> run-level dict (R:259-265 semantics)."""
    out = {}
    for name, idx in sums:
        out[name] = int(per_rank[:, idx].sum())
    for name, idx in maxes:
        out[name] = int(per_rank[:, idx].max())
    return out


def fast_bins(world: World, local_bins: np.ndarray) -> np.ndarray:
    """Rank-ordered left fold of per-rank bin sums."""
    allb = allgather_array(world, local_bins)
    total = np.zeros_like(local_bins)
    for r in range(allb.shape[0]):
        total += allb[r]
    return total


def chained_fold(world: World, fold_local, n_bins: int) -> np.ndarray:
    """Deterministic reduction across ranks: rank 0 folds from zeros, rank r
    from rank r-1's result; the last rank's sums are broadcast.
    `fold_local(init: np.ndarray | None) -> np.ndarray`."""
    if not world.distributed:
        return fold_local(None)
    if world.threads:
        g = world.group
        for r in range(world.size):          # the chain: one rank folds at a time, in order
            if world.rank == r:
                g.shared = fold_local(None if r == 0 else g.shared)
            g.wait()
        final = np.array(g.shared, copy=True)
        g.wait()
        return final
    import torch
    import torch.distributed as dist
    dev = _tensor_device(world)
    init = None
    if world.rank > 0:
        t = torch.empty(n_bins, dtype=torch.float64, device=dev)
        dist.recv(t, src=world.rank - 1)
        init = t.cpu().numpy()
    mine = fold_local(init)
    if world.rank < world.size - 1:
        dist.send(torch.as_tensor(mine).to(dev), dst=world.rank + 1)
    final = torch.as_tensor(mine).to(dev)
    dist.broadcast(final, src=world.size - 1)
    return final.cpu().numpy()


BANK_FIELDS = ("parent", "ordinal", "x", "y", "z", "dx", "dy", "dz", "energy")
BANK_DTYPES = ("int64", "int32") + ("float64",) * 7


def gather_bank(world: World, local_cols, counts: np.ndarray):
    """Gather the rank banks into the global canonical bank on rank 0 only
    (the run's single full-bank movement, after the last batch).

    `local_cols`: 9 torch tensors (parent, ordinal, x..energy) of this rank's
    canonical bank; `counts`: int64[W] site counts.  Returns, on rank 0, 9
    HOST torch tensors of length sum(counts) in rank order; None elsewhere."""
    import torch
    total = int(counts.sum())
    if not world.distributed:
        return [c[:total].cpu() for c in local_cols]
    n = int(counts[world.rank])
    if world.threads:
        parts = world.group.allgather(world.rank, [c[:n] for c in local_cols])
        if world.rank != 0:
            return None
        return [torch.cat([parts[r][k].cpu() for r in range(world.size)])
                for k in range(len(local_cols))]
    import torch.distributed as dist
    mx = int(counts.max())
    dev = _tensor_device(world)
    out = []
    for col in local_cols:
        padded = torch.zeros(max(mx, 1), dtype=col.dtype, device=dev)
        if n:
            padded[:n] = col[:n].to(dev)
        parts = [torch.empty_like(padded) for _ in range(world.size)] if world.rank == 0 else None
        dist.gather(padded, parts, dst=0)
        if world.rank == 0:
            out.append(torch.cat([parts[r][:int(counts[r])].cpu() for r in range(world.size)]))
    return out if world.rank == 0 else None


def device_view(ptr: int, n: int, dtype: str, device: int):
    """Zero-copy torch view of a libemc device buffer (__cuda_array_interface__)."""
    import torch

    class _Iface:
        __cuda_array_interface__ = {
            "shape": (n,), "typestr": np.dtype(dtype).str, "data": (int(ptr), False),
            "version": 3, "strides": None,
        }

    return torch.as_tensor(_Iface(), device=torch.device("cuda", device))


def resample_index(g: int, n: int, ppb: int, u: float) -> int:
    """Bank index particle g resamples (transport.py:188-200), with the same
    IEEE double expression the device evaluates (floor(((g + u) * n) / ppb))."""
    if n >= ppb:
        i = int(np.floor(((float(g) + u) * float(n)) / float(ppb)))
        return min(max(i, 0), n - 1)
    return g % n


def needed_window(g_lo: int, g_hi: int, n: int, ppb: int, u: float) -> tuple[int, int]:
    """(lo, length): the particles [g_lo, g_hi) resample from bank indices
    lo, lo+1, ..., lo+length-1 taken modulo n (resample_index is monotone in
    g when n >= ppb, and g mod n otherwise)."""
    if g_hi <= g_lo or n < 1:
        return 0, 0
    if n >= ppb:
        a, b = resample_index(g_lo, n, ppb, u), resample_index(g_hi - 1, n, ppb, u)
        return a, b - a + 1
    if g_hi - g_lo >= n:
        return 0, n
    return g_lo % n, g_hi - g_lo


def _segments(lo: int, length: int, n: int) -> list[tuple[int, int]]:
    """Cyclic window -> up to two linear [a, b) ranges, in window order."""
    if length <= 0:
        return []
    if lo + length <= n:
        return [(lo, lo + length)]
    return [(lo, n), (0, lo + length - n)]


def exchange_bank(world: World, local_cols, counts: np.ndarray, ppb: int, u: float):
    """Move to every rank the window of the global canonical bank its block
    resamples from.  `local_cols`: this rank's canonical bank (any number of
    same-length 1-D tensors, rank-ordered global offsets from `counts`).
    Returns (window_cols, lo): window_cols[c][j] = global_col[c][(lo + j) % n]."""
    import torch
    import torch.distributed as dist
    n = int(counts.sum())
    offs = np.concatenate(([0], np.cumsum(counts))).astype(np.int64)
    wins = [needed_window(*block_of(q, world.size, ppb), n, ppb, u) for q in range(world.size)]
    if not world.distributed:
        lo, length = wins[0]
        segs = _segments(lo, length, n)
        return [torch.cat([c[a:b] for a, b in segs]) if segs else c[:0] for c in local_cols], lo

    def pieces(q: int, r: int) -> list[tuple[int, int]]:
        """parts of rank r's bank that rank q needs, in q's window order (global indices)"""
        out = []
        for a, b in _segments(*wins[q], n):
            lo_, hi_ = max(a, int(offs[r])), min(b, int(offs[r + 1]))
            if hi_ > lo_:
                out.append((lo_, hi_))
        return out

    me = world.rank
    if world.threads:
        return _exchange_threads(world, local_cols, offs, wins, n), wins[me][0]
    send_plan = [pieces(q, me) for q in range(world.size)]
    recv_plan = [pieces(me, r) for r in range(world.size)]
    send_splits = [sum(b - a for a, b in pl) for pl in send_plan]
    recv_splits = [sum(b - a for a, b in pl) for pl in recv_plan]
    # receive buffer order is rank-major; the window order is segment-major
    seg_list = _segments(*wins[me], n)
    order = []                      # (recv buffer offset, global a, global b)
    pos = 0
    for r in range(world.size):
        for a, b in recv_plan[r]:
            order.append((pos, a, b))
            pos += b - a
    dest = []                       # window offset of each received piece
    for _, a, b in order:
        wpos = 0
        for sa, sb in seg_list:
            if sa <= a < sb:
                dest.append(wpos + (a - sa))
                break
            wpos += sb - sa
    dev = _tensor_device(world)
    out_cols = []
    for col in local_cols:
        col = col.to(dev)
        base = int(offs[me])
        send = torch.cat([col[a - base:b - base] for pl in send_plan for a, b in pl]) \
            if sum(send_splits) else col[:0]
        recv = torch.empty(sum(recv_splits), dtype=col.dtype, device=dev)
        dist.all_to_all_single(recv, send.contiguous(), recv_splits, send_splits)
        win = torch.empty_like(recv)
        for (p, a, b), d in zip(order, dest):
            win[d:d + (b - a)] = recv[p:p + (b - a)]
        out_cols.append(win)
    return out_cols, wins[me][0]


def _exchange_threads(world: World, local_cols, offs: np.ndarray, wins, n: int):
    """Thread-world bank exchange: every thread publishes its bank columns
    (tensors on its own GPU) and copies the pieces of its window straight from
    the owners' memory (device-to-device peer copies over NVLink), then waits
    until every thread has finished reading before anyone's next batch may
    overwrite its bank."""
    import torch
    dev = _tensor_device(world)
    parts = world.group.allgather(world.rank, list(local_cols))
    out = []
    for k in range(len(local_cols)):
        pieces = []
        for a, b in _segments(*wins[world.rank], n):
            for r in range(world.size):
                lo_, hi_ = max(a, int(offs[r])), min(b, int(offs[r + 1]))
                if hi_ > lo_:
                    src = parts[r][k][lo_ - int(offs[r]):hi_ - int(offs[r])]
                    pieces.append(src.to(dev, non_blocking=False))
        out.append(torch.cat(pieces) if pieces else local_cols[k][:0].to(dev))
    if dev.type == "cuda":
        torch.cuda.synchronize(dev)
    world.group.wait()
    return out


def allreduce_tensor(world: World, x):
    """Sum of a tensor over ranks (mesh tallies), rank order for threads."""
    if not world.distributed:
        return x
    if world.threads:
        parts = world.group.allgather(world.rank, x)
        tot = parts[0].to(x.device).clone()
        for r in range(1, world.size):
            tot += parts[r].to(x.device)
        world.group.wait()           # peers keep their buffers until everyone has summed
        return tot
    import torch.distributed as dist
    if world.device_backend:
        dist.all_reduce(x)
        return x
    h = x.cpu()                      # gloo (tests): through host memory
    dist.all_reduce(h)
    return h.to(x.device)
