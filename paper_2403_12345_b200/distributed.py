"""Per-batch collectives of domain replication over torch.distributed.

One process per GPU.  Rank r owns the contiguous particle block
``[r*P//W, (r+1)*P//W)`` (the reference uses gid mod W, replication.py:178;
physics is assignment-invariant, acceptance criterion 2, and contiguous
blocks make the canonical bank the rank-ordered concatenation of the
rank-local canonical banks).  Per batch:

  * fission bank: all-gather of per-rank site counts, then all-gather of the
    canonical rank banks (NCCL over NVLink on GPU, gloo on CPU tests) into
    one global bank every rank resamples from;
  * tallies, deterministic: the canonical per-bin fold is chained through the
    ranks in order (rank r folds its log starting from rank r-1's partial
    sums), which is bit-identical to a single-rank fold -- then broadcast;
  * tallies, fast: all-gather of per-rank bin sums, summed in rank order
    (the reference's `sums += w.wbins` in worker order, R:238-240);
  * counters: all-gather, sums and maxima on the host.

Everything here is plumbing on torch tensors; the transport arithmetic stays
in libemc.  The functions take/return plain numpy or torch tensors so the
host logic is testable with the gloo backend on CPU (tests/test_distributed.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class World:
    rank: int = 0
    size: int = 1
    device_backend: bool = False        # True: NCCL (tensors must be on CUDA)

    @property
    def distributed(self) -> bool:
        return self.size > 1


def current_world() -> World:
    try:
        import torch.distributed as dist
    except Exception:  # noqa: BLE001
        return World()
    if not (dist.is_available() and dist.is_initialized()):
        return World()
    return World(dist.get_rank(), dist.get_world_size(), dist.get_backend() == "nccl")


def block_of(rank: int, size: int, ppb: int) -> tuple[int, int]:
    """[lo, hi) particle indices owned by `rank`."""
    return rank * ppb // size, (rank + 1) * ppb // size


def _tensor_device(world: World):
    import torch
    return torch.device("cuda", torch.cuda.current_device()) if world.device_backend \
        else torch.device("cpu")


def allgather_array(world: World, arr: np.ndarray) -> np.ndarray:
    """Stack a small same-shape numpy array from every rank: [W, ...]."""
    if not world.distributed:
        return arr[None, ...].copy()
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
    """All-gather rank banks into the global canonical bank.

    `local_cols`: 9 torch tensors (parent, ordinal, x..energy) of this rank's
    canonical bank; `counts`: int64[W] site counts.  Returns 9 torch tensors
    of length sum(counts), rank order, on the collective's device."""
    import torch
    import torch.distributed as dist
    total = int(counts.sum())
    if not world.distributed:
        return [c[:total] for c in local_cols]
    mx = int(counts.max())
    dev = _tensor_device(world)
    out = []
    for col in local_cols:
        padded = torch.zeros(max(mx, 1), dtype=col.dtype, device=dev)
        n = int(counts[world.rank])
        if n:
            padded[:n] = col[:n].to(dev)
        parts = [torch.empty_like(padded) for _ in range(world.size)]
        dist.all_gather(parts, padded)
        out.append(torch.cat([parts[r][:int(counts[r])] for r in range(world.size)]))
    return out


def device_view(ptr: int, n: int, dtype: str, device: int):
    """Zero-copy torch view of a libemc device buffer (__cuda_array_interface__)."""
    import torch

    class _Iface:
        __cuda_array_interface__ = {
            "shape": (n,), "typestr": np.dtype(dtype).str, "data": (int(ptr), False),
            "version": 3, "strides": None,
        }

    return torch.as_tensor(_Iface(), device=torch.device("cuda", device))
