"""Multi-rank coordinator on the GPU: two ranks (gloo, sharing cuda:0 --
NCCL cannot put two ranks on one GPU, and gpurun provides one) run the C1
golden problem through run_replicated with the windowed bank exchange and
the chained deterministic reduction.  Domain replication is
partition-invariant (reference acceptance criterion 2), so both ranks must
reproduce the reference's single-worker fingerprint bit for bit."""

import os
import socket

import numpy as np
import pytest

from conftest import golden_library

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, q, run, pm):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2403_12345_b200 as P
        cell = P.Pincell(n_axial=pm["n_axial"], fuel_material_ids=pm["fuel_material_ids"],
                         moderator_material_id=pm["moderator_material_id"])
        cfg = P.RunConfig(**dict(run["config"], workers=world))
        res = P.run_replicated(cfg, golden_library(run["problem"]), cell)
        q.put((rank, res.physics_fingerprint(), res.keff.values.tolist(), len(res.bank)))
    except Exception as e:  # noqa: BLE001
        q.put((rank, f"error: {e!r}", None, None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_multirank_matches_reference_fingerprint(golden, world):
    run = golden["runs"]["c1_event"]
    pm = golden["problems"]["c1"]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, q, run, pm)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(60)
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "run_c1_event.npz"))
    for rank, fp, keff, nbank in res:
        assert np.array_equal(np.array(keff), z["keff"]), rank
        if rank == 0:          # the final bank is gathered to rank 0 only
            assert fp == run["fingerprint"], (rank, fp)
            assert nbank == run["bank_len"]
        else:
            assert nbank == 0


def _nccl_rank(q, run, pm, port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), EMC_FORCE_COLLECTIVES="1")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        import paper_2403_12345_b200 as P
        from paper_2403_12345_b200.distributed import current_world
        w = current_world()
        assert w.device_backend and w.distributed
        cell = P.Pincell(n_axial=pm["n_axial"], fuel_material_ids=pm["fuel_material_ids"],
                         moderator_material_id=pm["moderator_material_id"])
        res = P.run_replicated(P.RunConfig(**run["config"]), golden_library(run["problem"]), cell)
        q.put((res.physics_fingerprint(), len(res.bank)))
    except Exception as e:  # noqa: BLE001
        q.put((f"error: {e!r}", None))
    finally:
        dist.destroy_process_group()


def test_nccl_collective_path_single_gpu(golden):
    """The multi-GPU code path proper -- NCCL on device tensors, zero-copy
    views of libemc's bank, the windowed all-to-all exchange, the device
    source window and the final bank all-gather -- forced on at world size 1
    (the only NCCL world one GPU allows): the reference's C1 fingerprint."""
    run = golden["runs"]["c1_event"]
    pm = golden["problems"]["c1"]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_rank, args=(q, run, pm, _free_port()))
    p.start()
    fp, nbank = q.get(timeout=600)
    p.join(60)
    assert fp == run["fingerprint"], fp
    assert nbank == run["bank_len"]


@pytest.mark.parametrize("devices", [[0, 0], [0, 0, 0]])
def test_thread_ranks_match_reference_fingerprint(golden, devices):
    """Single-process multi-device coordinator (one host thread per rank,
    ThreadGroup collectives, device-to-device window copies): with several
    ranks sharing cuda:0 it must reproduce the reference's C1 fingerprint."""
    import paper_2403_12345_b200 as P
    run = golden["runs"]["c1_event"]
    pm = golden["problems"]["c1"]
    cell = P.Pincell(n_axial=pm["n_axial"], fuel_material_ids=pm["fuel_material_ids"],
                     moderator_material_id=pm["moderator_material_id"])
    cfg = P.RunConfig(**dict(run["config"], workers=len(devices)))
    res = P.run_replicated(cfg, golden_library(run["problem"]), cell, devices=devices)
    assert res.physics_fingerprint() == run["fingerprint"]
    assert res.timings["ranks"] == len(devices)


def test_thread_ranks_fast_reduction_and_errors(golden):
    """Fast reduction across thread ranks: the rank-ordered sum of per-rank
    bins (R:238-240) rounds differently from one rank's sum, exactly as the
    reference's worker-order sum does, so only batch 0 (same histories,
    k_run = 1) is compared, to 1e-12.  A device error in one rank surfaces as
    the reference's exception (every rank sees it in the packed all-gather)."""
    import paper_2403_12345_b200 as P
    run = golden["runs"]["c1_event"]
    pm = golden["problems"]["c1"]
    cell = P.Pincell(n_axial=pm["n_axial"], fuel_material_ids=pm["fuel_material_ids"],
                     moderator_material_id=pm["moderator_material_id"])
    lib = golden_library(run["problem"])
    cfg = P.RunConfig(**dict(run["config"], reduction="fast", workers=2))
    a = P.run_replicated(cfg, lib, cell, devices=[0, 0])
    b = P.run_replicated(cfg, lib, cell, devices=[0])
    assert abs(a.keff.values[0] - b.keff.values[0]) <= 1e-12 * b.keff.values[0]
    assert a.counters["sourced"] == b.counters["sourced"]

    grid = np.array([1.0e-5, 2.0e7])
    nuc = P.NuclideXS(grid, np.full(2, 5.0 + 2e-13), np.full(2, 5.0), np.full(2, 1e-13),
                      np.full(2, 1e-13), 0.0)
    scatter = P.Library([nuc], [P.Material(0, [(0, 1.0)])])
    with pytest.raises(P.StreamOverlapError):
        P.run_replicated(P.RunConfig(particles_per_batch=2, inactive_batches=1, active_batches=0,
                                     mode="event", seed=1, workers=2),
                         scatter, P.analytic_infinite_medium()[1], devices=[0, 0])


def _group_run(run, pm, lib, world):
    """A minimal host coordinator over the C-ABI group entry points (what a
    non-Python host would write): W contexts, one particle block each, then per
    batch emc_run_batch on every rank, emc_group_reduce_bins, k, and
    emc_group_exchange_bank for the next batch's source."""
    import ctypes as C
    import hashlib

    import paper_2403_12345_b200 as P
    from paper_2403_12345_b200 import _native as N
    from paper_2403_12345_b200 import prng
    from paper_2403_12345_b200.distributed import block_of
    from paper_2403_12345_b200.engine import DeviceEngine
    from paper_2403_12345_b200.tally import TallyLayout
    cell = P.Pincell(n_axial=pm["n_axial"], fuel_material_ids=pm["fuel_material_ids"],
                     moderator_material_id=pm["moderator_material_id"])
    cfg = P.RunConfig(**dict(run["config"], workers=world))
    ppb = cfg.particles_per_batch
    engs = []
    for r in range(world):
        e = DeviceEngine(0)
        e.upload_library(lib)
        e.upload_geometry(cell)
        e.set_extensions(cell, cfg)
        lo, hi = block_of(r, world, ppb)
        e.configure(cfg, lo, hi - lo)
        engs.append(e)
    lay = TallyLayout(cell.n_axial)
    arr = (C.c_void_p * world)(*[e._h.value for e in engs])
    grp = C.c_void_p()
    N.check(engs[0].lib.emc_group_create(arr, world, C.byref(grp)), "emc_group_create")
    try:
        keff, sums_all, k_run = [], [], 1.0
        for b in range(cfg.n_batches):
            for e in engs:
                out = e.run_batch(b, k_run, batch0=(b == 0), score=b >= cfg.inactive_batches)
                assert out.error == 0
            sums = np.zeros(lay.n_bins)
            N.check(engs[0].lib.emc_group_reduce_bins(grp, N.ptr(sums), lay.n_bins), "emc_group_reduce_bins")
            sums_all.append(sums)
            keff.append(sums[lay.keff_bin] / ppb)
            if b < cfg.n_batches - 1:
                u, _ = prng.next_uniform(prng.batch_stream(cfg.seed, b))
                n = C.c_int64()
                N.check(engs[0].lib.emc_group_exchange_bank(grp, ppb, u, C.byref(n)), "emc_group_exchange_bank")
                k_run = keff[-1]
        cols = [np.concatenate(c) for c in zip(*[e.bank_to_host() for e in engs])]
        bank = P.FissionBank(*cols)
        h = hashlib.sha256()
        h.update(np.ascontiguousarray(np.array(keff)).tobytes())
        h.update(np.ascontiguousarray(np.array(sums_all)).tobytes())
        h.update(bank.tobytes())
        return h.hexdigest(), np.array(keff)
    finally:
        engs[0].lib.emc_group_destroy(grp)
        for e in engs:
            e.close()


@pytest.mark.parametrize("world", [2, 3])
def test_c_abi_group_matches_reference_fingerprint(golden, world):
    """The C-ABI multi-GPU group (emc_group_*) driven by a minimal coordinator
    with W contexts on cuda:0 reproduces the reference's C1 fingerprint."""
    run = golden["runs"]["c1_event"]
    pm = golden["problems"]["c1"]
    fp, keff = _group_run(run, pm, golden_library(run["problem"]), world)
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "run_c1_event.npz"))
    assert np.array_equal(keff, z["keff"])
    assert fp == run["fingerprint"]
