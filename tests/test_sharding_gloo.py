"""Multi-process (gloo, CPU) tests of the request-sharding path (§8 a12 / e): every rank
computes the same native LPT partition without communication, runs its whole requests
(here a stand-in computation in TEST code — the product has no CPU path), and the one
collective gathers (request id, [CLS]) to rank 0, which reorders by id.  The result must
equal the single-process result for every world size, and the partition must equal the
independent oracle's bit-exactly."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _fake_cls(rid: int, L: int, d: int) -> torch.Tensor:
    # deterministic per-request stand-in for the encoder's [CLS] row (test code only)
    g = torch.Generator().manual_seed(1000 + rid)
    return (torch.randn(d, generator=g) * L).to(torch.bfloat16)


def _worker(rank, world, port, lens, d, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2006_03031_b200.serve import gather_results, shard
    from paper_2006_03031_b200 import nimble as nb
    ids = shard(lens, world, rank)
    max_count = int(max(np.bincount(nb.partition_lpt(lens, world), minlength=world)))
    cls = torch.stack([_fake_cls(int(i), int(lens[i]), d) for i in ids]) if len(ids) else torch.zeros((0, d), dtype=torch.bfloat16)
    gids, gcls = gather_results(torch.tensor(ids, dtype=torch.int64), cls, max_count, world, rank)
    if rank == 0:
        q.put((gids.numpy().tolist(), gcls.float().numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gather_equals_single_process(world, orc):
    from paper_2006_03031_b200 import build
    build.build()
    lens = np.random.default_rng(7).integers(1, 513, 37).astype(np.int64)
    d = 16
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, lens, d, q)) for r in range(world)]
    for p in procs:
        p.start()
    ids, cls = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert ids == list(range(len(lens)))                       # every request exactly once, in id order
    ref = torch.stack([_fake_cls(i, int(lens[i]), d) for i in range(len(lens))]).float().numpy()
    assert np.array_equal(cls, ref)                            # independent of the world size
    st, owner = orc.partition_lpt(lens, world)
    from paper_2006_03031_b200 import nimble as nb
    assert st == 0 and np.array_equal(nb.partition_lpt(lens, world), owner)


def test_shard_covers_and_balances():
    from paper_2006_03031_b200 import build
    build.build()
    from paper_2006_03031_b200 import nimble as nb
    from paper_2006_03031_b200.serve import shard
    lens = np.random.default_rng(3).integers(1, 513, 4096).astype(np.int64)
    for G in (1, 2, 4, 8):
        parts = [shard(lens, G, r) for r in range(G)]
        allids = np.sort(np.concatenate(parts))
        assert np.array_equal(allids, np.arange(len(lens)))
        loads = [sum(nb.request_cost(int(lens[i])) for i in p) for p in parts]
        assert max(loads) / (sum(loads) / G) < 1.001             # LPT at R = 4096: near-perfect balance


def _worker_steps(rank, world, port, lens, d, steps, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2006_03031_b200.serve import ResultGather, shard
    from paper_2006_03031_b200 import nimble as nb
    ids = shard(lens, world, rank)
    max_count = int(max(np.bincount(nb.partition_lpt(lens, world), minlength=world)))
    g = ResultGather(max_count, d, world, rank, "cpu")
    ids_t = torch.tensor(ids, dtype=torch.int64)
    for step in range(steps):              # the bench's hot loop: gather every step, no host compaction
        cls = torch.stack([_fake_cls(int(i) + 7919 * step, int(lens[i]), d) for i in ids]) if len(ids) else \
            torch.zeros((0, d), dtype=torch.bfloat16)
        g.step(ids_t, cls)
    gids, gcls = g.result()                # once, after the loop: the last step's rows by id
    if rank == 0:
        q.put((gids.numpy().tolist(), gcls.float().numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [1, 2])
def test_result_gather_multi_step_equals_single_process(world):
    """ResultGather (bench.py's per-step collective, no host sync inside the loop): after several
    steps rank 0 holds exactly the last step's [CLS] rows of every request, ordered by id, bit
    for bit the same for G = 1 and G = 2."""
    from paper_2006_03031_b200 import build
    build.build()
    lens = np.random.default_rng(11).integers(1, 513, 23).astype(np.int64)
    d, steps = 8, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_steps, args=(r, world, port, lens, d, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    ids, cls = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert ids == list(range(len(lens)))
    ref = torch.stack([_fake_cls(i + 7919 * (steps - 1), int(lens[i]), d) for i in range(len(lens))]).float().numpy()
    assert np.array_equal(cls, ref)
