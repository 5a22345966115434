"""World-size-2 gloo tests (CPU) of the batch-sharding host logic: shards are disjoint
and cover the batch, the timing reduction is a max over ranks, and gathered per-rank results come
back in image order.  The per-rank compute is stood in by the float64 oracle on each shard (no GPU
here), checked against the unsharded oracle run."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2003_12693_b200.dist import gather_batch, max_over_ranks, shard


@pytest.mark.parametrize("batch,world", [(64, 1), (64, 2), (64, 8), (7, 2), (5, 8), (1, 1)])
def test_shard_partition(batch, world):
    ranges = [shard(batch, world, r) for r in range(world)]
    seen = []
    for s, e in ranges:
        assert 0 <= s <= e <= batch
        seen += list(range(s, e))
    assert seen == list(range(batch))
    sizes = [e - s for s, e in ranges]
    assert max(sizes) - min(sizes) <= 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from synth import make_config
        B = 4
        s, e = shard(B, world, rank)
        cfg = make_config("c3", images=range(s, e), size=(32, 32))
        p = cfg["params"]
        outs = []
        for k in range(e - s):
            st = oracle.run(p, cfg["image"][k], cfg["phi0"][k], 3)
            outs.append(st["phi"])
        local = torch.from_numpy(np.stack(outs))
        full = gather_batch(local, B)
        t = max_over_ranks(float(rank + 1))
        if rank == 0:
            q.put((full.numpy(), t))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_sharded_run_matches_unsharded_gloo():
    import oracle
    from synth import make_config
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    full, t = q.get(timeout=120)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert t == 2.0                                      # max over ranks
    cfg = make_config("c3", images=range(4), size=(32, 32))
    for k in range(4):
        ref = oracle.run(cfg["params"], cfg["image"][k], cfg["phi0"][k], 3)["phi"]
        assert np.array_equal(full[k], ref)              # image order restored, bitwise


def _id_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2003_12693_b200.dist import broadcast_unique_id
        ident = broadcast_unique_id((lambda: bytes(range(128))) if rank == 0 else None)
        q.put((rank, ident))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_unique_id_broadcast_gloo():
    """DistSolver's plumbing: rank 0's NCCL unique id reaches every rank byte for byte."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_id_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert got[0] == got[1] == bytes(range(128))
