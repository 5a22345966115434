"""Multi-GPU host logic for batch sharding: one process per GPU, images of a batch
split across ranks, no collective inside the iteration loop.  torch.distributed is plumbing only
(barrier, max-over-ranks timing, gathering results); the hot path runs in libsrsb.so per rank.

The functions take a process group / backend-agnostic torch.distributed and are exercised with
the gloo backend on CPU by tests/test_dist.py (world size 2) and with NCCL by bench.py.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard(batch: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous image range [start, stop) of `rank`.  Images are independent problems
    (BASELINE configs[2]); ranks take equal shares and the first batch % world ranks one more."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(batch, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (device time of the timed region) over all ranks."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_batch(local: torch.Tensor, batch: int, device=None) -> torch.Tensor | None:
    """Gather per-rank [n_r, ...] results (in shard order) into the full [batch, ...] tensor on
    rank 0 (None elsewhere).  Shards may differ in size by one image."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return local
    world, rank = dist.get_world_size(), dist.get_rank()
    shape = list(local.shape[1:])
    nmax = -(-batch // world)
    buf = torch.zeros([nmax] + shape, dtype=local.dtype, device=device if device is not None else local.device)
    buf[: local.shape[0]] = local
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf)
    if rank != 0:
        return None
    out = []
    for r in range(world):
        s, e = shard(batch, world, r)
        out.append(parts[r][: e - s])
    return torch.cat(out, 0)


def broadcast_unique_id(make_id=None, group=None, device=None, nbytes: int = 128) -> bytes:
    """Rank 0 calls make_id() (sr_sb_nccl_unique_id) and broadcasts the bytes to every rank of
    `group` (NCCL needs a device tensor: pass device; gloo works on CPU).  Returns the id bytes."""
    rank = dist.get_rank(group)
    buf = torch.zeros(nbytes, dtype=torch.uint8, device=device)
    if rank == 0:
        raw = make_id()
        if len(raw) != nbytes:
            raise ValueError("unexpected unique-id size")
        buf.copy_(torch.frombuffer(bytearray(raw), dtype=torch.uint8))
    src = dist.get_global_rank(group, 0) if group is not None else 0
    dist.broadcast(buf, src, group=group)
    return bytes(buf.cpu().numpy().tobytes())
