"""Multi-GPU batch sharding (one process per GPU, torch.distributed).

The transforms of different coefficient vectors are independent
(SURVEY.md 8(e)), so a batch is split into contiguous per-rank shards with
no data-path collective; the only communication is the optional gather of
the results (NCCL all_gather over NVLink on GPUs, gloo in the CPU tests).
"""

import torch
import torch.distributed as dist


def shard_range(n_items, rank, world):
    """Contiguous balanced [lo, hi) of rank's share of n_items."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n_items, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def gather_rows(local, n_items, group=None):
    """All-gather row shards (produced with shard_range) into the full
    (n_items, ...) tensor on every rank, in rank order."""
    world = dist.get_world_size(group)
    sizes = [shard_range(n_items, r, world) for r in range(world)]
    width = max(hi - lo for lo, hi in sizes)
    pad = local.new_zeros((width,) + tuple(local.shape[1:]))
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([b[: hi - lo] for b, (lo, hi) in zip(bufs, sizes)], dim=0)


def sharded_transform(fn, C, group=None, gather=True):
    """Apply fn (a batched transform, rows = vectors) to this rank's shard of
    C (n_items, N) and optionally gather the full result."""
    if not dist.is_available() or not dist.is_initialized():
        return fn(C)
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    lo, hi = shard_range(C.shape[0], rank, world)
    out = fn(C[lo:hi])
    return gather_rows(out, C.shape[0], group) if gather else out
