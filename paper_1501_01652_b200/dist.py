"""Multi-GPU execution (one process per GPU, torch.distributed).

Batches: the transforms of different coefficient vectors are independent
(SURVEY.md 8(e)), so a batch is split into contiguous per-rank shards with
no data-path collective; the only communication is the optional gather of
the results (NCCL all_gather over NVLink on GPUs, gloo in the CPU tests).

One transform over several GPUs: the T = 2M(2P+1) asymptotic DCT/DST pairs
and the near-field tiles of an application are independent, so every rank
runs the whole call with the work split of _device.sharding (rank r of W
computes term pairs [M r/W, M (r+1)/W) of every block and near-field tiles
t = r mod W; direct sums on rank 0) and the partial outputs are summed by
one all-reduce (NCCL over NVLink/NVSwitch) -- the "shard the pairs, then
reduce" form of SURVEY.md 8(e).
"""

import numpy as np
import torch
import torch.distributed as dist

from . import _device


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


def all_to_all_exchange(group=None):
    """The exchange callable of the distributed four-step: equal chunks of
    the send buffer go to every rank (NCCL all-to-all over NVLink/NVSwitch on
    the current stream)."""
    def xfn(send, recv, bytes_per_peer):
        world = dist.get_world_size(group)
        m = world * bytes_per_peer
        dist.all_to_all_single(recv[:m], send[:m], group=group)
    return xfn


def distributed_transform(fn, *args, group=None, exchange="pairs", **kwargs):
    """Evaluate ONE transform call fn(*args, **kwargs) (e.g.
    schlomilch_fast(params, c)) split across the ranks of `group`; every rank
    passes the same arguments and receives the full result (sum of the rank
    partials).  Pass CUDA tensors to keep the result on the device; a numpy
    result is reduced through a tensor on the backend's device.

    exchange="pairs"    -- each rank computes a share of the term pairs of every
                           block (no exchange before the final all-reduce);
    exchange="alltoall" -- full blocks of power-of-two grids run as a
                           distributed four-step FFT with one all-to-all per
                           round (north star: the FFT transpose over NVLink);
                           other work as "pairs"."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return fn(*args, **kwargs)
    if exchange not in ("pairs", "alltoall"):
        raise ValueError("exchange must be 'pairs' or 'alltoall'")
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    xfn = all_to_all_exchange(group) if exchange == "alltoall" else None
    with _device.sharding(rank, world, exchange=xfn):
        out = fn(*args, **kwargs)
    if isinstance(out, torch.Tensor):
        dist.all_reduce(out, group=group)
        return out
    arr = np.asarray(out)
    on_gpu = dist.get_backend(group) == "nccl"
    t = torch.from_numpy(np.ascontiguousarray(arr))
    if on_gpu:
        t = t.to(_device.device())
    if t.is_complex():
        t = torch.view_as_real(t)
        dist.all_reduce(t, group=group)
        return torch.view_as_complex(t).cpu().numpy()
    dist.all_reduce(t, group=group)
    return t.cpu().numpy()
