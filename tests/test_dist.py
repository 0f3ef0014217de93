"""Batch sharding over ranks (world_size 2, gloo on CPU).  The GPU transform
is replaced by a row-wise CPU stand-in; what is tested is the host logic:
balanced contiguous shards, no collective on the data path, rank-ordered
gather."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1501_01652_b200.dist import gather_rows, shard_range, sharded_transform


def test_shard_range_partitions_exactly():
    for n in (0, 1, 7, 64, 65, 256):
        for world in (1, 2, 3, 8):
            spans = [shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_items, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        C = torch.arange(n_items * 5, dtype=torch.float64).reshape(n_items, 5)
        calls = []

        def fn(x):
            calls.append(x.shape[0])
            return 3.0 * x + 1.0

        full = sharded_transform(fn, C)
        lo, hi = shard_range(n_items, rank, world)
        ok = torch.equal(full, 3.0 * C + 1.0) and calls == [hi - lo]
        local = sharded_transform(fn, C, gather=False)
        ok = ok and torch.equal(local, 3.0 * C[lo:hi] + 1.0)
        g = gather_rows(local, n_items)
        ok = ok and torch.equal(g, 3.0 * C + 1.0)
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_items", [7, 64])
def test_two_rank_sharded_transform(n_items):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_items, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    res = dict(q.get(timeout=10) for _ in range(2))
    assert res == {0: True, 1: True}
    assert all(p.exitcode == 0 for p in procs)


# ----------------------------------------------- one transform over the ranks
def _split_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import numpy as np

        from paper_1501_01652_b200 import _device
        from paper_1501_01652_b200.dist import distributed_transform

        terms = torch.arange(1, 11, dtype=torch.float64)            # 10 "pairs"
        seen = []

        def fn(scale, as_numpy=False):
            # stand-in for an engine call: contributes the pairs of its shard
            s, n = _device.shard()
            seen.append((s, n))
            lo, hi = (len(terms) * s) // n, (len(terms) * (s + 1)) // n
            part = torch.zeros(4, dtype=torch.float64)
            part += scale * terms[lo:hi].sum()
            if s == 0:
                part[0] += 100.0                                      # "direct" part on shard 0 only
            return part.numpy() if as_numpy else part

        full = torch.full((4,), 2.0 * terms.sum().item())
        full[0] += 100.0
        out_t = distributed_transform(fn, 2.0)
        out_n = distributed_transform(fn, 2.0, as_numpy=True)
        ok = torch.equal(out_t, full) and np.array_equal(out_n, full.numpy())
        ok = ok and seen == [(rank, world), (rank, world)] and _device.shard() == (0, 1)
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def test_two_rank_split_single_transform():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_split_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    res = dict(q.get(timeout=10) for _ in range(2))
    assert res == {0: True, 1: True}
    assert all(p.exitcode == 0 for p in procs)


def test_sharding_context_validation():
    from paper_1501_01652_b200 import _device

    with pytest.raises(ValueError):
        with _device.sharding(2, 2):
            pass
    with _device.sharding(1, 3):
        assert _device.shard() == (1, 3)
        with _device.sharding(0, 2):
            assert _device.shard() == (0, 2)
        assert _device.shard() == (1, 3)
    assert _device.shard() == (0, 1)


def _a2a_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1501_01652_b200.dist import all_to_all_exchange

        bpp = 24
        send = torch.zeros(world * bpp + 16, dtype=torch.uint8)    # buffers may be larger than used
        for s in range(world):
            send[s * bpp:(s + 1) * bpp] = 10 * rank + s
        recv = torch.full((world * bpp + 16,), 255, dtype=torch.uint8)
        all_to_all_exchange()(send, recv, bpp)
        ok = all(bool((recv[s * bpp:(s + 1) * bpp] == 10 * s + rank).all()) for s in range(world))
        ok = ok and bool((recv[world * bpp:] == 255).all())
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_two_rank_all_to_all_exchange():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_a2a_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    res = dict(q.get(timeout=10) for _ in range(2))
    assert res == {0: True, 1: True}
