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
