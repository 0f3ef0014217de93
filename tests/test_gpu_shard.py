"""One transform split over W workers (dist.distributed_transform).

On the single GPU of the test box the W shards run one after the other in
this process (_device.sharding); their sum must equal the unsplit transform
to rounding, for every far-field form (one-pass, pruned two-pass, chirp-z)
and for the nested Fourier-Bessel / DHT drivers (direct parts on shard 0,
the DHT's overwritten rows zero elsewhere).  W = 1 is the plain call,
bitwise.  The NCCL all-reduce itself is covered by the gloo test in
test_dist.py.
"""

import numpy as np
import pytest
import torch

import paper_1501_01652_b200 as fh
from paper_1501_01652_b200 import _device

pytestmark = pytest.mark.gpu


def _split_sum(fn, world):
    parts = []
    for s in range(world):
        with _device.sharding(s, world):
            parts.append(fn().clone())
    return torch.stack(parts).sum(0)


def _close(a, b, c, eps=1e-15):
    tol = 2 * eps * float(np.abs(np.asarray(c)).sum()) + 1e-300
    return float((a - b).abs().max()) <= tol


@pytest.mark.parametrize("n", [1024, 8192, 3000])          # one-pass, two-pass (pruned), chirp-z
@pytest.mark.parametrize("world", [2, 3, 7])
def test_schlomilch_split_sums_to_full(cuda_dev, n, world):
    rng = np.random.default_rng([5, n])
    c = torch.from_numpy(rng.standard_normal((2, n)) / np.arange(1, n + 1)).to(cuda_dev)
    params = fh.select_params(4, n, 1e-15, gamma=4.0)
    fn = lambda: fh.schlomilch_fast(params, c)
    full = fn()
    assert _close(_split_sum(fn, world), full, c[0].cpu().numpy() + c[1].cpu().numpy())


def test_single_shard_is_plain_call(cuda_dev):
    c = torch.from_numpy(np.random.default_rng(2).standard_normal(8192)).to(cuda_dev)
    params = fh.select_params(0, 8192, 1e-15)
    plain = fh.schlomilch_fast(params, c)
    with _device.sharding(0, 1):
        one = fh.schlomilch_fast(params, c)
    assert torch.equal(plain, one)


def test_fourier_bessel_split(cuda_dev):
    n = 3000
    roots = fh.bessel_roots_j0(n)
    c = torch.from_numpy(np.random.default_rng(9).uniform(-1, 1, n)).to(cuda_dev)
    fn = lambda: fh.fourier_bessel_eval(0, c, 1e-12, roots=roots)
    full = fn()
    assert _close(_split_sum(fn, 3), full, c.cpu().numpy(), eps=1e-12)


def test_dht_split(cuda_dev):
    n = 600
    plan = fh.dht_plan(n, 1e-15)
    c = torch.from_numpy(np.random.default_rng(4).standard_normal(n)).to(cuda_dev)
    fn = lambda: fh.dht(plan, c)
    full = fn()
    assert _close(_split_sum(fn, 2), full, c.cpu().numpy())
    # rows <= row_split come from the direct sums of shard 0 only
    with _device.sharding(1, 2):
        other = fn()
    assert float(other[: plan.row_split].abs().max()) == 0.0


def test_distributed_transform_single_process(cuda_dev):
    from paper_1501_01652_b200.dist import distributed_transform

    c = torch.from_numpy(np.random.default_rng(1).standard_normal(4096)).to(cuda_dev)
    params = fh.select_params(0, 4096, 1e-8)
    assert torch.equal(distributed_transform(fh.schlomilch_fast, params, c), fh.schlomilch_fast(params, c))


# ------------------------------------------- distributed four-step (exchange)
def _exchange_split(fn, world, budget=None):
    """Run `world` simulated ranks as threads on the one GPU (own stream
    each); their exchange callbacks implement the all-to-all by copies between
    the ranks' buffers, bracketed by barriers.  Returns the rank outputs and
    the number of exchange rounds seen by each rank."""
    import threading

    from paper_1501_01652_b200.schlomilch import _Grid

    barrier = threading.Barrier(world)
    sends, outs, rounds, errs = {}, {}, {r: 0 for r in range(world)}, []
    old_budget = _Grid.X_BUDGET
    if budget is not None:
        _Grid.X_BUDGET = budget

    def rank_main(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                def xfn(send, recv, bpp):
                    st.synchronize()
                    sends[r] = send
                    barrier.wait()
                    for s in range(world):
                        recv[s * bpp:(s + 1) * bpp].copy_(sends[s][r * bpp:(r + 1) * bpp])
                    st.synchronize()
                    rounds[r] += 1
                    barrier.wait()

                with _device.sharding(r, world, exchange=xfn):
                    out = fn()
                st.synchronize()
                outs[r] = out.clone()
        except Exception as exc:                         # pragma: no cover - reported below
            errs.append(exc)
            barrier.abort()

    ths = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    try:
        for t in ths:
            t.start()
        for t in ths:
            t.join(300)
    finally:
        _Grid.X_BUDGET = old_budget
    if errs:
        raise errs[0]
    return [outs[r] for r in range(world)], rounds


@pytest.mark.parametrize("n,nu,gamma,world", [(2 ** 14, 0, 0.0, 2), (2 ** 14, 4, 4.0, 4), (2 ** 16, 4, 4.0, 8)])
def test_alltoall_four_step_sums_to_full(cuda_dev, n, nu, gamma, world):
    rng = np.random.default_rng([8, n, world])
    C = torch.from_numpy(rng.standard_normal((3, n)) / np.arange(1, n + 1)).to(cuda_dev)
    params = fh.select_params(nu, n, 1e-15, gamma=gamma)
    fn = lambda: fh.schlomilch_fast(params, C)
    full = fn()
    from paper_1501_01652_b200.schlomilch import _grid
    sc = fh.build_partition(params)
    g = _grid(params.n, params.gamma, params.m_terms, sc.blocks, sc.mask_segments, [nu])
    unit = g._lib.fhtb_apply_x_unit_bytes(g.handle, world)
    assert unit > 0                                      # the exchange path is taken
    outs, rounds = _exchange_split(fn, world, budget=unit)   # one unit per round
    assert all(v == rounds[0] and v >= 3 for v in rounds.values())
    tot = torch.stack(outs).sum(0)
    l1 = float(C.abs().sum(1).max())
    assert float((tot - full).abs().max()) <= 2e-15 * l1


def test_alltoall_default_budget_single_round(cuda_dev):
    n = 2 ** 15
    C = torch.from_numpy(np.random.default_rng(3).standard_normal((2, n))).to(cuda_dev)
    params = fh.select_params(0, n, 1e-8)
    fn = lambda: fh.schlomilch_fast(params, C)
    full = fn()
    outs, rounds = _exchange_split(fn, 2)
    assert rounds == {0: 1, 1: 1}
    tot = outs[0] + outs[1]
    assert float((tot - full).abs().max()) <= 2e-15 * float(C.abs().sum(1).max())


def test_alltoall_falls_back_without_full_blocks(cuda_dev):
    # chirp-z grid (non-power-of-two N): no exchange rounds, pair split
    n = 3000
    C = torch.from_numpy(np.random.default_rng(5).standard_normal(n)).to(cuda_dev)
    params = fh.select_params(0, n, 1e-15)
    fn = lambda: fh.schlomilch_fast(params, C)
    full = fn()
    outs, rounds = _exchange_split(fn, 3)
    assert rounds == {0: 0, 1: 0, 2: 0}
    assert _close(outs[0] + outs[1] + outs[2], full, C.cpu().numpy())


def test_alltoall_single_2_24_transform_over_8(cuda_dev):
    """BASELINE configs[4]: one N = 2^24 transform split over 8 ranks with the
    all-to-all four-step (2L = 2^25: 8192-point pass-1 column slabs of 512
    columns per rank); the rank outputs sum to the one-GPU transform."""
    n, eps = 2 ** 24, 1e-15
    C = torch.from_numpy(np.random.default_rng(24).standard_normal((1, n))).to(cuda_dev)
    params = fh.select_params(0, n, eps)
    fn = lambda: fh.schlomilch_fast(params, C)
    full = fn()
    outs, rounds = _exchange_split(fn, 8)
    assert all(v == rounds[0] and v >= 1 for v in rounds.values())
    tot = torch.stack(outs).sum(0)
    assert float((tot - full).abs().max()) <= 2e-15 * float(C.abs().sum())
