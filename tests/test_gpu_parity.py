"""GPU parity against golden vectors produced by the reference package
(tests/golden/make_golden.py).  Bar (BASELINE.json north star): fast paths
within 10*eps*||c||_1 of the reference output; direct sums and point
evaluations at rounding level."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fh(cuda_dev):
    import paper_1501_01652_b200 as m
    return m


def maxerr(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))))


def test_bessel_j(fh, golden):
    meta, A = golden
    z = A["bessel_z"]
    for nu in meta["bessel"]:
        assert maxerr(fh.bessel_j(nu, z), A["bessel_j_%d" % nu]) <= 1e-14, nu


def test_hankel_taylor(fh, golden):
    _, A = golden
    assert maxerr(fh.hankel_asy_eval(0, 10, A["hankel_z"]), A["hankel_0_10"]) <= 2e-16
    assert maxerr(fh.hankel_asy_eval(3, 6, A["hankel_z"]), A["hankel_3_6"]) <= 2e-16
    assert maxerr(fh.taylor_eval(0, 5, A["taylor_z"]), A["taylor_0_5"]) <= 2e-16
    assert maxerr(fh.taylor_eval(2, 9, A["taylor_z"]), A["taylor_2_9"]) <= 2e-16


def test_roots(fh, golden):
    _, A = golden
    t = fh.bessel_roots_j0(3001)
    # Newton iterates to rounding level: agree to a few ulps of the root
    ulp = 8 * 2.0 ** -52 * np.abs(A["roots"])
    assert np.all(np.abs(t.roots - A["roots"]) <= ulp)
    assert np.all(np.abs(t.perturbations - A["perturb"]) <= ulp)
    assert maxerr(t.ratio_perturbation(np.arange(1, 501), 500), A["ratio_500"]) <= 1e-15


def test_trig(fh, golden):
    meta, A = golden
    for kind, n in meta["trig"]:
        key = "trig_%s_%d" % (kind, n)
        v = A[key + "_in"]
        got = fh.apply(fh.make_plan(n, kind), v)
        assert got.shape == v.shape
        assert maxerr(got, A[key + "_out"]) <= 1e-13 * np.abs(v).sum(axis=-1).max(), key
    vc = A["trig_cplx_in"]
    assert maxerr(fh.apply(fh.make_plan(33, fh.DCT1), vc), A["trig_cplx_dct"]) <= 1e-13 * np.abs(vc).sum()
    assert maxerr(fh.apply(fh.make_plan(33, fh.DST1), vc), A["trig_cplx_dst"]) <= 1e-13 * np.abs(vc).sum()


def test_schlomilch(fh, golden):
    meta, A = golden
    for rec in meta["schlomilch"]:
        i = rec["i"]
        c = A["schl_%d_c" % i]
        p = fh.select_params(rec["nu"], rec["n"], rec["eps"], gamma=rec["gamma"])
        tol = 10 * rec["eps"] * np.abs(c).sum()
        st = {}
        got = fh.schlomilch_fast(p, c, stats=st)
        assert got.dtype == A["schl_%d_fast" % i].dtype
        assert maxerr(got, A["schl_%d_fast" % i]) <= tol, (rec, maxerr(got, A["schl_%d_fast" % i]), tol)
        assert st == rec["stats"], (st, rec["stats"])
        assert maxerr(fh.schlomilch_single_partition(p, c), A["schl_%d_single" % i]) <= tol
        if rec["has_direct"]:
            d = fh.schlomilch_direct(rec["nu"], rec["gamma"], c)
            assert maxerr(d, A["schl_%d_direct" % i]) <= 1e-13 * np.abs(c).sum(), rec


def test_blocks(fh, golden):
    meta, A = golden
    for rec in meta["block"]:
        i = rec["i"]
        c = A["block_%d_c" % i]
        p = fh.select_params(rec["nu"], rec["n"], rec["eps"])
        st = {}
        got = fh.asy_block_apply(p, tuple(rec["rows"]), tuple(rec["cols"]), c, st)
        assert maxerr(got, A["block_%d_out" % i]) <= 1e-13 * np.abs(c).sum(), rec
        assert st == rec["stats"]


def test_engine(fh, golden):
    from paper_1501_01652_b200.schlomilch import SchlomilchEngine
    meta, A = golden
    for rec in meta["engine"]:
        i = rec["i"]
        eng = SchlomilchEngine(rec["n"], rec["gamma"], rec["eps"], rec["orders"])
        reqs = [(tuple(map(tuple, r[0])), A["eng_%d_%d_c" % (i, j)]) for j, r in enumerate(rec["reqs"])]
        st = {}
        ys = eng.apply_many(reqs, st)
        for j, y in enumerate(ys):
            assert maxerr(y, A["eng_%d_%d_y" % (i, j)]) <= 10 * rec["eps"] * np.abs(reqs[j][1]).sum()
        assert st == rec["stats"]


def test_fourier_bessel(fh, golden):
    meta, A = golden
    for rec in meta["fb"]:
        i = rec["i"]
        c = A["fb_%d_c" % i]
        tol = 10 * rec["eps"] * np.abs(c).sum()
        st = {}
        got = fh.fourier_bessel_eval(rec["nu"], c, rec["eps"], stats=st)
        assert maxerr(got, A["fb_%d_fast" % i]) <= tol, (rec, maxerr(got, A["fb_%d_fast" % i]), tol)
        assert st == rec["stats"], (st, rec["stats"])
        st = {}
        got = fh.fourier_bessel_eval(rec["nu"], c, rec["eps"], stats=st, prune=True)
        assert maxerr(got, A["fb_%d_prune" % i]) <= tol
        assert st == rec["stats_prune"], (st, rec["stats_prune"])
        d = fh.fourier_bessel_direct(rec["nu"], c)
        assert maxerr(d, A["fb_%d_direct" % i]) <= 1e-13 * np.abs(c).sum()


def test_dht(fh, golden):
    meta, A = golden
    for rec in meta["dht"]:
        i = rec["i"]
        c = A["dht_%d_c" % i]
        plan = fh.dht_plan(rec["n"], rec["eps"])
        assert (plan.k_terms, plan.t_terms, plan.row_split) == (rec["K"], rec["T"], rec["row_split"])
        assert maxerr(plan.weights, A["dht_%d_weights" % i]) <= 1e-12 * np.abs(plan.weights).max()
        tol = 10 * rec["eps"] * np.abs(c).sum()
        st = {}
        got = fh.dht(plan, c, stats=st)
        assert maxerr(got, A["dht_%d_fast" % i]) <= tol, (rec, maxerr(got, A["dht_%d_fast" % i]), tol)
        assert st == rec["stats"], (st, rec["stats"])
        d = fh.dht_direct(plan, c)
        assert maxerr(d, A["dht_%d_direct" % i]) <= 1e-13 * np.abs(c).sum()


def test_self_inverse(fh, golden):
    meta, A = golden
    for rec in meta["selfinv"]:
        r = fh.dht_self_inverse_residual(rec["n"], rec["eps"], A["selfinv_%d_c" % rec["i"]])
        assert abs(r - rec["residual"]) <= 1e-10 + 1e-3 * rec["residual"]


def test_numpy_batch_pipeline_matches_device_path(fh, cuda_dev):
    """Large numpy batches take the pinned-staging pipeline (schlomilch.py
    _run_numpy_pipelined: chunks of vectors on two streams, host copies on
    worker threads); same bits as the device-resident application, any batch
    size (ragged last chunk, odd counts)."""
    import torch
    n = 2 ** 18
    params = fh.select_params(4, n, 1e-15, gamma=4.0)
    for B in (16, 21, 4):
        if B * n < (1 << 22):
            continue
        c = np.random.default_rng([31, B]).standard_normal((B, n)) / np.arange(1, n + 1)
        got = fh.schlomilch_fast(params, c)
        want = fh.schlomilch_fast(params, torch.from_numpy(c).to(cuda_dev)).cpu().numpy()
        assert isinstance(got, np.ndarray) and got.shape == (B, n)
        assert np.array_equal(got, want)
    st = {}
    c = np.random.default_rng(32).standard_normal((16, n))
    fh.schlomilch_fast(params, c, stats=st)
    st2 = {}
    fh.schlomilch_fast(params, torch.from_numpy(c).to(cuda_dev), stats=st2)
    assert st == st2
