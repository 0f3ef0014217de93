"""The reference's own test strategy (pkg/tests/test_trig.py, test_bessel.py,
test_schlomilch.py; SPEC.md acceptance criteria 2-4, 7, 8), restated against
the drop-in package on the GPU.  Oracles are in-test matrices, scipy and the
GPU direct sums, exactly as the reference tests use them."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fh(cuda_dev):
    import paper_1501_01652_b200 as m
    return m


def cmat(n):
    k = np.arange(n)
    return np.cos(np.outer(k, k) * np.pi / (n - 1))


def smat(n):
    k = np.arange(1, n + 1)
    return np.sin(np.outer(k, k) * np.pi / (n + 1))


# ------------------------------------------------------------------ trig ---

def test_trig_known_small_matrices(fh):
    p = fh.make_plan(2, fh.DCT1)
    got = np.column_stack([fh.apply(p, e) for e in np.eye(2)])
    assert np.allclose(got, [[1.0, 1.0], [1.0, -1.0]], atol=1e-15)
    assert fh.apply(fh.make_plan(1, fh.DST1), np.array([1.0]))[0] == pytest.approx(1.0, abs=1e-15)
    e0 = np.zeros(9)
    e0[0] = 1.0
    assert np.allclose(fh.apply(fh.make_plan(9, fh.DCT1), e0), np.ones(9), atol=1e-14)
    got = fh.apply(fh.make_plan(3, fh.DST1), np.array([1.0, 0.0, 0.0]))
    assert np.allclose(got, np.sin(np.array([1, 2, 3]) * np.pi / 4), atol=1e-15)


@pytest.mark.parametrize("n", list(range(2, 65)))
def test_dct_vs_matrix(fh, n):
    v = np.random.default_rng(n).standard_normal(n)
    assert np.abs(fh.apply(fh.make_plan(n, fh.DCT1), v) - cmat(n) @ v).max() <= 1e-13 * np.abs(v).sum()


@pytest.mark.parametrize("n", list(range(1, 65)))
def test_dst_vs_matrix(fh, n):
    v = np.random.default_rng(n).standard_normal(n)
    assert np.abs(fh.apply(fh.make_plan(n, fh.DST1), v) - smat(n) @ v).max() <= 1e-13 * np.abs(v).sum()


@pytest.mark.parametrize("n,kind", [(500, "dct1"), (500, "dst1"), (1024, "dst1"), (4096, "dct1")])
def test_trig_large(fh, n, kind):
    v = np.random.default_rng(3 * n).standard_normal(n)
    mat = cmat(n) if kind == "dct1" else smat(n)
    assert np.abs(fh.apply(fh.make_plan(n, kind), v) - mat @ v).max() <= 1e-13 * np.abs(v).sum()


def test_trig_linearity_involution_complex_batch(fh):
    p = fh.make_plan(40, fh.DST1)
    g = np.random.default_rng(5)
    u, v = g.standard_normal(40), g.standard_normal(40)
    rhs = 2.5 * fh.apply(p, u) - 1.25 * fh.apply(p, v)
    assert np.abs(fh.apply(p, 2.5 * u - 1.25 * v) - rhs).max() <= 1e-13 * max(1.0, np.abs(rhs).max())
    p = fh.make_plan(51, fh.DST1)
    v = np.random.default_rng(8).standard_normal(51)
    assert np.abs(fh.apply(p, fh.apply(p, v)) - 26.0 * v).max() <= 1e-12 * 26.0 * np.abs(v).max()
    g = np.random.default_rng(44)
    v = g.standard_normal(33) + 1j * g.standard_normal(33)
    for kind, mat in ((fh.DCT1, cmat(33)), (fh.DST1, smat(33))):
        assert np.abs(fh.apply(fh.make_plan(33, kind), v) - mat @ v).max() <= 1e-13 * np.abs(v).sum()
    v = np.random.default_rng(2).standard_normal((5, 20))
    got = fh.apply(fh.make_plan(20, fh.DCT1), v)
    for i in range(5):
        assert np.allclose(got[i], fh.apply(fh.make_plan(20, fh.DCT1), v[i]), atol=1e-14)


# ---------------------------------------------------------------- bessel ---

def test_hankel_eval_vs_scipy(fh):
    special = pytest.importorskip("scipy.special")
    z = np.linspace(17.8, 60.0, 200)
    assert np.abs(fh.hankel_asy_eval(0, 10, z) - special.j0(z)).max() <= 1.6e-15
    assert fh.hankel_asy_eval(0, 3, 200.0) == pytest.approx(-0.015437439930565091592, abs=1.1e-15)
    got = fh.hankel_asy_eval(0, 1, 10.0)
    bound = math.sqrt(2.0 / (10.0 * math.pi)) * (abs(fh.asy_coeff(0, 2)) / 100.0 + abs(fh.asy_coeff(0, 3)) / 1000.0)
    assert abs(got - (-0.2459357644513483352)) <= bound


def test_taylor_eval_points(fh):
    assert fh.taylor_eval(0, 1, 0.0) == 1.0
    assert fh.taylor_eval(1, 1, 0.0) == 0.0
    assert fh.taylor_eval(0, 5, 0.165) == pytest.approx(0.99320532250516262361, abs=1e-15)


def test_bessel_j_special_points_and_scipy(fh):
    special = pytest.importorskip("scipy.special")
    assert fh.bessel_j(0, 0.0) == 1.0
    assert fh.bessel_j(3, 0.0) == 0.0
    assert abs(fh.bessel_j(0, 2.4048255576957727686)) <= 1e-13
    z = np.linspace(0.0, 200.0, 4001)
    for nu in (0, 1, 2, 3, 5, 10, 20):
        assert np.abs(fh.bessel_j(nu, z) - special.jv(nu, z)).max() <= 1e-14, nu
    z = np.random.default_rng(1234).uniform(0.0, 500.0, 20000)
    for nu in (0, 1, 4, 9):
        assert np.abs(fh.bessel_j(nu, z)).max() <= 1.0 + 1e-14


def test_bessel_branch_consistency(fh):
    rng = np.random.default_rng(7)
    for nu, m, eps in ((0, 5, 1e-10), (2, 8, 1e-13), (10, 10, 1e-12)):
        s = fh.asy_cutoff(nu, m, eps)
        z = rng.uniform(s, 3 * s, 500)
        assert np.abs(fh.bessel_j(nu, z) - fh.hankel_asy_eval(nu, m, z)).max() <= 2 * eps
    for nu, t, eps in ((0, 4, 1e-10), (1, 6, 1e-13)):
        z = rng.uniform(0.0, fh.taylor_cutoff(nu, t, eps), 500)
        assert np.abs(fh.bessel_j(nu, z) - fh.taylor_eval(nu, t, z)).max() <= 2 * eps


def test_neumann_addition_lemma_sampled(fh):
    # |J_nu(z+dz) - sum_{|s|<K} J_{nu-s}(z) J_s(dz)| <= 5.2 (e|dz|/2)^K  (Lemma 3.1)
    rng = np.random.default_rng(99)
    cases = []
    for _ in range(300):
        cases.append((int(rng.integers(-10, 11)), rng.uniform(1e-3, 50.0),
                      rng.uniform(-1.0 / math.e, 1.0 / math.e) * 0.999, int(rng.integers(1, 11))))
    # evaluate every needed J on the device in one call per order
    need = {}
    for nu, z, dz, K in cases:
        for s in range(-K + 1, K):
            need.setdefault(abs(nu - s), []).append(z)
            need.setdefault(abs(s), []).append(abs(dz))
        need.setdefault(abs(nu), []).append(abs(z + dz))
    vals = {o: dict(zip(zs, fh.bessel_j(o, np.array(zs)))) for o, zs in need.items()}
    for nu, z, dz, K in cases:
        total = 0.0
        for s in range(-K + 1, K):
            j1 = vals[abs(nu - s)][z] * (-1.0) ** (nu - s if nu < s else 0)
            j2 = vals[abs(s)][abs(dz)]
            if s < 0:
                j2 *= (-1.0) ** s
            if dz < 0:
                j2 *= (-1.0) ** s
            total += j1 * j2
        target = vals[abs(nu)][abs(z + dz)]
        if nu < 0:
            target *= (-1.0) ** nu
        if z + dz < 0:
            target *= (-1.0) ** nu
        assert abs(target - total) <= 5.2 * (math.e * abs(dz) / 2.0) ** K + 5e-14


def test_roots_tables(fh):
    t = fh.bessel_roots_j0(2)
    assert 3 * math.pi / 4 <= t.roots[0] <= 3 * math.pi / 4 + 1.0 / (6 * math.pi)
    assert t.roots[1] == pytest.approx(5.5200781102863106496, abs=1e-12)
    t = fh.bessel_roots_j0(2000)
    n = np.arange(1, 2001)
    assert np.all(np.diff(t.roots) > 0)
    assert np.abs(fh.bessel_j(0, t.roots)).max() <= 1e-13
    slack = 4 * np.finfo(float).eps * t.roots
    assert np.all(t.perturbations >= -slack)
    assert np.all(t.perturbations <= 1.0 / (8 * (n - 0.25) * math.pi) + slack)
    t = fh.bessel_roots_j0(501)
    k = np.arange(1, 501)
    assert np.all(np.abs(t.ratio_perturbation(k, 500)) <= 1.0 / (8 * (500.75) * (k - 0.25) * math.pi ** 2))
    with pytest.raises(ValueError):
        fh.bessel_roots_j0(10).ratio_perturbation(1, 10)


# ------------------------------------------------------------ schlomilch ---

def test_direct_known_answers(fh):
    c = np.zeros(50)
    c[0] = 1.0
    k = np.arange(1, 51)
    assert np.allclose(fh.schlomilch_direct(2, 0.0, c), fh.bessel_j(2, k * np.pi / 50), atol=1e-14, rtol=0)
    assert np.all(fh.schlomilch_direct(0, 0.0, np.zeros(30)) == 0.0)


def test_asy_blocks_vs_masked_matrix(fh):
    n, eps = 64, 1e-8
    for nu, seed in ((0, 0), (1, 5)):
        p = fh.select_params(nu, n, eps)
        lo = math.ceil(p.alpha * math.sqrt(n))
        k = np.arange(1, n + 1)
        mat = fh.bessel_j(nu, np.outer(k, k) * np.pi / n)
        rng = np.random.default_rng(seed)
        blocks = [((lo, n + 1), (lo, n + 1))]
        for _ in range(5):
            r0, c0 = int(rng.integers(lo, n)), int(rng.integers(lo, n))
            blocks.append(((r0, int(rng.integers(r0 + 1, n + 2))), (c0, int(rng.integers(c0 + 1, n + 2)))))
        c = rng.standard_normal(n)
        for (r0, r1), (c0, c1) in blocks:
            got = fh.asy_block_apply(p, (r0, r1), (c0, c1), c)
            mask = (k[:, None] >= r0) & (k[:, None] < r1) & (k[None, :] >= c0) & (k[None, :] < c1)
            assert np.abs(got - (mat * mask) @ c).max() <= 2 * eps * np.abs(c).sum()
    p = fh.select_params(0, 32, 1e-8)
    lo = math.ceil(p.alpha * math.sqrt(32))
    assert np.all(fh.asy_block_apply(p, (lo, 33), (lo, 33), np.zeros(32)) == 0.0)


def test_single_partition_and_border(fh):
    c = np.random.default_rng(17).standard_normal(200)
    p = fh.select_params(0, 200, 1e-15)
    assert np.abs(fh.schlomilch_single_partition(p, c) - fh.schlomilch_direct(0, 0.0, c)).max() <= \
        10e-15 * np.abs(c).sum()
    c = np.zeros(120)
    c[0] = 1.0
    p = fh.select_params(3, 120, 1e-15)
    k = np.arange(1, 121)
    assert np.abs(fh.schlomilch_single_partition(p, c) - fh.bessel_j(3, k * np.pi / 120)).max() <= 1e-14


def test_degenerate_partition_is_bitwise_direct(fh):
    p = fh.select_params(10, 10, 1e-3)
    assert math.ceil(p.alpha * math.sqrt(10)) > 10
    c = np.random.default_rng(4).standard_normal(10)
    assert np.array_equal(fh.schlomilch_single_partition(p, c), fh.schlomilch_direct(10, 0.0, c))


@pytest.mark.parametrize("n,nu,gamma,eps", [(2000, 0, 0.0, 1e-15), (500, 2, 0.0, 1e-8), (500, 2, 0.5, 1e-8),
                                             (400, 0, -0.25, 1e-15), (4096, 4, 4.0, 1e-15)])
def test_fast_vs_direct(fh, n, nu, gamma, eps):
    c = np.random.default_rng(n + nu).standard_normal(n)
    p = fh.select_params(nu, n, eps, gamma=gamma)
    assert np.abs(fh.schlomilch_fast(p, c) - fh.schlomilch_direct(nu, gamma, c)).max() <= 10 * eps * np.abs(c).sum()


def test_fast_equals_single_bitwise_for_every_p0_size(fh):
    # SPEC acceptance 8: every N <= 158 at eps = 1e-15
    for n in range(1, 159):
        p = fh.select_params(0, n, 1e-15)
        assert p.partitions == 0
        c = np.random.default_rng(n).standard_normal(n)
        assert np.array_equal(fh.schlomilch_fast(p, c), fh.schlomilch_single_partition(p, c)), n


def test_fast_vs_single_and_complex_linearity(fh):
    c = np.random.default_rng(12).standard_normal(700)
    p = fh.select_params(0, 700, 1e-8)
    assert p.partitions >= 1
    assert np.abs(fh.schlomilch_single_partition(p, c) - fh.schlomilch_fast(p, c)).max() <= 20e-8 * np.abs(c).sum()
    g = np.random.default_rng(3)
    cr, ci = g.standard_normal(300), g.standard_normal(300)
    p = fh.select_params(0, 300, 1e-13)
    both = fh.schlomilch_fast(p, cr + 1j * ci)
    split = fh.schlomilch_fast(p, cr) + 1j * fh.schlomilch_fast(p, ci)
    assert np.abs(both - split).max() <= 1e-13 * max(1.0, np.abs(split).max())


def test_instrumented_costs_and_validation(fh):
    p = fh.select_params(0, 2000, 1e-15)
    sc = fh.build_partition(p)
    st = {}
    fh.schlomilch_fast(p, np.random.default_rng(1).standard_normal(2000), stats=st)
    assert st["transform_applications"] == 2 * p.m_terms * (2 * p.partitions + 1)
    assert st["pointwise_evaluations"] == sc.mask_size()
    with pytest.raises(ValueError):
        fh.schlomilch_fast(fh.select_params(0, 100, 1e-8), np.zeros(99))


@pytest.mark.parametrize("n", [64, 256, 1024, 4096])
@pytest.mark.parametrize("eps", [1e-3, 1e-8, 1e-15])
def test_acceptance_schlomilch_grid(fh, n, eps):
    # SPEC acceptance 2
    for nu in (0, 1, 2, 10):
        c = np.random.default_rng(7 * n + nu).standard_normal(n)
        p = fh.select_params(nu, n, eps)
        assert np.abs(fh.schlomilch_fast(p, c) - fh.schlomilch_direct(nu, 0.0, c)).max() <= 10 * eps * np.abs(c).sum()


# -------------------------------------------------------- FB / DHT (SPEC) ---

@pytest.mark.parametrize("n", [64, 256, 1024, 4096])
@pytest.mark.parametrize("eps", [1e-3, 1e-8, 1e-15])
def test_acceptance_fourier_bessel(fh, n, eps):
    # SPEC acceptance 3
    roots = fh.bessel_roots_j0(n)
    for nu in (0, 1):
        c = np.random.default_rng(11 * n + nu).standard_normal(n)
        got = fh.fourier_bessel_eval(nu, c, eps, roots=roots)
        ref = fh.fourier_bessel_direct(nu, c, roots=roots)
        assert np.abs(got - ref).max() <= 10 * eps * np.abs(c).sum()


def test_fourier_bessel_single_column(fh):
    n = 300
    c = np.zeros(n)
    c[0] = 1.0
    roots = fh.bessel_roots_j0(n)
    got = fh.fourier_bessel_eval(0, c, 1e-15, roots=roots)
    assert np.abs(got - fh.bessel_j(0, np.arange(1, n + 1) * roots.roots[0] / n)).max() <= 1e-14


def test_neumann_matvec_high_columns(fh):
    n = 300
    q = fh.select_neumann_params(1e-15)
    c = np.random.default_rng(21).standard_normal(n)
    c[:q.n_split] = 0.0
    roots = fh.bessel_roots_j0(n)
    got = fh.neumann_matvec(0, c, q, 1e-15 / 10, roots=roots)
    ref = fh.fourier_bessel_direct(0, c, roots=roots)
    assert np.abs(got - ref).max() <= 10e-15 * np.abs(c).sum()
    with pytest.raises(AssertionError):
        fh.neumann_matvec(0, np.ones(n), q, 1e-16, roots=roots)


@pytest.mark.parametrize("n", [64, 256, 1024, 2048])
@pytest.mark.parametrize("eps", [1e-3, 1e-8, 1e-15])
def test_acceptance_dht(fh, n, eps):
    # SPEC acceptance 4
    plan = fh.dht_plan(n, eps)
    c = np.random.default_rng(13 * n).standard_normal(n)
    assert np.abs(fh.dht(plan, c) - fh.dht_direct(plan, c)).max() <= 10 * eps * np.abs(c).sum()


def test_dht_edge_cases(fh):
    plan = fh.dht_plan(1, 1e-15)
    r = plan.roots.roots
    assert fh.dht(plan, np.array([1.0]))[0] == pytest.approx(fh.bessel_j(0, float(r[0] * r[0] / r[1])), abs=1e-15)
    plan = fh.dht_plan(300, 1e-8)
    assert np.all(fh.dht(plan, np.zeros(300)) == 0.0)
    with pytest.raises(ValueError):
        fh.dht(plan, np.zeros(299))


def test_self_inverse_trend(fh):
    # SPEC acceptance 7 (shape only): residual decays then grows with N
    res = {}
    for n in (128, 256, 512, 1024, 2048):
        c = np.random.default_rng(n).standard_normal(n)
        res[n] = fh.dht_self_inverse_residual(n, 1e-15, c)
    assert res[256] < res[128] and res[512] < res[256]
    c3 = lambda n: np.arange(1, n + 1, dtype=float) ** -3.0
    vals = [fh.dht_self_inverse_residual(n, 1e-15, c3(n)) for n in (128, 512, 2048)]
    assert max(vals) < 1.0
