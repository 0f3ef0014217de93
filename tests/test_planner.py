"""Host planner of the drop-in package (CPU only): Table-4 parameters,
partitions, Neumann/Taylor truncations, folded terms, pruning inputs --
pinned bit for bit against the reference (golden.json) and the paper's
known answers (Tables 1-4, SPEC.md examples)."""

import math

import numpy as np
import pytest

import paper_1501_01652_b200 as fh
from paper_1501_01652_b200.fourier_bessel import _order_universe, folded_terms
from paper_1501_01652_b200.schlomilch import SchlomilchEngine, _select_params
from oracle import fht_oracle as O


def test_params_and_partitions_match_reference(golden):
    meta, _ = golden
    for rec in meta["params"]:
        p = _select_params(rec["nu"], rec["n"], rec["eps"], rec["gamma"])
        assert (p.m_terms, p.s, p.alpha, p.beta, p.partitions) == (
            rec["m"], rec["s"], rec["alpha"], rec["beta"], rec["P"])
        sc = fh.build_partition(p)
        assert [list(map(list, b)) for b in sc.blocks] == rec["blocks"]
        assert [list(s) for s in sc.mask_segments] == rec["segments"]
        assert sc.row_min == rec["row_min"] and sc.mask_size() == rec["mask"]


def test_neumann_params_match_reference(golden):
    meta, _ = golden
    for rec in meta["neumann"]:
        q = fh.select_neumann_params(rec["eps"], rec["margin"])
        assert (q.k_terms, q.t_terms, q.p_cut, q.q_cut, q.n_split) == (
            rec["K"], rec["T"], rec["p"], rec["q"], rec["n_split"])


def test_engine_params_match_reference(golden):
    meta, _ = golden
    for rec in meta["engine"]:
        eng = SchlomilchEngine(rec["n"], rec["gamma"], rec["eps"], rec["orders"])
        assert (eng.params.m_terms, eng.params.s, eng.params.partitions) == (rec["m"], rec["s"], rec["P"])


# ---- known answers (restating the reference's planner tests) ---------------

def test_m_terms_known_values():
    assert fh.select_params(0, 1000, 1e-15).m_terms == 10
    assert fh.select_params(0, 1000, 1e-3).m_terms == 3     # floor(2.07) clamped to 3
    assert fh.select_params(0, 1000, 1e-8).m_terms == 5


def test_table4_formulas():
    p = fh.select_params(0, 5000, 1e-15)
    assert p.beta == pytest.approx(3.0 / math.log(5000), rel=1e-12)
    assert p.s == pytest.approx(17.8, abs=0.1)                # PAPER Table 1, s_{0,10}
    assert p.alpha == pytest.approx(math.sqrt(p.s / math.pi), rel=1e-12)


def test_single_partition_up_to_158():
    assert all(fh.select_params(0, n, 1e-15).partitions == 0 for n in range(1, 159))
    assert fh.select_params(0, 159, 1e-15).partitions >= 1


def test_select_params_rejects_bad_arguments():
    for args, kw in (((0, 100, 2.0 ** -53), {}), ((0, 100, 1.5), {}), ((-1, 100, 1e-8), {}),
                     ((0, 100, 1e-8), {"gamma": -1.0})):
        with pytest.raises(ValueError):
            fh.select_params(*args, **kw)


@pytest.mark.parametrize("n", [1, 2, 5, 10, 30, 158, 159, 200, 400, 600])
@pytest.mark.parametrize("eps", [1e-3, 1e-8, 1e-15])
def test_partition_covers_square_once(n, eps):
    sc = fh.build_partition(_select_params(0, n, eps, 0.0))
    cover = np.zeros((n, n), dtype=int)
    for (r0, r1), (c0, c1) in sc.blocks:
        cover[r0 - 1:r1 - 1, c0 - 1:c1 - 1] += 1
    for r0, r1, ce in sc.mask_segments:
        cover[r0 - 1:r1 - 1, :ce - 1] += 1
    assert np.all(cover == 1)


@pytest.mark.parametrize("n", [200, 1024, 5000, 100000, 2 ** 20])
@pytest.mark.parametrize("eps", [1e-3, 1e-8, 1e-15])
def test_blocks_respect_asymptotic_cutoff(n, eps):
    p = _select_params(0, n, eps, 0.0)
    for (r0, r1), (c0, c1) in fh.build_partition(p).blocks:
        if r1 > r0 and c1 > c0:
            assert r0 * c0 >= p.alpha ** 2 * n * (1.0 - 1e-12)


def test_paper_table_values():
    # Table 1 (s_{nu,M}(1e-15)), Table 2 (t_{nu,T}(1e-15)), Table 3 (Neumann radius)
    assert fh.asy_cutoff(0, 10, 1e-15) == pytest.approx(17.8, abs=0.1)
    assert fh.asy_cutoff(2, 6, 1e-15) == pytest.approx(30.8, abs=0.1)
    assert fh.asy_cutoff(10, 5, 1e-15) == pytest.approx(149.0, abs=0.5)
    assert fh.taylor_cutoff(0, 5, 1e-15) == pytest.approx(0.165, abs=0.005)
    assert fh.taylor_cutoff(10, 1, 1e-15) == pytest.approx(0.484, abs=0.005)
    assert fh.taylor_cutoff(1, 9, 1e-15) == pytest.approx(1.411, abs=0.005)
    assert fh.neumann_radius(10, 1e-15) == pytest.approx(0.020, rel=0.10)
    assert fh.neumann_radius(3, 1e-15) == pytest.approx(4e-6, rel=0.10)
    for nu in (0, 1, 2, 10):
        for m in range(3, 13):
            for eps in (1e-3, 1e-8, 1e-15):
                assert fh.asy_error_bound(nu, m, fh.asy_cutoff(nu, m, eps)) <= (1.0 + 1e-3) * eps


def test_asy_coefficients():
    assert fh.asy_coeff(0, 0) == 1.0 and fh.asy_coeff(0, 1) == -0.125
    assert fh.asy_coeff(0, 2) == 0.0703125
    for nu in (0, 1, 2, 5, 10):
        for m in range(1, 9):
            num = 1.0
            for i in range(1, m + 1):
                num *= 4.0 * nu * nu - (2 * i - 1) ** 2
            assert fh.asy_coeff(nu, m) == pytest.approx(num / (math.factorial(m) * 8.0 ** m), rel=1e-13)
    with pytest.raises(ValueError):
        fh.asy_coeff(-1, 2)


def test_neumann_known_answers():
    q = fh.select_neumann_params(1e-15)
    assert (q.k_terms, q.t_terms, q.n_split) == (6, 3, 22)                  # PAPER 5, SPEC fourier_bessel
    assert q.p_cut == pytest.approx(22.7, abs=0.1) and q.q_cut == pytest.approx(3.7, abs=0.1)
    assert 2 * q.t_terms + q.k_terms - 2 == 10                              # PAPER 5.1: 33 -> 10
    assert fh.select_neumann_params(1e-15, margin=1.01).n_split == 22        # DHT row_split
    with pytest.raises(ValueError):
        fh.select_neumann_params(0.0)


def test_folded_terms_match_oracle():
    for base in (((0, 1.0),), ((3, 1.0),), ((0, 1.0), (2, -0.5))):
        for K, T in ((6, 3), (5, 2), (1, 1)):
            for u in range(2 * T + K - 1):
                assert folded_terms(base, u, K, T) == O.fold(base, u, K, T)
            assert _order_universe(base, K) == O.universe(base, K)


def test_dht_plan_validation_is_cpu_side():
    with pytest.raises(ValueError):
        fh.dht_plan(10, 2.0 ** -53)
    with pytest.raises(ValueError):
        fh.dht_plan(0, 1e-8)
    with pytest.raises(ValueError):
        fh.fourier_bessel_eval(0, np.ones(4), 2.0 ** -53)
    with pytest.raises(ValueError):
        fh.fourier_bessel_eval(-1, np.ones(4), 1e-8)


def test_trig_plan_validation():
    with pytest.raises(ValueError):
        fh.make_plan(1, fh.DCT1)
    with pytest.raises(ValueError):
        fh.make_plan(0, fh.DST1)
    with pytest.raises(ValueError):
        fh.make_plan(4, "dct2")
    with pytest.raises(ValueError):
        fh.apply(fh.make_plan(4, fh.DCT1), np.zeros(5))


def test_bessel_argument_validation():
    with pytest.raises(ValueError):
        fh.bessel_j(-1, 1.0)
    with pytest.raises(ValueError):
        fh.bessel_j(0, -0.5)
    with pytest.raises(ValueError):
        fh.bessel_roots_j0(0)


def test_public_surface_matches_reference():
    names = set(fh.__all__)
    expected = {"BesselRootsTable", "asy_coeff", "asy_coeffs", "asy_cutoff", "asy_error_bound", "bessel_j",
                "bessel_roots_j0", "hankel_asy_eval", "neumann_radius", "taylor_cutoff", "taylor_eval",
                "DCT1", "DST1", "TransformPlan", "apply", "make_plan", "SchlomilchParams", "PartitionScheme",
                "select_params", "build_partition", "schlomilch_direct", "asy_block_apply",
                "schlomilch_single_partition", "schlomilch_fast", "NeumannParams", "neumann_column_cutoff",
                "taylor_column_cutoff", "select_neumann_params", "neumann_matvec", "fourier_bessel_eval",
                "fourier_bessel_direct", "DhtPlan", "dht_plan", "dht", "dht_direct",
                "dht_self_inverse_residual", "VectorFileError", "read_vector", "write_vector", "__version__"}
    assert expected <= names
    for n in expected - {"__version__"}:
        assert hasattr(fh, n)


def test_order_windows_cover_universe_once():
    """Engine universes wider than one device grid (16 orders inside 16
    consecutive orders) are split greedily; every order lands in exactly one
    window and each window satisfies both limits."""
    from paper_1501_01652_b200.schlomilch import _MAX_UNIVERSE, _order_windows
    for orders in ([0], list(range(11)), list(range(16)), list(range(17)), [0, 15], [0, 16], [3, 70, 5, 4, 64, 100],
                   list(range(0, 40, 2)) + [70], list(range(55, 66)), [1023, 0]):
        wins = _order_windows(orders)
        flat = [o for w in wins for o in w]
        assert sorted(flat) == sorted(set(orders))
        assert len(flat) == len(set(flat))
        for w in wins:
            assert 1 <= len(w) <= _MAX_UNIVERSE and w[-1] - w[0] < _MAX_UNIVERSE and w == sorted(w)
    assert _order_windows(list(range(16))) == [list(range(16))]
    assert len(_order_windows(list(range(17)))) == 2
