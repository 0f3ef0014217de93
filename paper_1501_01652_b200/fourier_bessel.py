"""Fourier-Bessel expansions f(k/N) = sum_n c_n J_nu(k j_{0,n} / N) (drop-in
for fasthankel.fourier_bessel, reference fourier_bessel.py).

j_{0,n} = (n - 1/4) pi + b_n turns the matrix into a perturbed Schlomilch
matrix (gamma = -1/4); the Neumann addition formula plus the Taylor series
of J_s(r b_n), rearranged into 2T+K-2 collected terms, gives one Schlomilch
application per term u with coefficients b^u * c and output scaling r^u.

On the device all collected terms of all vectors form ONE engine
application: the Taylor factor b^u is a fused column pre-multiplier and r^u
a fused row post-multiplier of the same far/near-field kernels (no
separate elementwise passes).  The low columns n <= n_split run through the
direct-sum kernel.
"""

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _device, _lib
from .bessel import bessel_roots_j0
from .schlomilch import MIN_EPS, SchlomilchEngine

__all__ = [
    "NeumannParams",
    "neumann_column_cutoff",
    "taylor_column_cutoff",
    "select_neumann_params",
    "neumann_matvec",
    "fourier_bessel_eval",
    "fourier_bessel_direct",
]


@dataclass(frozen=True)
class NeumannParams:
    """Truncation orders K, T and column split (fourier_bessel.py:38-51)."""

    k_terms: int
    t_terms: int
    p_cut: float
    q_cut: float
    n_split: int


def neumann_column_cutoff(k_terms, eps):
    """p_K(eps) = (e/(16 pi)) (5.2/eps)^(1/K) + 1/4 (fourier_bessel.py:54-57)."""
    return math.e / (16.0 * math.pi) * (5.2 / eps) ** (1.0 / k_terms) + 0.25


def taylor_column_cutoff(t_terms, eps):
    """q_T(eps) = eps^(-1/(2T)) / (16 pi (T!)^(1/T)) + 1/4 (fourier_bessel.py:60-64)."""
    root_fact = math.exp(math.lgamma(t_terms + 1) / t_terms)
    return eps ** (-1.0 / (2.0 * t_terms)) / (16.0 * math.pi * root_fact) + 0.25


def select_neumann_params(eps, margin=1.0):
    """Smallest K, T with margin * p_K, margin * q_T <= 30 (fourier_bessel.py:67-86)."""
    if not 0.0 < eps < 1.0:
        raise ValueError("eps must lie in (0, 1)")
    k_terms = 1
    while margin * neumann_column_cutoff(k_terms, eps) > 30.0:
        k_terms += 1
    t_terms = 1
    while margin * taylor_column_cutoff(t_terms, eps) > 30.0:
        t_terms += 1
    p = neumann_column_cutoff(k_terms, eps)
    q = taylor_column_cutoff(t_terms, eps)
    return NeumannParams(k_terms=k_terms, t_terms=t_terms, p_cut=p, q_cut=q, n_split=int(margin * max(p, q)))


def _reflected(order, weight):
    # J_{-n} = (-1)^n J_n
    if order >= 0:
        return order, weight
    return -order, weight * (-1.0) ** (-order)


def folded_terms(base_orders, u, k_terms, t_terms):
    """Weighted orders of collected term u = 2t + s (fourier_bessel.py:100-123)."""
    terms = {}
    t_lo = max(-(-(u - k_terms + 1) // 2), 0)
    t_hi = min(u // 2, t_terms - 1)
    for t in range(t_lo, t_hi + 1):
        s = u - 2 * t
        coef = (-1.0) ** t * 2.0 ** -u / (math.factorial(t) * math.factorial(u - t))
        if s == 0:
            coef *= 0.5
        for base, base_w in base_orders:
            for order, weight in (_reflected(base - s, base_w * coef),
                                  _reflected(base + s, base_w * coef * (-1.0) ** s)):
                terms[order] = terms.get(order, 0.0) + weight
    return tuple(sorted(terms.items()))


def _order_universe(base_orders, k_terms):
    orders = set()
    for base, _ in base_orders:
        for s in range(k_terms):
            orders.add(abs(base - s))
            orders.add(abs(base + s))
    return orders


def _bump(stats, key, amount=1):
    if stats is not None:
        stats[key] = stats.get(key, 0) + amount


def _direct_apply(row_val, col_val, n_cols, orders, requests, C, F, overwrite=False, r_scale=1.0):
    """Direct rank-1-argument sums on the device (fhtb_direct_apply).  Under
    a work split (_device.sharding) only shard 0 computes them; the others
    contribute zeros (an overwrite leaves zeros)."""
    if not requests:
        return F
    s, _ = _device.shard()
    if s != 0:
        if overwrite:
            F.zero_()
        return F
    from .schlomilch import _pack_requests
    lib = _lib.load()
    ords, ords_p = _lib.i32_array(orders)
    d = _lib.DirectDesc(n_rows=row_val.numel(), row_val=_device.ptr(row_val), n_cols=int(n_cols),
                        col_val=_device.ptr(col_val), n_data_cols=int(n_cols), r_scale=float(r_scale),
                        n_orders=len(orders), orders=ords_p)
    arr, keep = _pack_requests(requests)
    ws_n = lib.fhtb_direct_workspace(d, len(requests), C.shape[0])
    ws = _device.workspace(ws_n)
    flags = _lib.FHTB_OVERWRITE if overwrite else 0
    _lib.check(lib.fhtb_direct_apply(d, arr, len(requests), _device.ptr(C), C.stride(0), C.shape[0],
                                     _device.ptr(F), F.stride(0), flags, _device.ptr(ws), ws.numel(),
                                     _device.stream_ptr()))
    del keep
    return F


def _row_grid(n_grid, first, stride, n_out, dev):
    """r_k = k / n_grid at the output rows k = first + stride*j (fourier_bessel.py:240)."""
    k = first + stride * torch.arange(n_out, dtype=torch.float64, device=dev)
    return k / float(n_grid)


class _JobSet:
    """Collected-term requests of Fourier-Bessel jobs on one grid.

    A job is (base_orders, vector row, outer pre/post factors).  This mirrors
    _fb_jobs_apply (fourier_bessel.py:175-243) including its pruning rule
    (:218-225) and counters, but emits device requests instead of running
    the engine per term.
    """

    def __init__(self, params, n_grid, roots, n_data):
        self.params = params
        self.n_grid = n_grid
        self.n_data = n_data          # columns > n_data hold zeros
        self.roots = roots
        self.n_split = min(params.n_split, n_grid)
        self.low = []                 # direct low-column requests
        self.high = []                # engine requests
        self.high_terms = []

    def add(self, base_orders, vec, bmax, nonzero, stats, prune_eps=None, outer=None):
        """outer: dict(pre_a, pre_a_pow, post_e, post_e_pow) of the DHT row-side term."""
        outer = outer or {}
        if self.n_split > 0:
            r = dict(vec=vec, terms=list(base_orders))
            if outer:
                r.update(pre_a=outer["pre_a"], pre_a_pow=outer["pre_a_pow"], post_e=outer["post_e"],
                         post_e_pow=outer["post_e_pow"])
            self.low.append(r)
        if self.n_grid <= self.n_split or not nonzero:
            return
        top = 2 * self.params.t_terms + self.params.k_terms - 2
        _, b_dev = self.roots.device_arrays()
        for u in range(top):
            terms = folded_terms(base_orders, u, self.params.k_terms, self.params.t_terms)
            if not terms:
                continue
            if prune_eps is not None:
                if not bmax ** u * sum(abs(w) for _, w in terms) >= 0.02 * prune_eps:
                    continue
            r = dict(vec=vec, terms=list(terms), col_lo=self.n_split + 1, pre_b=b_dev, pre_b_pow=u,
                     post_r_pow=u)
            if outer:
                r.update(pre_a=outer["pre_a"], pre_a_pow=outer["pre_a_pow"], post_e=outer["post_e"],
                         post_e_pow=outer["post_e_pow"])
            self.high.append(r)
            self.high_terms.append(terms)
            _bump(stats, "schlomilch_evaluations")

    def low_count(self, stats):
        """pointwise counter of _direct_columns_many (fourier_bessel.py:163-168)."""
        if stats is None or not self.low or self.n_split == 0:
            return
        orders = {o for r in self.low for o, _ in r["terms"]}
        _bump(stats, "pointwise_evaluations", len(orders) * self.n_grid * self.n_split)


def _high_stats(C_rows, n_split, roots):
    """Per-vector (bmax, nonzero) of the high part c[n_split:] (planning only):
    one library reduction (fhtb_coef_stats) and one small copy."""
    _, b_dev = roots.device_arrays()
    _, bm, anyz = _device.coef_stats(C_rows, n_split, b_dev)
    return bm, anyz


def fourier_bessel_eval(nu, c, eps, roots=None, stats=None, prune=False):
    """sum_n c_n J_nu(k j_{0,n}/N), k = 1..N, to O(eps ||c||_1)
    (fourier_bessel.py:312-337).  c may be (N,), (B, N) or a CUDA tensor."""
    if eps < MIN_EPS:
        raise ValueError("eps below 2^-52 is not resolvable in double precision")
    nu = int(nu)
    if nu < 0:
        raise ValueError("nu must be >= 0")
    c_arr = c if isinstance(c, torch.Tensor) else np.asarray(c)
    if c_arr.shape[-1] < 1:
        raise ValueError("need at least one coefficient")
    n = c_arr.shape[-1]
    params = select_neumann_params(eps)
    if roots is None:
        roots = bessel_roots_j0(n)
    inner_eps = eps / (2 * params.t_terms + params.k_terms - 2)
    C, meta = _device.as_real_batch(c_arr)
    F = _device.zeros_like(C)
    _fb_apply(((nu, 1.0),), C, F, n, params, inner_eps, roots, stats, eps if prune else None, meta)
    return _device.from_real_batch(F, meta)


def _fb_apply(base_orders, C, F, n, params, inner_eps, roots, stats, prune_eps, meta):
    support = min(n, roots.n_max)
    if support < n and bool((C[:, support:] != 0).any()):
        raise ValueError("roots table too short for the coefficient support")
    js = _JobSet(params, n, roots, n)
    bmax, nz = _high_stats(C, js.n_split, roots)
    per = 2 if meta["complex"] else 1
    if per == 2:
        # a complex vector is two real rows; the reference plans (and prunes,
        # fourier_bessel.py:208-225) on the complex vector: c_n != 0 if either part is
        bmax = np.repeat(np.maximum(bmax[0::2], bmax[1::2]), 2)
        nz = np.repeat(nz[0::2] | nz[1::2], 2)
    for v in range(C.shape[0]):
        st = stats if v % per == 0 else None
        js.add(base_orders, v, float(bmax[v]), bool(nz[v]), st, prune_eps)
    js.low_count(stats if C.shape[0] else None)
    r_dev, _ = roots.device_arrays()
    if js.low:
        orders = sorted({o for r in js.low for o, _ in r["terms"]})
        rows = _row_grid(n, 1, 1, n, C.device)
        _direct_apply(rows, r_dev, js.n_split, orders, js.low, C, F, r_scale=float(n))
    if js.high:
        uni = sorted(_order_universe(base_orders, params.k_terms))
        eng = SchlomilchEngine(n, -0.25, inner_eps, uni)
        eng.grid().apply(js.high, C, F)
        # both rows of a complex vector carry the same term lists; counted once (rows of even index)
        eng.count([t for t, r in zip(js.high_terms, js.high) if r["vec"] % per == 0], stats)
    return F


def neumann_matvec(nu, c, params, schlomilch_eps, roots=None, stats=None):
    """Truncated-Neumann part only; requires c_n = 0 for n <= n_split
    (fourier_bessel.py:250-289).  Never prunes."""
    c_arr = np.asarray(c)
    assert not np.any(c_arr[: min(params.n_split, c_arr.shape[0])]), "coefficients below n_split must be zero"
    n = c_arr.shape[0]
    if roots is None:
        roots = bessel_roots_j0(n)
    support = min(n, roots.n_max)
    if np.any(c_arr[support:]):
        raise ValueError("roots table too short for the coefficient support")
    C, meta = _device.as_real_batch(c_arr)
    F = _device.zeros_like(C)
    _, b_dev = roots.device_arrays()
    top = 2 * params.t_terms + params.k_terms - 2
    reqs, terms_l = [], []
    for u in range(top):
        terms = folded_terms(((int(nu), 1.0),), u, params.k_terms, params.t_terms)
        if terms:
            for v in range(C.shape[0]):
                reqs.append(dict(vec=v, terms=list(terms), col_lo=1, pre_b=b_dev, pre_b_pow=u, post_r_pow=u))
            terms_l.append(terms)
            _bump(stats, "schlomilch_evaluations")
    if reqs:
        eng = SchlomilchEngine(n, -0.25, schlomilch_eps, _order_universe(((int(nu), 1.0),), params.k_terms))
        eng.grid().apply(reqs, C, F)
        eng.count(terms_l, stats)
    return _device.from_real_batch(F, meta)


def fourier_bessel_direct(nu, c, roots=None):
    """Direct O(N^2) sum (fourier_bessel.py:292-309), on the GPU."""
    c_arr = c if isinstance(c, torch.Tensor) else np.asarray(c)
    n = c_arr.shape[-1]
    if roots is None:
        roots = bessel_roots_j0(n)
    C, meta = _device.as_real_batch(c_arr)
    F = _device.zeros_like(C)
    r_dev, _ = roots.device_arrays()
    rows = _row_grid(n, 1, 1, n, C.device)
    reqs = [dict(vec=v, terms=[(int(nu), 1.0)]) for v in range(C.shape[0])]
    _direct_apply(rows, r_dev, n, [int(nu)], reqs, C, F, r_scale=float(n))
    return _device.from_real_batch(F, meta)
