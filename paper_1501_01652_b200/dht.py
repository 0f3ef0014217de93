"""Order-0 discrete Hankel transform f_k = sum_n c_n J0(j_{0,k} j_{0,n} / j_{0,N+1})
(drop-in for fasthankel.dht, reference dht.py).

Row side: j_{0,k}/j_{0,N+1} = r~_k + e_{k,N}, r~_k = (4k-1)/(4N+3), and the
Neumann/Taylor split again gives collected terms u_out with pre-multiplier
j0^u_out and post-multiplier e^u_out around a Fourier-Bessel evaluation on
the padded uniform grid 4N+3 (dht.py:123-176).  Every (u_out, u_in) term of
every vector is one request of ONE device engine application whose output
rows are exactly the needed padded rows 4k-1 (chirp-z far field on the
row-restricted grid, near field evaluated on those rows only), so the
reference's padding by 3N+3 zeros and its 4x redundant rows are never
materialised.  Rows k <= row_split are summed directly (dht.py:175).
"""

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device, _lib
from .bessel import BesselRootsTable, bessel_j, bessel_roots_j0
from .fourier_bessel import (_bump, _direct_apply, _high_stats, _JobSet, _order_universe, _row_grid,
                             folded_terms, select_neumann_params)
from .schlomilch import MIN_EPS, SchlomilchEngine

__all__ = ["DhtPlan", "dht_plan", "dht", "dht_direct", "dht_self_inverse_residual"]


@dataclass(eq=False)
class DhtPlan:
    """Precomputed state for transforms of one size and accuracy (dht.py:36-55)."""

    n: int
    eps: float
    k_terms: int
    t_terms: int
    p_cut: float
    q_cut: float
    row_split: int
    roots: BesselRootsTable
    weights: np.ndarray
    _shared: object = field(default=None, repr=False)


def dht_plan(n, eps):
    """K, T with 1.01 max(p_K, q_T) <= 30; roots to N+1; v_n = 2/J1(j_{0,n})^2
    (dht.py:58-79)."""
    if eps < MIN_EPS:
        raise ValueError("eps below 2^-52 is not resolvable in double precision")
    if n < 1:
        raise ValueError("n must be >= 1")
    neumann = select_neumann_params(eps, margin=1.01)
    roots = bessel_roots_j0(n + 1)
    r_dev, _ = roots.device_arrays()
    j1 = bessel_j(1, r_dev[:n])
    weights = (2.0 / (j1 * j1)).cpu().numpy()
    return DhtPlan(n=n, eps=eps, k_terms=neumann.k_terms, t_terms=neumann.t_terms, p_cut=neumann.p_cut,
                   q_cut=neumann.q_cut, row_split=neumann.n_split, roots=roots, weights=weights)


def _rows_direct(plan, C, F, k1, stats=None, per=1):
    """Rows 1..k1-1 by direct summation, overwriting F (dht.py:82-94)."""
    n = plan.n
    r_dev, _ = plan.roots.device_arrays()
    scale = (r_dev[: k1 - 1] / r_dev[n]).contiguous()
    reqs = [dict(vec=v, terms=[(0, 1.0)]) for v in range(C.shape[0])]
    Fv = F[:, : k1 - 1]
    out = torch.zeros((C.shape[0], k1 - 1), dtype=torch.float64, device=C.device)
    _direct_apply(scale, r_dev, n, [0], reqs, C, out)
    Fv.copy_(out)
    _bump(stats, "pointwise_evaluations", (C.shape[0] // per) * (k1 - 1) * n)
    return F


def dht_direct(plan, c):
    """O(N^2) direct transform on the GPU (dht.py:97-102)."""
    c_arr = c if isinstance(c, torch.Tensor) else np.asarray(c)
    if c_arr.shape[-1] != plan.n:
        raise ValueError("coefficient length does not match plan.n")
    C, meta = _device.as_real_batch(c_arr)
    F = _device.zeros_like(C)
    _rows_direct(plan, C, F, plan.n + 1)
    return _device.from_real_batch(F, meta)


def _shared(plan):
    """Inner FB params, nested Schlomilch eps and the padded-grid engine
    (dht.py:105-120)."""
    if plan._shared is None:
        fb_params = select_neumann_params(plan.eps)
        r_outer = 2 * plan.t_terms + plan.k_terms - 2
        r_inner = 2 * fb_params.t_terms + fb_params.k_terms - 2
        schl_eps = plan.eps / (r_outer * r_inner)
        base = [(s, 1.0) for s in range(plan.k_terms)]
        universe = _order_universe(base, fb_params.k_terms)
        engine = SchlomilchEngine(4 * plan.n + 3, -0.25, schl_eps, universe)
        n = plan.n
        r_dev, _ = plan.roots.device_arrays()
        ks = torch.arange(1, n + 1, dtype=torch.float64, device=r_dev.device)
        e = (r_dev[:n] / r_dev[n] - (ks - 0.25) / (n + 0.75)).contiguous()
        plan._shared = dict(fb=fb_params, eps=schl_eps, engine=engine, e=e)
    return plan._shared


def dht(plan, c, stats=None):
    """Fast transform, error O(eps ||c||_1) (dht.py:123-176).  c may be
    (N,), (B, N) or a CUDA tensor."""
    c_arr = c if isinstance(c, torch.Tensor) else np.asarray(c)
    n = plan.n
    if c_arr.shape[-1] != n:
        raise ValueError("coefficient length does not match plan.n")
    C, meta = _device.as_real_batch(c_arr)
    per = 2 if meta["complex"] else 1
    F = _device.zeros_like(C)
    split = min(plan.row_split, n)
    if split >= n:
        _rows_direct(plan, C, F, n + 1, stats, per)
        return _device.from_real_batch(F, meta)
    sh = _shared(plan)
    fbp, eng = sh["fb"], sh["engine"]
    n_pad = 4 * n + 3
    r_dev, _ = plan.roots.device_arrays()
    g_max = 1.01 / (8.0 * (split + 0.75) * math.pi)
    js = _JobSet(fbp, n_pad, plan.roots, n)
    support = min(n_pad, plan.roots.n_max)
    if support < n:
        raise ValueError("roots table too short for the coefficient support")
    _, b_dev = plan.roots.device_arrays()
    norm1, bmax, nz = _device.coef_stats(C, js.n_split, b_dev)
    K, T = plan.k_terms, plan.t_terms
    for v in range(C.shape[0]):
        st = stats if v % per == 0 else None
        for u in range(2 * T + K - 2):
            terms = folded_terms(((0, 1.0),), u, K, T)
            if not (terms and norm1[v] > 0.0):
                continue
            if not g_max ** u * sum(abs(w) for _, w in terms) >= 0.02 * plan.eps:
                continue
            _bump(st, "fb_evaluations")
            outer = dict(pre_a=r_dev, pre_a_pow=u, post_e=sh["e"], post_e_pow=u)
            js.add(terms, v, float(bmax[v]), bool(nz[v]), st, plan.eps, outer)
    # low columns n <= n_split of every FB job at the padded rows 4k-1
    if js.low:
        orders = sorted({o for r in js.low for o, _ in r["terms"]})
        rows = _row_grid(n_pad, 3, 4, n, C.device)
        _direct_apply(rows, r_dev, js.n_split, orders, js.low, C, F, r_scale=float(n_pad))
        if stats is not None:
            lo = {o for r in js.low if r["vec"] % per == 0 for o, _ in r["terms"]}
            # reference: one _direct_columns_many over all jobs, each order once
            _bump(stats, "pointwise_evaluations", len(lo) * n_pad * js.n_split)
    if js.high:
        g = eng.grid(row_first=3, row_stride=4, n_out=n, n_data_cols=n)
        g.apply(js.high, C, F)
        eng.count([t for t, r in zip(js.high_terms, js.high) if r["vec"] % per == 0], stats)
    _rows_direct(plan, C, F, split + 1, stats, per)
    return _device.from_real_batch(F, meta)


def dht_self_inverse_residual(n, eps, c, method="fast", plan=None):
    """max |j_{0,N+1}^-2 DHT(D_v DHT(D_v c)) - c| (dht.py:179-194)."""
    c = np.asarray(c)
    if plan is None:
        plan = dht_plan(n, eps)
    apply_fn = dht if method == "fast" else dht_direct
    if np.iscomplexobj(c) or c.ndim != 1:
        y = apply_fn(plan, plan.weights * c)
        y = apply_fn(plan, plan.weights * y)
        return float(np.max(np.abs(y / plan.roots.roots[n] ** 2 - c)))
    # the N-length scalings and the residual run in the library (device-resident throughout)
    C = _device.to_dev_f64(c).reshape(1, -1)
    w = plan.__dict__.get("_w_dev")
    if w is None or w.device != C.device:
        w = _device.to_dev_f64(plan.weights)
        object.__setattr__(plan, "_w_dev", w)
    t = torch.empty_like(C)
    for src in (C, None):
        a = C if src is not None else y
        _lib.call("fhtb_mul_rows", _device.ptr(t), t.stride(0), _device.ptr(a), a.stride(0), _device.ptr(w), 1.0,
                  n, 1, _device.stream_ptr())
        y = apply_fn(plan, t)
    res = ctypes.c_double(0.0)
    _lib.call("fhtb_max_abs_diff", _device.ptr(y), 1.0 / float(plan.roots.roots[n]) ** 2, _device.ptr(C), n,
              ctypes.byref(res), _device.stream_ptr())
    return float(res.value)
