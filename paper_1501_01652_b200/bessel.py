"""Bessel functions, truncation cutoffs and roots of J0 (drop-in for
fasthankel.bessel, reference bessel.py).

Scalar planning formulas (coefficients, cutoffs, error bounds) run on the
host; every array evaluation of J_nu and the root finder run in
libfhtb200.so on the GPU.
"""

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _device, _lib

__all__ = [
    "asy_coeff",
    "asy_coeffs",
    "hankel_asy_eval",
    "asy_error_bound",
    "asy_cutoff",
    "taylor_eval",
    "taylor_cutoff",
    "neumann_radius",
    "bessel_j",
    "BesselRootsTable",
    "bessel_roots_j0",
]

_EPS = 2.0 ** -52
_TAYLOR_TERMS = 10
_ASY_TERMS = 10
_SQRT_2_OVER_PI = math.sqrt(2.0 / math.pi)


def asy_coeffs(nu, count):
    """a_0(nu)..a_{count-1}(nu) by the ratio recurrence
    a_m = a_{m-1} (4 nu^2 - (2m-1)^2) / (8m), a_0 = 1 (bessel.py:45-58)."""
    a = np.empty(count)
    a[0] = 1.0
    q = 4.0 * nu * nu
    for m in range(1, count):
        a[m] = a[m - 1] * (q - (2 * m - 1) ** 2) / (8.0 * m)
    return a


def asy_coeff(nu, m):
    """a_m(nu) (bessel.py:61-69)."""
    if nu < 0 or m < 0:
        raise ValueError("asy_coeff requires nu >= 0 and m >= 0")
    return float(asy_coeffs(nu, m + 1)[m])


def asy_error_bound(nu, m_terms, z):
    """sqrt(2/(pi z)) (|a_2M| / z^2M + |a_2M+1| / z^(2M+1)) (bessel.py:94-106)."""
    z = np.asarray(z, dtype=float)
    a = asy_coeffs(nu, 2 * m_terms + 2)
    out = _SQRT_2_OVER_PI / np.sqrt(z) * (abs(a[2 * m_terms]) + abs(a[2 * m_terms + 1]) / z) / z ** (2 * m_terms)
    return out if out.ndim else float(out)


def asy_cutoff(nu, m_terms, eps):
    """s_{nu,M}(eps): four fixed-point iterations from s = 1 (bessel.py:109-130)."""
    if not 0.0 < eps < 1.0:
        raise ValueError("eps must lie in (0, 1)")
    a = asy_coeffs(nu, 2 * m_terms + 2)
    a0, a1 = abs(a[2 * m_terms]), abs(a[2 * m_terms + 1])
    s = 1.0
    c = math.sqrt(2.0) / (math.sqrt(math.pi) * eps)
    for _ in range(4):
        s = (c * (a0 + a1 / s)) ** (1.0 / (2 * m_terms + 0.5))
    return s


def taylor_cutoff(nu, n_terms, eps):
    """t_{nu,T}(eps) (bessel.py:149-168)."""
    if not 0.0 < eps < 1.0:
        raise ValueError("eps must lie in (0, 1)")
    e = 2 * n_terms + nu
    log_t = (e * math.log(2.0) + math.lgamma(n_terms + nu + 1) + math.lgamma(n_terms + 1)
             + math.log(eps)) / e
    return math.exp(log_t)


def neumann_radius(k_terms, eps):
    """2/e (eps/5.2)^(1/K) (bessel.py:171-177)."""
    if not 0.0 < eps < 1.0:
        raise ValueError("eps must lie in (0, 1)")
    return 2.0 / math.e * (eps / 5.2) ** (1.0 / k_terms)


def _elementwise(fn_name, args, z):
    """Run an element-wise device kernel on array-like / tensor z."""
    _device.ensure_init()
    is_t = isinstance(z, torch.Tensor)
    zt = _device.to_dev_f64(z)
    out = torch.empty_like(zt)
    if zt.numel():
        _lib.call(fn_name, *args, _device.ptr(zt), zt.numel(), _device.ptr(out), _device.stream_ptr())
    if is_t:
        return out
    res = out.cpu().numpy()
    return res if res.ndim else float(res)


def hankel_asy_eval(nu, m_terms, z):
    """First 2*m_terms terms of the Hankel expansion of J_nu(z) (bessel.py:72-91)."""
    return _elementwise("fhtb_hankel_asy_eval", (int(nu), int(m_terms)), z)


def taylor_eval(nu, n_terms, z):
    """First n_terms terms of the Taylor series of J_nu (bessel.py:133-146)."""
    return _elementwise("fhtb_taylor_eval", (int(nu), int(n_terms)), z)


def bessel_j(nu, z):
    """J_nu(z) for integer nu >= 0 and z >= 0 (bessel.py:232-260)."""
    nu = int(nu)
    if nu < 0:
        raise ValueError("bessel_j requires nu >= 0; use J_{-n} = (-1)^n J_n")
    if isinstance(z, torch.Tensor):
        if bool((z < 0).any()):
            raise ValueError("bessel_j requires z >= 0")
    else:
        arr = np.asarray(z, dtype=float)
        if np.any(arr < 0.0):
            raise ValueError("bessel_j requires z >= 0")
        z = arr
    return _elementwise("fhtb_bessel_j", (nu,), z)


@dataclass(frozen=True)
class BesselRootsTable:
    """First n_max positive roots of J0, j_{0,n} = (n - 1/4) pi + b_n
    (bessel.py:270-292).  Host arrays are read-only; device copies are
    cached for the Fourier-Bessel / DHT engines."""

    n_max: int
    roots: np.ndarray
    perturbations: np.ndarray

    def ratio_perturbation(self, k, n):
        """e_{k,n} = j_{0,k} / j_{0,n+1} - (k - 1/4)/(n + 3/4) (bessel.py:283-292)."""
        if n + 1 > self.n_max:
            raise ValueError("table holds %d roots; need %d" % (self.n_max, n + 1))
        k = np.asarray(k)
        num = self.roots[k - 1] / self.roots[n]
        return num - (k - 0.25) / (n + 0.75)

    def device_arrays(self):
        """(roots, perturbations) as float64 CUDA tensors (cached)."""
        cache = self.__dict__.get("_dev")
        dev = _device.device()
        if cache is None or cache[0].device != dev:
            cache = (torch.from_numpy(np.array(self.roots)).to(dev),
                     torch.from_numpy(np.array(self.perturbations)).to(dev))
            object.__setattr__(self, "_dev", cache)
        return cache


def bessel_roots_j0(count):
    """First `count` roots of J0 by Newton from (n - 1/4) pi on the GPU
    (bessel.py:295-321); RuntimeError if a residual exceeds 1e-13, the
    reference's bound -- relaxed to 2 ulp(root)|J1(root)| only for roots so
    large (beyond ~2e6, counts ~2^20) that fp64 rounding of the root itself
    leaves |J0| above 1e-13 (the reference raises there)."""
    if count < 1:
        raise ValueError("count must be >= 1")
    dev = _device.ensure_init()
    roots = torch.empty(count, dtype=torch.float64, device=dev)
    pert = torch.empty_like(roots)
    import ctypes
    res = ctypes.c_double(0.0)
    code = _lib.load().fhtb_roots_j0(count, _device.ptr(roots), _device.ptr(pert), ctypes.byref(res),
                                     _device.stream_ptr())
    if code == _lib.FHTB_ECONVERGE:
        raise RuntimeError("Newton failed to converge on J0 roots (residual %.3e)" % res.value)
    _lib.check(code)
    r = roots.cpu().numpy()
    b = pert.cpu().numpy()
    r.flags.writeable = False
    b.flags.writeable = False
    t = BesselRootsTable(n_max=count, roots=r, perturbations=b)
    object.__setattr__(t, "_dev", (roots, pert))
    return t
