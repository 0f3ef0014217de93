"""CPU oracle for the fast Hankel transform hot path (arXiv 1501.01652).

TEST INFRASTRUCTURE ONLY.  This module is a NumPy restatement of the
reference `fasthankel` package's algorithm, written from the paper and the
reference's observable behaviour, and used solely as the *checker*:

  * tests/ (parity tests, golden-vector pins),
  * __graft_entry__.smoke() (one small GPU-vs-oracle comparison),
  * bench.py's `cpu_baseline` leg and `--impl reference` arm (the timed CPU
    implementation of the path, since the Python reference cannot travel to
    the GPU box).

The product package `paper_1501_01652_b200` never imports this file; its
numerical work runs in the CUDA library and fails loudly when that library
is missing.

Every routine cites the reference location (file:line under
/root/reference/pkg/src/fasthankel/) whose behaviour it restates.  Results
are pinned against golden vectors produced by the reference itself
(tests/golden/make_golden.py -> tests/golden/*.npz).
"""

import math

import numpy as np

U = 2.0 ** -52                     # unit roundoff used by the dispatch cutoffs
MIN_EPS = 2.0 ** -52               # schlomilch.py:41
PT_TERMS = 10                      # bessel.py:39 (_TAYLOR_TERMS)
PA_TERMS = 10                      # bessel.py:40 (_ASY_TERMS)
NEAR_ROWS = 2048                   # schlomilch.py:48 (_ROW_CHUNK)
NEAR_COLS = 512                    # schlomilch.py:47 (_COL_CHUNK)
FFT_ROWS = 264                     # schlomilch.py:420 (SchlomilchEngine._FFT_ROWS)
SQ2PI = math.sqrt(2.0 / math.pi)


# ===========================================================================
# L1: Bessel-function kernels                          (bessel.py:45-321)
# ===========================================================================

def hankel_coeffs(nu, count):
    """a_0..a_{count-1} of the Hankel expansion by the ratio recurrence
    a_m = a_{m-1} (4 nu^2 - (2m-1)^2) / (8m)  (bessel.py:45-58)."""
    out = np.ones(count)
    q = 4.0 * nu * nu
    for m in range(1, count):
        out[m] = out[m - 1] * (q - (2 * m - 1) ** 2) / (8.0 * m)
    return out


def hankel_series(nu, mt, z):
    """2*mt-term Hankel asymptotic value of J_nu(z), Horner in z^-2
    (bessel.py:72-91)."""
    z = np.asarray(z, dtype=float)
    a = hankel_coeffs(nu, 2 * mt)
    w = 1.0 / (z * z)
    top = (-1.0) ** (mt - 1)
    pe = np.full_like(z, a[2 * mt - 2] * top)
    po = np.full_like(z, a[2 * mt - 1] * top)
    for m in range(mt - 2, -1, -1):
        sg = (-1.0) ** m
        pe = pe * w + sg * a[2 * m]
        po = po * w + sg * a[2 * m + 1]
    phase = z - (2 * nu + 1) * (math.pi / 4.0)
    val = SQ2PI / np.sqrt(z) * (np.cos(phase) * pe - np.sin(phase) * po / z)
    return val if val.ndim else float(val)


def hankel_bound(nu, mt, z):
    """First-neglected-pair error bound of hankel_series (bessel.py:94-106)."""
    z = np.asarray(z, dtype=float)
    a = hankel_coeffs(nu, 2 * mt + 2)
    val = SQ2PI / np.sqrt(z) * (abs(a[2 * mt]) + abs(a[2 * mt + 1]) / z) / z ** (2 * mt)
    return val if val.ndim else float(val)


def hankel_cutoff(nu, mt, eps):
    """s_{nu,M}(eps): four fixed-point sweeps from s=1 (bessel.py:109-130)."""
    if not 0.0 < eps < 1.0:
        raise ValueError("eps must lie in (0, 1)")
    a = hankel_coeffs(nu, 2 * mt + 2)
    e0, e1 = abs(a[2 * mt]), abs(a[2 * mt + 1])
    k = math.sqrt(2.0) / (math.sqrt(math.pi) * eps)
    s = 1.0
    for _ in range(4):
        s = (k * (e0 + e1 / s)) ** (1.0 / (2 * mt + 0.5))
    return s


def taylor_series(nu, nt, z):
    """nt-term Maclaurin series of J_nu (bessel.py:133-146)."""
    z = np.asarray(z, dtype=float)
    h = 0.5 * z
    term = h ** nu / math.gamma(nu + 1)
    acc = term.copy() if term.ndim else np.asarray(term, dtype=float)
    h2 = h * h
    for t in range(1, nt):
        term = -term * h2 / (t * (t + nu))
        acc = acc + term
    return acc if acc.ndim else float(acc)


def taylor_cutoff(nu, nt, eps):
    """t_{nu,T}(eps) (bessel.py:149-168)."""
    if not 0.0 < eps < 1.0:
        raise ValueError("eps must lie in (0, 1)")
    e = 2 * nt + nu
    lg = (e * math.log(2.0) + math.lgamma(nt + nu + 1) + math.lgamma(nt + 1)
          + math.log(eps)) / e
    return math.exp(lg)


def neumann_radius(kt, eps):
    """2/e (eps/5.2)^(1/K) (bessel.py:171-177)."""
    if not 0.0 < eps < 1.0:
        raise ValueError("eps must lie in (0, 1)")
    return 2.0 / math.e * (eps / 5.2) ** (1.0 / kt)


_CUTS = {}


def dispatch_cutoffs(nu):
    """(taylor_cutoff(nu,10,u), hankel_cutoff(nu,10,u)) (bessel.py:183-194)."""
    if nu not in _CUTS:
        _CUTS[nu] = (taylor_cutoff(nu, PT_TERMS, U), hankel_cutoff(nu, PA_TERMS, U))
    return _CUTS[nu]


def miller(nu, z):
    """Backward recurrence with J0 + 2 sum J_2k = 1 (bessel.py:197-229).

    The start order uses the largest argument of the whole array, as the
    reference does (bessel.py:206-207).
    """
    top = max(float(nu), float(z.max()))
    kstart = int(math.ceil(top + 10.0 + 11.0 * top ** (1.0 / 3.0)))
    hi = np.zeros_like(z)
    cur = np.full_like(z, 1e-30)
    nrm = np.zeros_like(z)
    cap = np.zeros_like(z)
    rz = 1.0 / z
    for k in range(kstart, 0, -1):
        lo = (2.0 * k) * rz * cur - hi
        hi, cur = cur, lo
        order = k - 1
        if order == nu:
            cap = cur.copy()
        if order % 2 == 0:
            nrm = nrm + (cur if order == 0 else 2.0 * cur)
        huge = np.abs(cur) > 1e250
        if huge.any():
            f = np.where(huge, 1e-250, 1.0)
            cur, hi, nrm, cap = cur * f, hi * f, nrm * f, cap * f
    return cap / nrm


def besselj(nu, z):
    """J_nu(z), integer nu >= 0, z >= 0 (bessel.py:232-260)."""
    nu = int(nu)
    if nu < 0:
        raise ValueError("bessel_j requires nu >= 0")
    zz = np.asarray(z, dtype=float)
    if np.any(zz < 0.0):
        raise ValueError("bessel_j requires z >= 0")
    lo, hi = dispatch_cutoffs(nu)
    flat = np.atleast_1d(zz).ravel()
    res = np.empty_like(flat)
    a = flat <= lo
    b = flat >= hi
    c = ~(a | b)
    if a.any():
        res[a] = taylor_series(nu, PT_TERMS, flat[a])
    if b.any():
        res[b] = hankel_series(nu, PA_TERMS, flat[b])
    if c.any():
        res[c] = miller(nu, flat[c])
    if zz.ndim == 0:
        return float(res[0])
    return res.reshape(zz.shape)


def j0_roots(count):
    """(roots, perturbations) of J0 by Newton from (n-1/4)pi
    (bessel.py:295-321)."""
    if count < 1:
        raise ValueError("count must be >= 1")
    grid = (np.arange(1, count + 1, dtype=float) - 0.25) * math.pi
    x = grid.copy()
    for _ in range(20):
        d = besselj(0, x) / besselj(1, x)
        x = x + d
        if np.max(np.abs(d)) <= 4.0 * U * x[-1]:
            break
    if np.max(np.abs(besselj(0, x))) > 1e-13:
        raise RuntimeError("Newton failed on J0 roots")
    return x, x - grid


# ===========================================================================
# L1: DCT-I / DST-I                                           (trig.py:38-92)
# ===========================================================================

def dct1(v):
    """C[k,n] = cos(k n pi/(L-1)) along the last axis (trig.py:59-66)."""
    v = np.asarray(v)
    n = v.shape[-1]
    w = np.full(n, 0.5)
    w[0] = w[-1] = 1.0
    u = v * w
    ext = np.concatenate([u, u[..., -2:0:-1]], axis=-1)
    if np.iscomplexobj(v):
        return np.fft.fft(ext, axis=-1)[..., :n]
    return np.fft.rfft(ext, axis=-1).real[..., :n]


def dst1(v):
    """S[k,n] = sin((k+1)(n+1) pi/(L+1)) along the last axis (trig.py:69-77)."""
    v = np.asarray(v)
    n = v.shape[-1]
    ext = np.zeros(v.shape[:-1] + (2 * n + 2,), dtype=v.dtype)
    ext[..., 1:n + 1] = v
    ext[..., n + 2:] = -v[..., ::-1]
    if np.iscomplexobj(v):
        return 0.5j * np.fft.fft(ext, axis=-1)[..., 1:n + 1]
    return -0.5 * np.fft.rfft(ext, axis=-1).imag[..., 1:n + 1]


# ===========================================================================
# L2: Schlomilch planner, near field and far field       (schlomilch.py)
# ===========================================================================

def m_terms(eps):
    """M = max(floor(0.3 ln(1/eps)), 3) (schlomilch.py:72-73)."""
    return max(int(0.3 * math.log(1.0 / eps)), 3)


def plan_params(nu, n, eps, gamma=0.0, s=None, public=True):
    """Table-4 parameters as a dict (schlomilch.py:76-112).  public=True adds
    the eps >= 2^-52 check of select_params."""
    if public and eps < MIN_EPS:
        raise ValueError("eps below 2^-52")
    if not 0.0 < eps < 1.0:
        raise ValueError("eps must lie in (0, 1)")
    if n < 1 or nu < 0 or gamma <= -1.0:
        raise ValueError("bad arguments")
    m = m_terms(eps)
    if s is None:
        s = hankel_cutoff(nu, m, eps)
    alpha = math.sqrt(s / math.pi)
    beta = 1.0 if n <= 20 else min(3.0 / math.log(n), 1.0)
    x = 30.0 / (alpha * math.sqrt(n))
    p = 0 if (x >= 1.0 or beta >= 1.0) else max(math.ceil(math.log(x) / math.log(beta)), 0)
    return dict(eps=eps, nu=nu, gamma=gamma, n=n, m_terms=m, s=s, alpha=alpha,
                beta=beta, partitions=p)


def partition(par, levels=None):
    """(blocks, segments, row_min) of the index square (schlomilch.py:139-170)."""
    n = par["n"]
    P = par["partitions"] if levels is None else levels
    rn = math.sqrt(n)
    lo = [min(math.ceil(par["alpha"] * par["beta"] ** p * rn), n + 1) for p in range(P + 1)]
    hi = [None] + [min(math.ceil(par["alpha"] * par["beta"] ** -p * rn), n + 1)
                   for p in range(1, P + 1)]
    blocks = [((lo[0], n + 1), (lo[0], n + 1))]
    for p in range(1, P + 1):
        blocks += [((lo[p], lo[p - 1]), (hi[p], n + 1)),
                   ((hi[p], n + 1), (lo[p], lo[p - 1]))]
    segs = []
    bands = [(1, lo[P], n + 1)]
    bands += [(lo[p], lo[p - 1], hi[p]) for p in range(P, 0, -1)]
    prev = lo[0]
    for p in range(1, P + 1):
        bands.append((prev, hi[p], lo[p - 1]))
        prev = hi[p]
    bands.append((prev, n + 1, lo[P]))
    for r0, r1, ce in bands:
        if r1 > r0 and ce > 1:
            segs.append((r0, r1, ce))
    return blocks, segs, lo[P]


def mask_size(segs):
    return sum((r1 - r0) * (ce - 1) for r0, r1, ce in segs)


def _bump(stats, key, v):
    if stats is not None:
        stats[key] = stats.get(key, 0) + v


def near_field(order_weights, gamma, n, segs, c, out, stats=None, kahan=True):
    """Pointwise border evaluation, 2048x512 tiles (schlomilch.py:193-220);
    kahan=False gives the engine's plain accumulation (schlomilch.py:504-531)."""
    h = math.pi / n
    for r0, r1, ce in segs:
        nc = ce - 1
        if r1 <= r0 or nc <= 0:
            continue
        fr = (np.arange(1, ce, dtype=float) + gamma) * h
        cc = c[:nc]
        for a in range(r0, r1, NEAR_ROWS):
            b = min(a + NEAR_ROWS, r1)
            ks = np.arange(a, b, dtype=float)
            tot = np.zeros(b - a, dtype=out.dtype)
            cmp_ = np.zeros_like(tot)
            for j0 in range(0, nc, NEAR_COLS):
                j1 = min(j0 + NEAR_COLS, nc)
                z = np.multiply.outer(ks, fr[j0:j1])
                g = None
                for o, w in order_weights:
                    t = w * besselj(o, z)
                    g = t if g is None else g + t
                part = g @ cc[j0:j1]
                if kahan:
                    y = part - cmp_
                    t = tot + y
                    cmp_ = (t - tot) - y
                    tot = t
                else:
                    tot = tot + part
                _bump(stats, "pointwise_evaluations", z.size * len(order_weights))
            out[a - 1:b - 1] += tot


def direct(nu, gamma, c):
    """O(N^2) Schlomilch sum (schlomilch.py:223-229)."""
    c = np.asarray(c)
    n = c.shape[0]
    out = np.zeros(n, dtype=np.result_type(c.dtype, np.float64))
    near_field(((int(nu), 1.0),), gamma, n, ((1, n + 1, n + 1),), c, out)
    return out


class FarField:
    """Diagonal-scaled DCT/DST machinery of one grid (schlomilch.py:236-329)."""

    def __init__(self, par, row_min):
        n, m = par["n"], par["m_terms"]
        self.n, self.m, self.row_min, self.par = n, m, row_min, par
        om = (np.arange(1, n + 1, dtype=float) + par["gamma"]) * math.pi
        cw = np.empty((2 * m, n))
        cw[0] = 1.0 / np.sqrt(om)
        for i in range(1, 2 * m):
            cw[i] = cw[i - 1] / om
        self.cw = cw
        ks = np.arange(row_min, n + 1, dtype=float)
        self.nrows = ks.shape[0]
        ir = n / ks if self.nrows else ks
        rw = np.empty((2 * m, self.nrows))
        if self.nrows:
            rw[0] = np.sqrt(ir)
            for i in range(1, 2 * m):
                rw[i] = rw[i - 1] * ir
        self.rw = rw
        self.theta = -par["gamma"] * ks * (math.pi / n)
        self.cache = {}

    def _diag(self, o):
        if o not in self.cache:
            ph = self.theta + (2 * o + 1) * (math.pi / 4.0)
            self.cache[o] = (np.cos(ph), np.sin(ph), hankel_coeffs(o, 2 * self.m))
        return self.cache[o]

    def weights(self, order_weights):
        """A, B (2M x nrows) of the row-side combination (schlomilch.py:280-299)."""
        m = self.m
        A = np.zeros((2 * m, self.nrows))
        B = np.zeros((2 * m, self.nrows))
        for o, w in order_weights:
            cd, sd, a = self._diag(o)
            for q in range(m):
                lam = w * SQ2PI * (-1.0) ** q
                A[2 * q] += (lam * a[2 * q]) * cd
                B[2 * q] += (lam * a[2 * q]) * sd
                A[2 * q + 1] += (lam * a[2 * q + 1]) * sd
                B[2 * q + 1] -= (lam * a[2 * q + 1]) * cd
        return A * self.rw, B * self.rw

    def blocks_apply(self, items, rows, cols, outs, stats=None):
        """items: list of (AB, c, out_index).  One batched DCT/DST pass over
        all items (schlomilch.py:301-329 and :470-502)."""
        n, m = self.n, self.m
        r0, r1 = rows
        c0, c1 = cols
        dt = np.result_type(*(it[1].dtype for it in items), np.float64)
        U_ = np.zeros((len(items) * 2 * m, n + 1), dtype=dt)
        if c1 > c0:
            wc = self.cw[:, c0 - 1:c1 - 1]
            for q, (_, c, _) in enumerate(items):
                U_[q * 2 * m:(q + 1) * 2 * m, c0:c1] = wc * c[c0 - 1:c1 - 1]
        cp = dct1(U_)[:, 1:]
        sp = np.zeros_like(cp)
        if n >= 2:
            sp[:, :n - 1] = dst1(U_[:, 1:n])
        _bump(stats, "transform_applications", len(items) * 2 * m)
        if r1 <= r0:
            return
        a, b = r0 - self.row_min, r1 - self.row_min
        for q, (AB, _, oi) in enumerate(items):
            s = slice(q * 2 * m, (q + 1) * 2 * m)
            outs[oi][r0 - 1:r1 - 1] += (AB[0][:, a:b] * cp[s, r0 - 1:r1 - 1]
                                       + AB[1][:, a:b] * sp[s, r0 - 1:r1 - 1]).sum(axis=0)


def block_apply(par, rows, cols, c, stats=None):
    """Single asymptotic block increment (schlomilch.py:341-360)."""
    c = np.asarray(c)
    n = par["n"]
    r0, r1 = rows
    c0, c1 = cols
    ff = FarField(par, max(min(r0, n), 1))
    AB = ff.weights(((par["nu"], 1.0),))
    out = [np.zeros(n, dtype=np.result_type(c.dtype, np.float64))]
    ff.blocks_apply([(AB, c, 0)], (r0, r1), (c0, c1), out, stats)
    return out[0]


def schlomilch(par, c, stats=None, levels=None):
    """Full evaluator: blocks then border (schlomilch.py:367-396).  levels=0
    gives schlomilch_single_partition."""
    c = np.asarray(c)
    if c.shape[0] != par["n"]:
        raise ValueError("coefficient length does not match params.n")
    blocks, segs, rmin = partition(par, levels)
    out = [np.zeros(par["n"], dtype=np.result_type(c.dtype, np.float64))]
    ff = FarField(par, rmin)
    ow = ((par["nu"], 1.0),)
    AB = ff.weights(ow)
    for rows, cols in blocks:
        ff.blocks_apply([(AB, c, 0)], rows, cols, out, stats)
    near_field(ow, par["gamma"], par["n"], segs, c, out[0], stats)
    return out[0]


class Engine:
    """Multi-order shared-partition engine (schlomilch.py:405-531)."""

    def __init__(self, n, gamma, eps, orders):
        orders = sorted(set(int(o) for o in orders))
        m = m_terms(eps)
        s = max(hankel_cutoff(o, m, eps) for o in orders)
        self.par = plan_params(orders[-1], n, eps, gamma, s=s, public=False)
        self.blocks, self.segs, self.row_min = partition(self.par)
        self.orders = frozenset(orders)
        self.ff = FarField(self.par, self.row_min)

    def apply_many(self, reqs, stats=None):
        n, m = self.par["n"], self.par["m_terms"]
        reqs = [(tuple(ow), np.asarray(c)) for ow, c in reqs]
        for ow, c in reqs:
            if any(o not in self.orders for o, _ in ow):
                raise ValueError("order outside engine universe")
        outs = [np.zeros(n, dtype=np.result_type(c.dtype, np.float64)) for _, c in reqs]
        ABs = [self.ff.weights(ow) for ow, _ in reqs]
        per = max(FFT_ROWS // (2 * m), 1)
        for rows, cols in self.blocks:
            for i0 in range(0, len(reqs), per):
                idx = range(i0, min(i0 + per, len(reqs)))
                self.ff.blocks_apply([(ABs[i], reqs[i][1], i) for i in idx],
                                     rows, cols, outs, stats)
        # border: Bessel values shared per distinct order (schlomilch.py:504-531)
        users = {}
        for i, (ow, _) in enumerate(reqs):
            for o, w in ow:
                users.setdefault(o, []).append((i, w))
        h = math.pi / n
        for o in sorted(users):
            for r0, r1, ce in self.segs:
                nc = ce - 1
                fr = (np.arange(1, ce, dtype=float) + self.par["gamma"]) * h
                for a in range(r0, r1, NEAR_ROWS):
                    b = min(a + NEAR_ROWS, r1)
                    ks = np.arange(a, b, dtype=float)
                    for j0 in range(0, nc, NEAR_COLS):
                        j1 = min(j0 + NEAR_COLS, nc)
                        z = np.multiply.outer(ks, fr[j0:j1])
                        v = besselj(o, z)
                        _bump(stats, "pointwise_evaluations", z.size)
                        for i, w in users[o]:
                            outs[i][a - 1:b - 1] += w * (v @ reqs[i][1][j0:j1])
        return outs


# ===========================================================================
# L3: Fourier-Bessel                                  (fourier_bessel.py)
# ===========================================================================

def p_cut(kt, eps):
    """p_K(eps) (fourier_bessel.py:54-57)."""
    return math.e / (16.0 * math.pi) * (5.2 / eps) ** (1.0 / kt) + 0.25


def q_cut(tt, eps):
    """q_T(eps) (fourier_bessel.py:60-64)."""
    return eps ** (-1.0 / (2.0 * tt)) / (16.0 * math.pi * math.exp(math.lgamma(tt + 1) / tt)) + 0.25


def neumann_params(eps, margin=1.0):
    """(K, T, p, q, n_split) (fourier_bessel.py:67-86)."""
    if not 0.0 < eps < 1.0:
        raise ValueError("eps must lie in (0, 1)")
    K = 1
    while margin * p_cut(K, eps) > 30.0:
        K += 1
    T = 1
    while margin * q_cut(T, eps) > 30.0:
        T += 1
    p, q = p_cut(K, eps), q_cut(T, eps)
    return dict(k_terms=K, t_terms=T, p_cut=p, q_cut=q, n_split=int(margin * max(p, q)))


def fold(base, u, K, T):
    """Weighted orders of collected term u (fourier_bessel.py:93-123)."""
    acc = {}
    tl = max(-(-(u - K + 1) // 2), 0)
    th = min(u // 2, T - 1)
    for t in range(tl, th + 1):
        s = u - 2 * t
        cf = (-1.0) ** t * 2.0 ** -u / (math.factorial(t) * math.factorial(u - t))
        if s == 0:
            cf *= 0.5
        for b, bw in base:
            for o, w in ((b - s, bw * cf), (b + s, bw * cf * (-1.0) ** s)):
                if o < 0:
                    o, w = -o, w * (-1.0) ** (-o)
                acc[o] = acc.get(o, 0.0) + w
    return tuple(sorted(acc.items()))


def universe(base, K):
    """(fourier_bessel.py:126-132)"""
    return {abs(b + sg * s) for b, _ in base for s in range(K) for sg in (-1, 1)}


def fb_low_columns(jobs, ngrid, roots, outs, stats):
    """Direct low-column part, 4096-row tiles (fourier_bessel.py:148-172)."""
    users = {}
    for i, (base, cl) in enumerate(jobs):
        if cl.shape[0]:
            for o, w in base:
                users.setdefault(o, []).append((i, w))
    if not users:
        return
    ncm = max(c.shape[0] for _, c in jobs)
    r = np.arange(1, ngrid + 1, dtype=float) / ngrid
    fr = roots[:ncm]
    for o in sorted(users):
        for k0 in range(0, ngrid, 4096):
            k1 = min(k0 + 4096, ngrid)
            z = np.multiply.outer(r[k0:k1], fr)
            v = besselj(o, z)
            _bump(stats, "pointwise_evaluations", z.size)
            for i, w in users[o]:
                nc = jobs[i][1].shape[0]
                if nc:
                    outs[i][k0:k1] += w * (v[:, :nc] @ jobs[i][1])


def fb_jobs(jobs, np_, seps, roots, pert, stats=None, engine=None, prune_eps=None):
    """Batched FB evaluation of (base_orders, c) jobs (fourier_bessel.py:175-243)."""
    ng = jobs[0][1].shape[0]
    ns = min(np_["n_split"], ng)
    outs, low = [], []
    for base, c in jobs:
        if c.shape[0] != ng:
            raise ValueError("all jobs must share one grid size")
        outs.append(np.zeros(ng, dtype=np.result_type(c.dtype, np.float64)))
        low.append((base, c[:ns]))
    fb_low_columns(low, ng, roots, outs, stats)
    if ng <= ns:
        return outs
    sup = min(ng, roots.shape[0])
    b = np.zeros(ng)
    b[:sup] = pert[:sup]
    top = 2 * np_["t_terms"] + np_["k_terms"] - 2
    reqs, place = [], []
    for i, (base, c) in enumerate(jobs):
        if np.any(c[sup:]):
            raise ValueError("roots table too short")
        ch = c.copy()
        ch[:ns] = 0.0
        if np.sum(np.abs(ch)) == 0.0:
            continue
        bmax = float(np.max(np.abs(b[ch != 0.0])))
        bp = np.ones(ng)
        for u in range(top):
            tm = fold(base, u, np_["k_terms"], np_["t_terms"])
            if tm:
                keep = True
                if prune_eps is not None:
                    keep = bmax ** u * sum(abs(w) for _, w in tm) >= 0.02 * prune_eps
                if keep:
                    reqs.append((tm, bp * ch))
                    place.append((i, u))
                    _bump(stats, "schlomilch_evaluations", 1)
            bp = bp * b
    if not reqs:
        return outs
    if engine is None:
        uni = set()
        for base, _ in jobs:
            uni |= universe(base, np_["k_terms"])
        engine = Engine(ng, -0.25, seps, uni)
    ys = engine.apply_many(reqs, stats)
    r = np.arange(1, ng + 1, dtype=float) / ng
    for (i, u), y in zip(place, ys):
        outs[i] += r ** u * y
    return outs


def fourier_bessel(nu, c, eps, roots=None, stats=None, prune=False):
    """(fourier_bessel.py:312-337); roots = (roots, perturbations) or None."""
    if eps < MIN_EPS:
        raise ValueError("eps below 2^-52")
    c = np.asarray(c)
    if roots is None:
        roots = j0_roots(c.shape[0])
    np_ = neumann_params(eps)
    ie = eps / (2 * np_["t_terms"] + np_["k_terms"] - 2)
    return fb_jobs([(((int(nu), 1.0),), c)], np_, ie, roots[0], roots[1], stats,
                   prune_eps=eps if prune else None)[0]


def fourier_bessel_direct(nu, c, roots=None):
    """(fourier_bessel.py:292-309)"""
    c = np.asarray(c)
    n = c.shape[0]
    rt = j0_roots(n)[0] if roots is None else roots[0]
    out = np.zeros(n, dtype=np.result_type(c.dtype, np.float64))
    cmp_ = np.zeros_like(out)
    r = np.arange(1, n + 1, dtype=float) / n
    for c0 in range(0, n, 512):
        c1 = min(c0 + 512, n)
        part = np.zeros_like(out)
        for k0 in range(0, n, 2048):
            k1 = min(k0 + 2048, n)
            part[k0:k1] = besselj(nu, np.multiply.outer(r[k0:k1], rt[c0:c1])) @ c[c0:c1]
        y = part - cmp_
        t = out + y
        cmp_ = (t - out) - y
        out = t
    return out


# ===========================================================================
# L4: discrete Hankel transform                                    (dht.py)
# ===========================================================================

class DhtOracle:
    """Plan + transforms (dht.py:36-176)."""

    def __init__(self, n, eps):
        if eps < MIN_EPS:
            raise ValueError("eps below 2^-52")
        if n < 1:
            raise ValueError("n must be >= 1")
        self.n, self.eps = n, eps
        self.np_ = neumann_params(eps, margin=1.01)
        self.roots, self.pert = j0_roots(n + 1)
        j1 = besselj(1, self.roots[:n])
        self.weights = 2.0 / (j1 * j1)
        self._eng = None

    def rows_direct(self, c, k0, k1, stats=None):
        """(dht.py:82-94)"""
        n = self.n
        sc = self.roots[k0 - 1:k1 - 1] / self.roots[n]
        out = np.zeros(k1 - k0, dtype=np.result_type(c.dtype, np.float64))
        cmp_ = np.zeros_like(out)
        for c0 in range(0, n, 512):
            c1 = min(c0 + 512, n)
            z = np.multiply.outer(sc, self.roots[c0:c1])
            _bump(stats, "pointwise_evaluations", z.size)
            y = besselj(0, z) @ c[c0:c1] - cmp_
            t = out + y
            cmp_ = (t - out) - y
            out = t
        return out

    def direct(self, c):
        c = np.asarray(c)
        if c.shape[0] != self.n:
            raise ValueError("coefficient length does not match plan.n")
        return self.rows_direct(c, 1, self.n + 1)

    def shared(self):
        """(dht.py:105-120)"""
        if self._eng is None:
            fbp = neumann_params(self.eps)
            ro = 2 * self.np_["t_terms"] + self.np_["k_terms"] - 2
            ri = 2 * fbp["t_terms"] + fbp["k_terms"] - 2
            se = self.eps / (ro * ri)
            uni = universe([(s, 1.0) for s in range(self.np_["k_terms"])], fbp["k_terms"])
            self._eng = (Engine(4 * self.n + 3, -0.25, se, uni), fbp, se)
        return self._eng

    def transform(self, c, stats=None):
        """(dht.py:123-176)"""
        c = np.asarray(c)
        n = self.n
        if c.shape[0] != n:
            raise ValueError("coefficient length does not match plan.n")
        sp = min(self.np_["n_split"], n)
        if sp >= n:
            return self.rows_direct(c, 1, n + 1, stats)
        eng, fbp, se = self.shared()
        e = self.roots[:n] / self.roots[n] - (np.arange(1, n + 1) - 0.25) / (n + 0.75)
        j0 = self.roots[:n]
        npad = 4 * n + 3
        out = np.zeros(n, dtype=np.result_type(c.dtype, np.float64))
        nrm = float(np.sum(np.abs(c)))
        gmax = 1.01 / (8.0 * (sp + 0.75) * math.pi)
        jobs, us = [], []
        jp = np.ones(n)
        K, T = self.np_["k_terms"], self.np_["t_terms"]
        for u in range(2 * T + K - 2):
            tm = fold(((0, 1.0),), u, K, T)
            if tm and nrm > 0.0 and gmax ** u * sum(abs(w) for _, w in tm) >= 0.02 * self.eps:
                pad = np.zeros(npad, dtype=np.result_type(c.dtype, np.float64))
                pad[:n] = jp * c
                jobs.append((tm, pad))
                us.append(u)
                _bump(stats, "fb_evaluations", 1)
            jp = jp * j0
        if jobs:
            ys = fb_jobs(jobs, fbp, se, self.roots, self.pert, stats, eng, prune_eps=self.eps)
            ep = np.ones(n)
            epow = {0: ep.copy()}
            for u in range(1, us[-1] + 1):
                ep = ep * e
                epow[u] = ep.copy()
            for u, y in zip(us, ys):
                out += epow[u] * y[2:4 * n:4]
        out[:sp] = self.rows_direct(c, 1, sp + 1, stats)
        return out

    def self_inverse_residual(self, c, method="fast"):
        """(dht.py:179-194)"""
        c = np.asarray(c)
        f = self.transform if method == "fast" else self.direct
        y = f(self.weights * c)
        y = f(self.weights * y)
        return float(np.max(np.abs(y / self.roots[self.n] ** 2 - c)))
