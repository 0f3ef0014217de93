"""Schlomilch expansions f_k = sum_n c_n J_nu((n+gamma) pi k / N), k = 1..N
(drop-in for fasthankel.schlomilch, reference schlomilch.py).

Host: the eps-driven planner (Table 4 parameters, block partition), the
request lists and the instrumentation counters.  Device (libfhtb200.so): the
whole N-length computation -- fused DCT-I/DST-I far field and the DMMA
near field -- on one CUDA stream, deterministic reduction order.

Extensions over the reference (same results for the reference's inputs):
coefficients may be a (batch, N) matrix (rows are independent vectors) or a
CUDA torch tensor, in which case the result stays on the device.
"""

import collections
import ctypes
import math
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _device, _lib
from .bessel import asy_coeffs, asy_cutoff  # noqa: F401  (re-exported like the reference)

__all__ = [
    "SchlomilchParams",
    "PartitionScheme",
    "select_params",
    "build_partition",
    "schlomilch_direct",
    "asy_block_apply",
    "schlomilch_single_partition",
    "schlomilch_fast",
]

MIN_EPS = 2.0 ** -52


# ---------------------------------------------------------------------------
# Planner (host).  Formulas and floating-point expression order follow
# schlomilch.py:72-170 so that every ceil() edge agrees bit for bit.

@dataclass(frozen=True)
class SchlomilchParams:
    """Table-4 parameters of one (nu, N, eps, gamma) problem (schlomilch.py:51-69)."""

    eps: float
    nu: int
    gamma: float
    n: int
    m_terms: int
    s: float
    alpha: float
    beta: float
    partitions: int


def _m_terms(eps):
    return max(int(0.3 * math.log(1.0 / eps)), 3)


def _select_params(nu, n, eps, gamma, s=None):
    """Internal variant without the 2^-52 floor (schlomilch.py:76-99)."""
    if not 0.0 < eps < 1.0:
        raise ValueError("eps must lie in (0, 1)")
    if n < 1:
        raise ValueError("n must be >= 1")
    if nu < 0:
        raise ValueError("nu must be >= 0")
    if gamma <= -1.0:
        raise ValueError("gamma must exceed -1 so all frequencies are positive")
    m = _m_terms(eps)
    if s is None:
        s = asy_cutoff(nu, m, eps)
    alpha = math.sqrt(s / math.pi)
    beta = 1.0 if n <= 20 else min(3.0 / math.log(n), 1.0)
    x = 30.0 / (alpha * math.sqrt(n))
    if x >= 1.0 or beta >= 1.0:
        p = 0
    else:
        p = max(math.ceil(math.log(x) / math.log(beta)), 0)
    return SchlomilchParams(eps=eps, nu=nu, gamma=gamma, n=n, m_terms=m, s=s, alpha=alpha,
                            beta=beta, partitions=p)


def select_params(nu, n, eps, gamma=0.0):
    """Derive M, s, alpha, beta, P from eps (schlomilch.py:102-112)."""
    if eps < MIN_EPS:
        raise ValueError("eps below 2^-52 is not resolvable in double precision")
    return _select_params(nu, n, eps, gamma)


@dataclass(frozen=True)
class PartitionScheme:
    """Blocks ((r0,r1),(c0,c1)) and border segments (r0,r1,c_end), 1-based
    half-open (schlomilch.py:119-136)."""

    n: int
    blocks: tuple
    mask_segments: tuple
    row_min: int

    def mask_size(self):
        return sum((r1 - r0) * (ce - 1) for r0, r1, ce in self.mask_segments)


def build_partition(params, partitions=None):
    """Partition for `params`, P overridable (schlomilch.py:139-170)."""
    n = params.n
    levels = params.partitions if partitions is None else partitions
    rn = math.sqrt(n)
    a = [min(math.ceil(params.alpha * params.beta ** p * rn), n + 1) for p in range(levels + 1)]
    b = [None] + [min(math.ceil(params.alpha * params.beta ** -p * rn), n + 1)
                  for p in range(1, levels + 1)]
    blocks = [((a[0], n + 1), (a[0], n + 1))]
    for p in range(1, levels + 1):
        blocks.append(((a[p], a[p - 1]), (b[p], n + 1)))
        blocks.append(((b[p], n + 1), (a[p], a[p - 1])))
    segs = []

    def add(r0, r1, ce):
        if r1 > r0 and ce > 1:
            segs.append((r0, r1, ce))

    add(1, a[levels], n + 1)
    for p in range(levels, 0, -1):
        add(a[p], a[p - 1], b[p])
    prev = a[0]
    for p in range(1, levels + 1):
        add(prev, b[p], a[p - 1])
        prev = b[p]
    add(prev, n + 1, a[levels])
    return PartitionScheme(n=n, blocks=tuple(blocks), mask_segments=tuple(segs), row_min=a[levels])


# ---------------------------------------------------------------------------
# Device grid objects and request plumbing.

class _Grid:
    """Owns one fhtb_grid (partition + device tables) on one device."""

    def __init__(self, L, gamma, m_terms, blocks, segments, orders, row_first=1, row_stride=1,
                 n_out=None, n_data_cols=None):
        _device.ensure_init()
        self.L = int(L)
        self.n_out = int(L if n_out is None else n_out)
        self.orders = [int(o) for o in orders]
        self.m_terms = int(m_terms)
        self.n_blocks = len(blocks)
        self._lib = _lib.load()
        blk, blk_p = _lib.i64_array([v for (r, c) in blocks for v in (r[0], r[1], c[0], c[1])] or [0])
        seg, seg_p = _lib.i64_array([v for s in segments for v in s] or [0])
        ords, ords_p = _lib.i32_array(self.orders)
        d = _lib.GridDesc(L=self.L, gamma=float(gamma), m_terms=self.m_terms, n_blocks=len(blocks),
                          blocks=blk_p, n_segments=len(segments), segments=seg_p,
                          row_first=int(row_first), row_stride=int(row_stride), n_out=self.n_out,
                          n_data_cols=int(self.L if n_data_cols is None else n_data_cols),
                          n_orders=len(self.orders), orders=ords_p)
        h = ctypes.c_void_p()
        _lib.check(self._lib.fhtb_grid_create(ctypes.byref(d), ctypes.byref(h)))
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self._lib.fhtb_grid_destroy(h)
            except Exception:
                pass

    def apply(self, requests, C, F, flags=_lib.FHTB_FAR | _lib.FHTB_NEAR):
        """F[vec] += application of each request; C, F are (B, *) float64 CUDA tensors."""
        if not requests:
            return F
        arr, keep = _pack_requests(requests)
        s, n = _device.shard()
        xfn = _device.shard_exchange()
        unit = self._lib.fhtb_apply_x_unit_bytes(self.handle, n) if (xfn is not None and n > 1) else 0
        if unit:
            return self._apply_exchange(arr, len(requests), C, F, flags, s, n, xfn, unit, keep)
        ws_n = self._lib.fhtb_apply_workspace(self.handle, len(requests), C.shape[0], flags)
        ws = _device.workspace(ws_n)
        _lib.check(self._lib.fhtb_apply_part(self.handle, arr, len(requests), _device.ptr(C), C.stride(0),
                                             C.shape[0], _device.ptr(F), F.stride(0), flags, s, n,
                                             _device.ptr(ws), ws.numel(), _device.stream_ptr()))
        del keep
        return F

    # apply_host vector groups: up to eight tapered groups (end groups 1/4 of
    # the inner ones), at least 8 vectors per group; measured on cfg2 (64
    # vectors, e2e transforms/s): 2 groups 719, 3 773, 4 795, 8 798, 10 799,
    # 16 788
    HOST_GROUPS = 8
    HOST_GROUP_MIN_VECS = 8

    def apply_host(self, requests, C, F, flags=_lib.FHTB_FAR | _lib.FHTB_NEAR, n_groups=None, sync=True):
        """F = application of the requests, C and F pinned host float64
        tensors (B, n_data_cols) / (B, n_out): fhtb_apply_host, the copies
        overlapped with the far field in vector groups.  Same bits as
        apply() on device copies with F = 0."""
        if n_groups is None:
            n_groups = min(self.HOST_GROUPS, max(1, C.shape[0] // self.HOST_GROUP_MIN_VECS))
        arr, keep = _pack_requests(requests)
        ws_n = self._lib.fhtb_apply_host_workspace(self.handle, len(requests), C.shape[0], flags)
        ws = _device.workspace(ws_n)
        _lib.check(self._lib.fhtb_apply_host(self.handle, arr, len(requests), C.data_ptr(), C.stride(0),
                                             C.shape[0], F.data_ptr(), F.stride(0), flags, int(n_groups),
                                             _device.ptr(ws), ws.numel(), _device.stream_ptr()))
        if sync:
            torch.cuda.current_stream().synchronize()
        del keep
        return F

    X_BUDGET = 1 << 30          # bytes per exchange buffer (send; recv the same)

    def _apply_exchange(self, arr, n_req, C, F, flags, s, n, xfn, unit, keep):
        """fhtb_apply_x: the all-to-all between pass 1 and pass 2 is xfn."""
        xbytes = max(1, self.X_BUDGET // unit) * unit
        dev = C.device
        send = torch.empty(xbytes, dtype=torch.uint8, device=dev)
        recv = torch.empty(xbytes, dtype=torch.uint8, device=dev)
        errors = []

        def _cb(user, rnd, bpp):
            try:
                xfn(send, recv, int(bpp))
                return 0
            except Exception as exc:          # surfaced after the library returns
                errors.append(exc)
                return 1

        cb = _lib.EXCHANGE_FN(_cb)
        ws_n = self._lib.fhtb_apply_x_workspace(self.handle, n_req, C.shape[0], flags, n, xbytes)
        ws = torch.empty(max(int(ws_n), 256), dtype=torch.uint8, device=dev)
        code = self._lib.fhtb_apply_x(self.handle, arr, n_req, _device.ptr(C), C.stride(0), C.shape[0],
                                      _device.ptr(F), F.stride(0), flags, s, n, _device.ptr(send),
                                      _device.ptr(recv), xbytes, cb, None, _device.ptr(ws), ws.numel(),
                                      _device.stream_ptr())
        if errors:
            raise errors[0]
        _lib.check(code)
        del keep, cb
        return F


def _pack_requests(requests):
    """requests: dicts with keys vec, terms[(order, weight)], and optional
    col_lo, pre_a (tensor), pre_a_pow, pre_b, pre_b_pow, post_r_pow, post_e, post_e_pow."""
    arr = (_lib.Request * len(requests))()
    keep = []
    for i, r in enumerate(requests):
        o, op = _lib.i32_array([t[0] for t in r["terms"]] or [0])
        w, wp = _lib.f64_array([t[1] for t in r["terms"]] or [0.0])
        keep += [o, w]
        q = arr[i]
        q.vec = int(r["vec"])
        q.n_terms = len(r["terms"])
        q.orders = op
        q.weights = wp
        q.col_lo = int(r.get("col_lo", 1))
        q.pre_a = _device.ptr(r.get("pre_a"))
        q.pre_a_pow = int(r.get("pre_a_pow", 0)) if r.get("pre_a") is not None else 0
        q.pre_b = _device.ptr(r.get("pre_b"))
        q.pre_b_pow = int(r.get("pre_b_pow", 0)) if r.get("pre_b") is not None else 0
        q.post_r_pow = int(r.get("post_r_pow", 0))
        q.post_e = _device.ptr(r.get("post_e"))
        q.post_e_pow = int(r.get("post_e_pow", 0)) if r.get("post_e") is not None else 0
    return arr, keep


_grid_lock = threading.Lock()
_grid_cache = collections.OrderedDict()
_GRID_CACHE_MAX = 24


_MAX_UNIVERSE = 16      # orders per fhtb_grid, inside a window of 16 consecutive orders (fhtb_types.h kMaxOrd)


def _order_windows(orders):
    """Greedy split of a sorted universe into groups one fhtb_grid can hold."""
    out, cur = [], []
    for o in sorted(set(int(o) for o in orders)):
        if cur and (len(cur) >= _MAX_UNIVERSE or o - cur[0] >= _MAX_UNIVERSE):
            out.append(cur)
            cur = []
        cur.append(o)
    if cur:
        out.append(cur)
    return out


class _MultiGrid:
    """A universe wider than one fhtb_grid holds (reference engines take any
    order set, schlomilch.py:422-431): one grid per order window, every
    request split by its terms; far and near field are linear in the terms."""

    def __init__(self, grids):
        self.grids = grids
        self.orders = [o for g in grids for o in g.orders]
        self.L, self.n_out, self.m_terms, self.n_blocks = grids[0].L, grids[0].n_out, grids[0].m_terms, grids[0].n_blocks

    def apply(self, requests, C, F, flags=_lib.FHTB_FAR | _lib.FHTB_NEAR):
        for g in self.grids:
            own = set(g.orders)
            part = []
            for r in requests:
                terms = [(o, w) for o, w in r["terms"] if int(o) in own]
                if terms:
                    part.append(dict(r, terms=terms))
            g.apply(part, C, F, flags)
        return F

    def apply_host(self, requests, C, F, flags=_lib.FHTB_FAR | _lib.FHTB_NEAR, n_groups=None):
        dev = _device.device()
        Cd = C.to(dev, non_blocking=True)
        Fd = torch.zeros((C.shape[0], self.n_out), dtype=torch.float64, device=dev)
        self.apply(requests, Cd, Fd, flags)
        F.copy_(Fd)
        return F


def _grid(L, gamma, m_terms, blocks, segments, orders, row_first=1, row_stride=1, n_out=None,
          n_data_cols=None):
    wins = _order_windows(orders)
    if len(wins) > 1:
        return _MultiGrid([_grid(L, gamma, m_terms, blocks, segments, w, row_first, row_stride, n_out, n_data_cols)
                           for w in wins])
    key = (torch.cuda.current_device(), int(L), float(gamma), int(m_terms), tuple(blocks), tuple(segments),
           tuple(int(o) for o in orders), int(row_first), int(row_stride), n_out, n_data_cols)
    with _grid_lock:
        g = _grid_cache.get(key)
        if g is not None:
            _grid_cache.move_to_end(key)
            return g
    g = _Grid(L, gamma, m_terms, blocks, segments, orders, row_first, row_stride, n_out, n_data_cols)
    with _grid_lock:
        _grid_cache[key] = g
        while len(_grid_cache) > _GRID_CACHE_MAX:
            _grid_cache.popitem(last=False)
    return g


def _bump(stats, key, amount):
    if stats is not None:
        stats[key] = stats.get(key, 0) + amount


def _host_pinned_real(c):
    """A pinned real float64 CPU tensor (vector or batch) takes the
    host-buffer path (fhtb_apply_host) unless a work split is active."""
    return (isinstance(c, torch.Tensor) and c.device.type == "cpu" and c.dtype == torch.float64
            and c.ndim in (1, 2) and c.is_contiguous() and c.is_pinned() and _device.shard()[1] == 1)


# numpy in / numpy out (the reference's calling convention) for large real
# batches: pageable memory cannot be copied asynchronously, so the rows are
# staged through pinned buffers (three slots) in vector chunks -- worker
# threads copy chunk i+1 in and chunk i-1 out (numpy copies release the GIL)
# while the GPU runs chunk i; consecutive chunks alternate between two CUDA
# streams so that one chunk's copy-out overlaps the next one's far field.
_NP_PIPE_MIN_ELEMS = 1 << 22
_NP_PIPE_THREADS = 4            # host copy workers (a fresh result array is first touched by the copy-out)
_np_pipe_lock = threading.Lock()
_np_pipe = {}


def _np_pipe_state(rows, n, n_out):
    key = (torch.cuda.current_device(), rows, n, n_out)
    st = _np_pipe.get(key)
    if st is None:
        import concurrent.futures
        _np_pipe.clear()                                   # one shape at a time (pinned memory is scarce)
        st = dict(pin_in=[torch.empty((rows, n), dtype=torch.float64, pin_memory=True) for _ in range(3)],
                  pin_out=[torch.empty((rows, n_out), dtype=torch.float64, pin_memory=True) for _ in range(3)],
                  streams=[torch.cuda.Stream() for _ in range(2)],
                  pool=concurrent.futures.ThreadPoolExecutor(_NP_PIPE_THREADS))
        _np_pipe[key] = st
    return st


def _run_numpy_pipelined(g, order_weights, c2, flags):
    B, n = c2.shape
    rows = 8 if B >= 16 else max(1, (B + 1) // 2)
    n_out = g.n_out
    out = np.empty((B, n_out))
    with _np_pipe_lock:
        st = _np_pipe_state(rows, n, n_out)
        pin_in, pin_out, streams, pool = st["pin_in"], st["pin_out"], st["streams"], st["pool"]
        chunks = [(lo, min(B, lo + rows)) for lo in range(0, B, rows)]
        np_in = [t.numpy() for t in pin_in]
        np_out = [t.numpy() for t in pin_out]

        class _Many:
            def __init__(self, fs):
                self.fs = fs

            def result(self):
                for f in self.fs:
                    f.result()

        def halves(lo, hi):
            mid = (lo + hi + 1) // 2
            return [(lo, mid), (mid, hi)] if hi - lo > 1 else [(lo, hi)]

        def stage_in(i):
            lo, hi = chunks[i]
            return _Many([pool.submit(np.copyto, np_in[i % 3][a - lo: b - lo], c2[a:b]) for a, b in halves(lo, hi)])

        def stage_out(i):
            lo, hi = chunks[i]
            return _Many([pool.submit(np.copyto, out[a:b], np_out[i % 3][a - lo: b - lo]) for a, b in halves(lo, hi)])

        cur = torch.cuda.current_stream()
        for s_ in streams:
            s_.wait_stream(cur)
        f_in = {0: stage_in(0)}
        f_out, done = {}, {}
        for i, (lo, hi) in enumerate(chunks):
            if i + 1 < len(chunks):
                f_in[i + 1] = stage_in(i + 1)              # slot (i+1) % 3: chunk i-2 was waited for at step i-1
            f_in[i].result()
            if i >= 3:
                f_out[i - 3].result()                      # pin_out[i % 3] is free again
            reqs = [dict(vec=v, terms=list(order_weights)) for v in range(hi - lo)]
            with torch.cuda.stream(streams[i % 2]):
                g.apply_host(reqs, pin_in[i % 3][: hi - lo], pin_out[i % 3][: hi - lo], flags, sync=False)
                done[i] = torch.cuda.Event()
                done[i].record()
            if i >= 1:
                done[i - 1].synchronize()
                f_out[i - 1] = stage_out(i - 1)
        last = len(chunks) - 1
        done[last].synchronize()
        f_out[last] = stage_out(last)
        for f in f_out.values():
            f.result()
        cur.wait_stream(streams[0])
        cur.wait_stream(streams[1])
    return out


def _run(params, scheme, order_weights, c, stats, flags=_lib.FHTB_FAR | _lib.FHTB_NEAR):
    """Apply the partitioned scheme to c (vector, batch or tensor)."""
    if (isinstance(c, np.ndarray) and c.dtype == np.float64 and c.ndim == 2 and c.shape[0] >= 4
            and c.size >= _NP_PIPE_MIN_ELEMS and _device.shard()[1] == 1 and c.shape[-1] == params.n):
        _device.ensure_init()
        orders = sorted({int(o) for o, _ in order_weights})
        g = _grid(params.n, params.gamma, params.m_terms, scheme.blocks, scheme.mask_segments, orders)
        if isinstance(g, _Grid):
            F = _run_numpy_pipelined(g, order_weights, c, flags)
            if flags & _lib.FHTB_FAR:
                _bump(stats, "transform_applications", c.shape[0] * 2 * params.m_terms * len(scheme.blocks))
            if flags & _lib.FHTB_NEAR:
                _bump(stats, "pointwise_evaluations", c.shape[0] * scheme.mask_size() * len(order_weights))
            return F
    if _host_pinned_real(c):
        if c.shape[-1] != params.n:
            raise ValueError("coefficient length does not match params.n")
        _device.ensure_init()
        orders = sorted({int(o) for o, _ in order_weights})
        g = _grid(params.n, params.gamma, params.m_terms, scheme.blocks, scheme.mask_segments, orders)
        C = c.reshape(-1, c.shape[-1]).contiguous()
        F = torch.empty(C.shape, dtype=torch.float64, pin_memory=True)
        reqs = [dict(vec=v, terms=list(order_weights)) for v in range(C.shape[0])]
        g.apply_host(reqs, C, F, flags)
        if flags & _lib.FHTB_FAR:
            _bump(stats, "transform_applications", C.shape[0] * 2 * params.m_terms * len(scheme.blocks))
        if flags & _lib.FHTB_NEAR:
            _bump(stats, "pointwise_evaluations", C.shape[0] * scheme.mask_size() * len(order_weights))
        return F[0] if c.ndim == 1 else F
    C, meta = _device.as_real_batch(c)
    if C.shape[-1] != params.n:
        raise ValueError("coefficient length does not match params.n")
    orders = sorted({int(o) for o, _ in order_weights})
    g = _grid(params.n, params.gamma, params.m_terms, scheme.blocks, scheme.mask_segments, orders)
    F = _device.zeros_like(C)
    reqs = [dict(vec=v, terms=list(order_weights)) for v in range(C.shape[0])]
    g.apply(reqs, C, F, flags)
    nvec = C.shape[0] // (2 if meta["complex"] else 1)
    if flags & _lib.FHTB_FAR:
        _bump(stats, "transform_applications", nvec * 2 * params.m_terms * len(scheme.blocks))
    if flags & _lib.FHTB_NEAR:
        _bump(stats, "pointwise_evaluations", nvec * scheme.mask_size() * len(order_weights))
    return _device.from_real_batch(F, meta)


def schlomilch_direct(nu, gamma, c):
    """Direct O(N^2) summation (schlomilch.py:223-229): one border segment
    covering the whole square, evaluated by the same near-field kernel as
    the fast schemes (so a degenerate partition is bitwise identical)."""
    n = (c.shape[-1] if hasattr(c, "shape") else len(c))
    c_arr = c if isinstance(c, torch.Tensor) else np.asarray(c)
    p = SchlomilchParams(eps=0.5, nu=int(nu), gamma=float(gamma), n=n, m_terms=3, s=0.0,
                         alpha=0.0, beta=1.0, partitions=0)
    sc = PartitionScheme(n=n, blocks=(), mask_segments=((1, n + 1, n + 1),), row_min=n + 1)
    return _run(p, sc, ((int(nu), 1.0),), c_arr, None, _lib.FHTB_NEAR)


def asy_block_apply(params, rows, cols, c, stats=None):
    """Asymptotic increment of one (rows x cols) block (schlomilch.py:341-360)."""
    c_arr = c if isinstance(c, torch.Tensor) else np.asarray(c)
    n = params.n
    r0, r1 = _as_bounds(rows)
    c0, c1 = _as_bounds(cols)
    if r1 > r0 and c1 > c0:
        assert r0 * (c0 + params.gamma) * math.pi / n >= params.s * (1.0 - 1e-12), \
            "block contains entries below the asymptotic cutoff"
    sc = PartitionScheme(n=n, blocks=(((r0, r1), (c0, c1)),), mask_segments=(), row_min=max(min(r0, n), 1))
    return _run(params, sc, ((params.nu, 1.0),), c_arr, stats, _lib.FHTB_FAR)


def _as_bounds(r):
    if isinstance(r, range):
        if r.step != 1:
            raise ValueError("index ranges must have step 1")
        return r.start, r.stop
    lo, hi = r
    return int(lo), int(hi)


def schlomilch_single_partition(params, c, stats=None):
    """Central asymptotic block + direct border, O(N^{3/2}) (schlomilch.py:381-386)."""
    c_arr = c if isinstance(c, torch.Tensor) else np.asarray(c)
    return _run(params, build_partition(params, partitions=0), ((params.nu, 1.0),), c_arr, stats)


def schlomilch_fast(params, c, stats=None):
    """Recursively partitioned evaluation (schlomilch.py:389-396).  With
    P == 0 this is the same device program as schlomilch_single_partition,
    hence bitwise identical."""
    c_arr = c if isinstance(c, torch.Tensor) else np.asarray(c)
    return _run(params, build_partition(params), ((params.nu, 1.0),), c_arr, stats)


class SchlomilchEngine:
    """Shared-partition multi-order engine (schlomilch.py:405-531): the
    partition cutoff is the maximum asymptotic cutoff over the order
    universe; a batch of (order_weights, c) requests runs as ONE device
    application (far-field FFTs and border Bessel values shared)."""

    def __init__(self, n, gamma, eps, orders):
        orders = sorted(set(int(o) for o in orders))
        if not orders or orders[0] < 0:
            raise ValueError("order universe must be non-empty, orders >= 0")
        m = _m_terms(eps)
        s = max(asy_cutoff(o, m, eps) for o in orders)
        self.params = _select_params(orders[-1], n, eps, gamma, s=s)
        self.scheme = build_partition(self.params)
        self.orders = frozenset(orders)
        self._order_list = orders

    def grid(self, row_first=1, row_stride=1, n_out=None, n_data_cols=None):
        p, sc = self.params, self.scheme
        return _grid(p.n, p.gamma, p.m_terms, sc.blocks, sc.mask_segments, self._order_list,
                     row_first, row_stride, n_out, n_data_cols)

    def count(self, requests, stats):
        """Reference instrumentation of apply_many (schlomilch.py:488-491, 524-527)."""
        if stats is None:
            return
        _bump(stats, "transform_applications", len(requests) * 2 * self.params.m_terms * len(self.scheme.blocks))
        used = {o for r in requests for o, _ in r}
        _bump(stats, "pointwise_evaluations", len(used) * self.scheme.mask_size())

    def apply(self, order_weights, c, stats=None):
        return self.apply_many([(order_weights, c)], stats)[0]

    def apply_many(self, requests, stats=None):
        n = self.params.n
        rows, dts = [], []
        # order_weights may be one-shot iterables (schlomilch.py:470-472 takes a tuple first)
        requests = [(tuple(ow), c) for ow, c in requests]
        for ow, c in requests:
            for o, _ in ow:
                if o not in self.orders:
                    raise ValueError("order %d outside engine universe" % o)
            c = np.asarray(c)
            if c.shape[0] != n:
                raise ValueError("coefficient length does not match engine grid")
            rows.append(c)
            dts.append(c.dtype)
        if not requests:
            return []
        cplx = any(np.iscomplexobj(r) for r in rows)
        mat = np.stack([r.astype(np.complex128 if cplx else np.float64) for r in rows])
        C, meta = _device.as_real_batch(mat)
        F = _device.zeros_like(C)
        per = 2 if cplx else 1
        reqs = []
        for i, (ow, _) in enumerate(requests):
            for part in range(per):
                reqs.append(dict(vec=per * i + part, terms=list(ow)))
        self.grid().apply(reqs, C, F)
        self.count([ow for ow, _ in requests], stats)
        out = _device.from_real_batch(F, dict(meta, one=False))
        return [out[i].astype(np.result_type(dts[i], np.float64)) for i in range(len(requests))]
