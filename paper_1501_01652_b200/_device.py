"""Device plumbing: torch tensors for memory/streams, workspace cache.

PyTorch is used only to own device memory, pick the current stream and move
host arrays; every numerical operation on N-length data runs in
libfhtb200.so.
"""

import contextlib
import ctypes
import threading

import numpy as np
import torch

from . import _lib

_ws_lock = threading.Lock()
_ws = {}
_tls = threading.local()


def shard():
    """(index, count) of the work split active in this thread (default (0, 1))."""
    return getattr(_tls, "shard", (0, 1))


def shard_exchange():
    """The all-to-all callable of the active split, or None (pair split)."""
    return getattr(_tls, "exchange", None)


@contextlib.contextmanager
def sharding(index, count, exchange=None):
    """Within the block, every engine application computes only shard
    `index` of `count`, and direct (non-engine) sums run on shard 0 only; the
    `count` partial results sum to the full transform
    (dist.distributed_transform).

    exchange=None: fhtb_apply_part (term pairs and near-field tiles).
    exchange=fn:   fhtb_apply_x -- full far-field blocks of power-of-two grids
                   as a distributed four-step FFT; fn(send, recv, bytes_per_peer)
                   must perform the all-to-all of the uint8 CUDA buffers
                   (count equal chunks of bytes_per_peer each) in stream order.
    """
    index, count = int(index), int(count)
    if count < 1 or not 0 <= index < count:
        raise ValueError("bad shard index/count")
    prev, prev_x = shard(), shard_exchange()
    _tls.shard = (index, count)
    _tls.exchange = exchange
    try:
        yield
    finally:
        _tls.shard = prev
        _tls.exchange = prev_x


def device():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1501_01652_b200 needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr():
    return ctypes_void(torch.cuda.current_stream().cuda_stream)


def ctypes_void(x):
    return x if x else None


def ptr(t):
    return t.data_ptr() if t is not None else None


_inited = set()


def ensure_init():
    dev = device()
    if dev.index not in _inited:
        _lib.load()
        _lib.call("fhtb_init")
        _inited.add(dev.index)
    return dev


def workspace(nbytes):
    """A cached uint8 device buffer of at least nbytes (per device/stream)."""
    dev = device()
    key = (dev.index, torch.cuda.current_stream().cuda_stream)
    with _ws_lock:
        buf = _ws.get(key)
        if buf is None or buf.numel() < nbytes:
            if buf is not None:
                del _ws[key]
                buf = None
            buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=dev)
            _ws[key] = buf
    return buf


def zeros_like(C):
    """A zeroed result matrix shaped like C (library memset on the current stream)."""
    F = torch.empty_like(C)
    if F.numel():
        _lib.call("fhtb_zero_rows", ptr(F), F.stride(0) if F.ndim == 2 else F.numel(),
                  F.shape[0] if F.ndim == 2 else 1, F.shape[-1], stream_ptr())
    return F


def coef_stats(C, n_split=0, b_dev=None):
    """Per row of the (B, N) device matrix C: (sum |c|, max |b_n| over the
    n >= n_split with c_n != 0, any such n) -- one library kernel and one
    small copy instead of a chain of eager tensor ops."""
    out = np.zeros((C.shape[0], 3))
    if C.shape[0]:
        nb = 0 if b_dev is None else int(b_dev.numel())
        _lib.call("fhtb_coef_stats", ptr(C), C.stride(0), C.shape[0], C.shape[1], int(n_split),
                  ptr(b_dev) if b_dev is not None else None, nb,
                  out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), stream_ptr())
    return out[:, 0], out[:, 1], out[:, 2] > 0


def to_dev_f64(x, dev=None):
    """Host array-like / tensor -> contiguous float64 CUDA tensor."""
    dev = dev or device()
    if isinstance(x, torch.Tensor):
        return x.to(device=dev, dtype=torch.float64).contiguous()
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    if not a.flags.writeable:
        a = a.copy()
    return torch.from_numpy(a).to(dev, non_blocking=False)


def as_real_batch(c):
    """Split coefficients into a real (B, N) float64 device tensor.

    Returns (tensor, meta) where meta records how to rebuild the caller's
    shape/dtype: complex inputs become two real rows (real, imag) per vector
    (the transforms are real-linear, test_schlomilch.py:256-264).
    """
    is_torch = isinstance(c, torch.Tensor)
    host_tensor = is_torch and c.device.type == "cpu"
    if is_torch:
        cplx = c.is_complex()
        arr = c.to(device(), non_blocking=True) if host_tensor else c
    else:
        arr = np.asarray(c)
        cplx = np.iscomplexobj(arr)
        if not cplx and not np.issubdtype(arr.dtype, np.floating):
            arr = arr.astype(np.float64)
    one = arr.ndim == 1
    if arr.ndim not in (1, 2):
        raise ValueError("coefficients must be a vector or a (batch, N) matrix")
    dev = device()
    if cplx:
        if is_torch:
            t = arr.to(dev)
            t = t.reshape(-1, t.shape[-1])
            both = torch.stack([t.real, t.imag], dim=1).reshape(-1, t.shape[-1])
            realt = both.to(torch.float64).contiguous()
        else:
            a2 = arr.reshape(-1, arr.shape[-1])
            both = np.stack([a2.real, a2.imag], axis=1).reshape(-1, arr.shape[-1])
            realt = to_dev_f64(both, dev)
    else:
        realt = to_dev_f64(arr.reshape(-1, arr.shape[-1]) if not is_torch else arr.reshape(-1, arr.shape[-1]), dev)
    return realt, dict(torch=is_torch, host_tensor=host_tensor, complex=cplx, one=one)


def from_real_batch(F, meta):
    """Inverse of as_real_batch for the (B', n_out) result tensor."""
    if meta["complex"]:
        F = F.reshape(-1, 2, F.shape[-1])
        F = torch.complex(F[:, 0], F[:, 1])
    if meta["one"]:
        F = F[0]
    if meta.get("host_tensor"):
        out = torch.empty(F.shape, dtype=F.dtype, pin_memory=True)
        out.copy_(F, non_blocking=False)
        return out
    if meta["torch"]:
        return F
    return F.cpu().numpy()
