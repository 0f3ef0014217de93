"""DCT-I / DST-I application (drop-in for fasthankel.trig, reference
trig.py).  The transform runs on the GPU as a chirp-z convolution on
shared-memory radix FFTs (libfhtb200.so, fhtb_chirp.cu)."""

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device, _lib

__all__ = ["DCT1", "DST1", "TransformPlan", "make_plan", "apply"]

DCT1 = "dct1"
DST1 = "dst1"


@dataclass(frozen=True)
class TransformPlan:
    """Plan for C (DCT-I) or S (DST-I) of a fixed size (trig.py:24-35)."""

    length: int
    kind: str
    _weights: np.ndarray = field(repr=False, default=None)


def make_plan(length, kind):
    """DCT-I needs length >= 2, DST-I length >= 1 (trig.py:38-56)."""
    if kind == DCT1:
        if length < 2:
            raise ValueError("DCT-I needs length >= 2")
        w = np.full(length, 0.5)
        w[0] = 1.0
        w[-1] = 1.0
        w.flags.writeable = False
        return TransformPlan(length=length, kind=DCT1, _weights=w)
    if kind == DST1:
        if length < 1:
            raise ValueError("DST-I needs length >= 1")
        return TransformPlan(length=length, kind=DST1)
    raise ValueError("kind must be DCT1 or DST1")


def apply(plan, v):
    """Apply the planned matrix along the last axis (trig.py:80-92)."""
    is_t = isinstance(v, torch.Tensor)
    arr = v if is_t else np.asarray(v)
    if arr.shape[-1] != plan.length:
        raise ValueError("vector length %d does not match plan length %d" % (arr.shape[-1], plan.length))
    if not is_t and not np.issubdtype(arr.dtype, np.inexact):
        arr = arr.astype(float)
    shape = tuple(arr.shape)
    cplx = arr.is_complex() if is_t else np.iscomplexobj(arr)
    flat = arr.reshape(-1, plan.length)
    _device.ensure_init()
    C, meta = _device.as_real_batch(flat)
    out = torch.empty_like(C)
    kind = _lib.FHTB_DCT1 if plan.kind == DCT1 else _lib.FHTB_DST1
    lib = _lib.load()
    ws_n = lib.fhtb_trig_workspace(kind, plan.length, C.shape[0])
    if ws_n == 0:
        _lib.check(lib.fhtb_trig_apply(kind, plan.length, None, 0, None, None, 0, None))
    ws = _device.workspace(ws_n)
    _lib.check(lib.fhtb_trig_apply(kind, plan.length, _device.ptr(C), C.shape[0], _device.ptr(out),
                                   _device.ptr(ws), ws.numel(), _device.stream_ptr()))
    res = _device.from_real_batch(out, dict(meta, one=False))
    if is_t:
        return res.reshape(shape)
    res = res.reshape(shape)
    if not cplx:
        res = res.astype(np.float64)
    return res
