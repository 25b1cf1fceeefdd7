"""Device plumbing: CUDA tensors, streams, and the device status word.

PyTorch provides device memory, streams and torch.distributed; all arithmetic on the hot
path runs in librandcp_b200.so.  There is no CPU fallback: `require_cuda()` raises when
no CUDA device is visible.
"""

from __future__ import annotations

import numpy as np

from . import _lib

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t
        _torch = t
    return _torch


class DegenerateWalkError(RuntimeError):
    """A tree walk hit a zero-mass node; h lies outside the row space
    (ref samplers.py:34-35)."""


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError("randcp_b200 needs a CUDA device (B200, sm_100a); there is no CPU "
                           "fallback on the product path")
    _lib.load()
    return t.device("cuda", t.cuda.current_device())


def ptr(x):
    """Raw data pointer of a torch tensor (None -> NULL)."""
    if x is None:
        return None
    return x.data_ptr()


def stream_handle():
    return torch().cuda.current_stream().cuda_stream


def f64(shape, dev, fill=None):
    t = torch()
    if fill is None:
        return t.empty(shape, dtype=t.float64, device=dev)
    return t.full(shape, float(fill), dtype=t.float64, device=dev)


def to_dev(a, dev, dtype=None):
    t = torch()
    if isinstance(a, t.Tensor):
        out = a.to(dev)
        return out.contiguous() if dtype is None else out.to(dtype).contiguous()
    arr = np.ascontiguousarray(a)
    out = t.from_numpy(arr).to(dev)
    if dtype is not None:
        out = out.to(dtype)
    return out.contiguous()


def to_host(x):
    return x.detach().cpu().numpy()


class Status:
    """One device int32 holding OR-ed RCP_ST_* flags raised by kernels."""

    def __init__(self, dev):
        t = torch()
        self.buf = t.zeros(1, dtype=t.int32, device=dev)

    @property
    def ptr(self):
        return self.buf.data_ptr()

    def reset(self):
        self.buf.zero_()

    def clear_flag(self, flag):
        self.buf.bitwise_and_(~int(flag))

    def check(self, where=""):
        v = int(self.buf.item())
        if not v:
            return
        self.buf.zero_()
        if v & _lib.ST_NONFINITE:
            raise FloatingPointError("non-finite factor entries %s" % where)
        if v & _lib.ST_DEGENERATE:
            raise DegenerateWalkError("zero-mass node in leverage tree walk %s" % where)
        if v & _lib.ST_ASYMMETRIC:
            raise ValueError("matrix is not symmetric %s" % where)
        if v & _lib.ST_ZERO_MASS:
            raise ValueError("zero total leverage mass; nothing to sample from %s" % where)
        if v & _lib.ST_ZERO_PROB:
            raise ValueError("sample with zero probability cannot have been drawn %s" % where)
        if v & _lib.ST_TIMEOUT:
            raise RuntimeError("device work queue watchdog expired %s" % where)
        if v & _lib.ST_CAPACITY:
            raise RuntimeError("sampled-MTTKRP workspace too small %s" % where)
        raise RuntimeError("device status 0x%x %s" % (v, where))
