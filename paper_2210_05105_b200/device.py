"""Device plumbing: CUDA tensors, streams, and the device status word.

PyTorch provides device memory, streams and torch.distributed; all arithmetic on the hot
path runs in librandcp_b200.so.  There is no CPU fallback: `require_cuda()` raises when
no CUDA device is visible.
"""

from __future__ import annotations

import os

import numpy as np

from . import _lib

# Debug: RCP_POISON=1 fills every uninitialised device allocation of the package (and the
# allocator's cached blocks, see poison_allocator) with 0xFF bytes -- NaN as fp64, -1 as
# integers -- so a kernel that reads memory it never wrote fails deterministically instead
# of depending on what the previous user of that memory left there.
POISON = os.environ.get("RCP_POISON", "") == "1"

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


def empty(shape, dtype, dev):
    """Uninitialised device tensor (0xFF-filled under RCP_POISON=1)."""
    t = torch()
    x = t.empty(shape, dtype=dtype, device=dev)
    if POISON:
        x.view(t.uint8).fill_(0xFF) if x.numel() else None
    return x


def poison_allocator(dev, large_gb=8, small_mb=512):
    """Fill a large block and many small blocks of the caching allocator with 0xFF and
    release them: later torch.empty() calls are carved from poisoned memory."""
    t = torch()
    big = t.empty(int(large_gb * (1 << 30)), dtype=t.uint8, device=dev)
    big.fill_(0xFF)
    smalls = []
    for _ in range(max(1, (small_mb << 20) >> 19)):   # 512 KB blocks: the small pool
        x = t.empty(1 << 19, dtype=t.uint8, device=dev)
        x.fill_(0xFF)
        smalls.append(x)
    t.cuda.synchronize()
    del big, smalls


def f64(shape, dev, fill=None):
    t = torch()
    if fill is None:
        return empty(shape, t.float64, dev)
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

    # Causal order: a flag raised upstream (sampler, workspace) explains everything the
    # same solve computed after it, so it is reported before the downstream ones (a
    # degenerate walk leaves its samples' rows unset, which the update then sees as
    # non-finite factors).  The raw word is part of every message.
    _ORDER = (
        ("ST_CAPACITY", RuntimeError, "sampled-MTTKRP workspace too small"),
        ("ST_TIMEOUT", RuntimeError, "device work queue watchdog expired"),
        ("ST_ASYMMETRIC", ValueError, "matrix is not symmetric"),
        ("ST_ZERO_MASS", ValueError, "zero total leverage mass; nothing to sample from"),
        ("ST_DEGENERATE", DegenerateWalkError, "zero-mass node in leverage tree walk"),
        ("ST_ZERO_PROB", ValueError, "sample with zero probability cannot have been drawn"),
        ("ST_NONFINITE", FloatingPointError, "non-finite factor entries"),
    )

    def peek(self):
        return int(self.buf.item())

    def check(self, where=""):
        v = int(self.buf.item())
        if not v:
            return
        self.buf.zero_()
        flags = [name for name, _, _ in self._ORDER if v & getattr(_lib, name)]
        for name, exc, msg in self._ORDER:
            if v & getattr(_lib, name):
                raise exc("%s %s (device status 0x%x: %s)" % (msg, where, v, "|".join(flags)))
        raise RuntimeError("device status 0x%x %s" % (v, where))
