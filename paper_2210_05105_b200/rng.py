"""Deterministic random-stream discipline (mirror of ref rng.py:1-32).

Every draw on the hot path comes from a counter-based Philox4x64-10 stream keyed by
(seed, purpose, *context).  The key derivation (numpy SeedSequence) and the buffered
uint32 permutation run in native code (librandcp_b200.so); the draws themselves are
generated on the device inside the sampler kernels, so the CUDA path consumes exactly the
uniforms numpy's ``Generator(Philox(SeedSequence(...)))`` would.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib

# Purpose codes -- identical numbering to the reference (ref rng.py:17-23).
INIT = 0
TENSOR_PERM = 1
MULTINOMIAL = 2
LOCAL_DRAW = 3
SHUFFLE = 4
WALK_UNIFORM = 5
GENERIC = 6


def stream_key(seed, purpose, *context):
    """(k0, k1): the Philox key of stream (seed, purpose, *context)."""
    ctx = np.array([int(c) for c in context], dtype=np.uint64)
    out = np.zeros(2, dtype=np.uint64)
    _lib.call("rcp_stream_key", C.c_uint64(int(seed) & 0xFFFFFFFFFFFFFFFF),
              C.c_uint64(int(purpose)), ctx.ctypes.data if ctx.size else None,
              int(ctx.size), out.ctypes.data)
    return int(out[0]), int(out[1])


def uniforms_host(key, n, first=0):
    """Generator.random() draws [first, first+n) of a stream (host, for tests/tools)."""
    k = np.array(key, dtype=np.uint64)
    out = np.empty(int(n), dtype=np.float64)
    _lib.call("rcp_uniform_host", k.ctypes.data, int(first), int(n), out.ctypes.data)
    return out


def permutation(key, n):
    """Generator.permutation(n) of a stream (host native code)."""
    k = np.array(key, dtype=np.uint64)
    out = np.empty(int(n), dtype=np.int64)
    _lib.call("rcp_permutation_host", k.ctypes.data, int(n), out.ctypes.data)
    return out


def stream(seed, purpose, *context) -> np.random.Generator:
    """numpy Generator for a key -- used only for the P-sized multinomial split and the
    host-side factor initialisation, exactly as the reference does (ref rng.py:26-32)."""
    key = np.random.SeedSequence(entropy=int(seed) & ((1 << 64) - 1),
                                 spawn_key=(int(purpose),) + tuple(int(c) for c in context))
    return np.random.Generator(np.random.Philox(key))


def permutations_into(keys, n, outs, threads=8):
    """Generator.permutation(n) of several streams at once (native threads), written into
    the int64 buffers `outs` (numpy arrays or CPU tensors, n elements each)."""
    k = np.ascontiguousarray(np.asarray(keys, dtype=np.uint64).reshape(-1, 2))
    ptrs = (C.c_void_p * len(outs))(*[C.c_void_p(o.data_ptr() if hasattr(o, "data_ptr")
                                                 else o.ctypes.data) for o in outs])
    _lib.call("rcp_permutations_host", k.ctypes.data, len(outs), int(n), ptrs, int(threads))
