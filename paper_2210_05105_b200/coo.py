"""Minimal coordinate-format tensor container used by the drop-in API.

The container carries (dims, idx, vals) with the reference's validation rules (ref
tensor.py:22-69) so the AS partition and ALS driver take the same inputs as the
reference; FROSTT parsing and result files live in tensorio.py.
"""

from __future__ import annotations

import numpy as np


class BoundsError(ValueError):
    """Index outside the declared mode dimensions (ref tensor.py:18-19)."""


class SparseTensorCOO:
    __slots__ = ("dims", "idx", "vals")

    def __init__(self, dims, idx, vals, validate=True):
        self.dims = tuple(int(d) for d in dims)
        self.idx = np.ascontiguousarray(idx, dtype=np.int64)
        self.vals = np.ascontiguousarray(vals, dtype=np.float64)
        if not validate:
            return
        if len(self.dims) < 3:
            raise ValueError("tensor needs at least 3 modes, got %d" % len(self.dims))
        if min(self.dims) <= 0:
            raise ValueError("mode dimensions must be positive: %s" % (self.dims,))
        if self.idx.ndim != 2 or self.idx.shape[1] != len(self.dims):
            raise ValueError("index matrix shape %s does not match %d modes"
                             % (self.idx.shape, len(self.dims)))
        if self.vals.shape != (self.idx.shape[0],):
            raise ValueError("value count %d != index row count %d"
                             % (self.vals.size, self.idx.shape[0]))
        if self.idx.size and (self.idx.min() < 0 or (self.idx >= np.asarray(self.dims)).any()):
            raise BoundsError("tensor index out of bounds for dims %s" % (self.dims,))

    @property
    def mode_count(self):
        return len(self.dims)

    @property
    def nnz(self):
        return int(self.vals.size)

    def norm_squared(self):
        return float(np.dot(self.vals, self.vals))


class ModePermutations:
    """Per-mode bijections (identity by default) used to un-permute output factors
    (ref tensor.py:170-197)."""

    def __init__(self, perms, seed=None):
        self.perms = [np.ascontiguousarray(p, dtype=np.int64) for p in perms]
        self.seed = seed

    @classmethod
    def identity(cls, dims):
        return cls([np.arange(int(d), dtype=np.int64) for d in dims])

    @classmethod
    def random(cls, dims, seed):
        from . import rng
        return cls([rng.permutation(rng.stream_key(seed, rng.TENSOR_PERM, j), int(d))
                    for j, d in enumerate(dims)], seed=seed)

    def unpermute_factor(self, U, mode):
        return U[self.perms[mode]]


def apply_permutations(t: SparseTensorCOO, mp: ModePermutations):
    """idx'[:, j] = perm_j[idx[:, j]] for every mode (ref tensor.py:199-205)."""
    idx = np.empty_like(t.idx)
    for j, p in enumerate(mp.perms):
        idx[:, j] = p[t.idx[:, j]]
    return SparseTensorCOO(t.dims, idx, t.vals.copy(), validate=False)


def permute_modes(t: SparseTensorCOO, seed):
    """Load-balancing random relabelling of every mode (ref tensor.py:182-210)."""
    mp = ModePermutations.random(t.dims, seed)
    return apply_permutations(t, mp), mp
