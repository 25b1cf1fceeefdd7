"""Mode-j matricized views backed by the device sorted store (drop-in for the
reference's Matricization / matricize / partition_to_grid, ref matricization.py).

A `Matricization` keeps the host coordinates (for API compatibility) and builds its
device `store.DeviceStore` on first use; `partition_to_grid` implements the
accumulator-stationary partition (one mode-aligned copy per rank and mode, ref
matricization.py:187-198).  The tensor-stationary schedule is out of scope for this build
 and raises.
"""

from __future__ import annotations

import numpy as np

from .coo import SparseTensorCOO
from .device import require_cuda, to_dev, torch
from .store import build_store, off_mode_strides


def column_keys(idx, dims, skip):
    """Off-mode mixed-radix key per entry (ref matricization.py:41-54), int64 only."""
    strides, exact = off_mode_strides(dims, skip)
    if not exact:
        raise ValueError("off-mode key space exceeds 2^62; not supported by the device store")
    idx = np.asarray(idx, dtype=np.int64)
    keys = np.zeros(idx.shape[0], dtype=np.int64)
    for m, s in enumerate(strides):
        if m != skip:
            keys += idx[:, m] * np.int64(s)
    return keys


class Matricization:
    def __init__(self, dims, idx, vals, mode, row_lo=0, row_hi=None):
        self.dims = tuple(int(d) for d in dims)
        self.mode = int(mode)
        self.idx = np.ascontiguousarray(idx, dtype=np.int64)
        self.vals = np.ascontiguousarray(vals, dtype=np.float64)
        self.row_lo = int(row_lo)
        self.row_hi = int(self.dims[mode] if row_hi is None else row_hi)
        rel = self.idx[:, self.mode] - self.row_lo
        if rel.size and (rel.min() < 0 or rel.max() >= self.n_rows):
            raise ValueError("entry rows outside block [%d, %d)" % (self.row_lo, self.row_hi))
        self._store = None

    @property
    def nnz(self):
        return int(self.vals.size)

    @property
    def n_rows(self):
        return self.row_hi - self.row_lo

    @property
    def store(self):
        if self._store is None:
            dev = require_cuda()
            t = torch()
            self._store = build_store(self.dims, to_dev(self.idx, dev, t.int64),
                                      to_dev(self.vals, dev, t.float64), self.mode,
                                      self.row_lo, self.row_hi)
        return self._store

    def lookup_columns(self, query_keys):
        """(lo, hi) positions of each query key in (key, row) order (ref
        matricization.py:112-121)."""
        t = torch()
        st = self.store
        q = to_dev(np.asarray(query_keys, dtype=np.int64), st.keys.device, t.int64)
        c = t.searchsorted(st.keys, q)
        cc = c.clamp(max=max(st.n_cols - 1, 0))
        hit = (c < st.n_cols) & (st.keys[cc] == q) if st.n_cols else t.zeros_like(q, dtype=t.bool)
        lo = st.colptr[c]
        hi = t.where(hit, st.colptr[(c + 1).clamp(max=st.n_cols)], lo)
        return lo.cpu().numpy(), hi.cpu().numpy()


def matricize(t: SparseTensorCOO, mode: int) -> Matricization:
    if not 0 <= mode < t.mode_count:
        raise ValueError("mode %d out of range for %d-mode tensor" % (mode, t.mode_count))
    return Matricization(t.dims, t.idx, t.vals, mode)


class LocalTensorSet:
    def __init__(self, schedule, grid, mats):
        self.schedule = schedule
        self.grid = grid
        self.mats = mats

    def local(self, rank, mode) -> Matricization:
        return self.mats[rank][mode]

    def stored_nnz(self) -> int:
        return sum(m.nnz for per_rank in self.mats for m in per_rank)


def partition_to_grid(t: SparseTensorCOO, grid, schedule: str) -> LocalTensorSet:
    if tuple(grid.tensor_dims) != tuple(t.dims):
        raise ValueError("grid built for dims %s, tensor has %s" % (grid.tensor_dims, t.dims))
    if schedule == "tensor-stationary":
        from .schedules import ScheduleError
        raise ScheduleError("tensor-stationary schedule is not part of this build (the "
                            "accumulator-stationary schedule is the hot path)")
    if schedule != "accumulator-stationary":
        raise ValueError("unknown schedule %r" % schedule)
    mats = [[None] * t.mode_count for _ in range(grid.P)]
    for j in range(t.mode_count):
        own = grid.row_owner(j, t.idx[:, j])
        for p in range(grid.P):
            sel = np.nonzero(own == p)[0]
            lo, hi = grid.block_range(j, p)
            mats[p][j] = Matricization(t.dims, t.idx[sel], t.vals[sel], j, row_lo=lo, row_hi=hi)
    return LocalTensorSet(schedule, grid, mats)
