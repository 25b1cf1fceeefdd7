"""Device-resident per-mode sorted nonzero store (the CSC analogue the sampled MTTKRP
gathers from).

Layout of one mode-j store on the GPU that owns rows [row_lo, row_hi):

    keys   int64 [n_cols]     distinct off-mode column keys, ascending
    colptr int64 [n_cols+1]   column c's nonzeros at [colptr[c], colptr[c+1])
    rows   int32 [nnz]        row - row_lo, ascending inside a column
    vals   fp64  [nnz]

12 bytes per nonzero plus 16 bytes per distinct column.  Column keys are the reference's
mixed-radix off-mode encoding with earlier modes varying fastest (ref
matricization.py:21-64); the sort order (key, row) is the reference's `col_order`
(ref matricization.py:95-100).  Built once per run with device sorts (torch), outside
the per-solve loop (the reference's equivalent is its one-time lexsort, "load" phase).
"""

from __future__ import annotations

import numpy as np

from .device import torch

INT64_SAFE = 1 << 62   # ref matricization.py:18


def off_mode_strides(dims, skip):
    """Mixed-radix strides over modes != skip (earlier modes fastest); `exact` is False
    when the key space exceeds 2^62 (ref matricization.py:21-38)."""
    strides = [0] * len(dims)
    span = 1
    for m, d in enumerate(dims):
        if m != skip:
            strides[m] = span
            span *= int(d)
    return strides, span <= INT64_SAFE


class DeviceStore:
    def __init__(self, dims, mode, row_lo, row_hi, keys, colptr, rows, vals, max_col):
        self.dims = tuple(int(d) for d in dims)
        self.mode = int(mode)
        self.row_lo = int(row_lo)
        self.row_hi = int(row_hi)
        self.keys, self.colptr, self.rows, self.vals = keys, colptr, rows, vals
        self.max_col = int(max_col)
        self.strides, _ = off_mode_strides(self.dims, self.mode)

    @property
    def n_rows(self):
        return self.row_hi - self.row_lo

    @property
    def n_cols(self):
        return int(self.keys.shape[0])

    @property
    def nnz(self):
        return int(self.vals.shape[0])

    def capacity(self, J):
        """Upper bound on gathered nonzeros of J distinct sampled fibers."""
        return min(self.nnz, int(J) * max(self.max_col, 1))

    def bytes(self):
        return (self.keys.numel() * 8 + self.colptr.numel() * 8 + self.rows.numel() * 4 +
                self.vals.numel() * 8)


def column_keys_dev(idx, dims, mode):
    t = torch()
    strides, exact = off_mode_strides(dims, mode)
    if not exact:
        raise ValueError("off-mode key space of mode %d exceeds 2^62 (object keys are not "
                         "supported on the device path)" % mode)
    key = t.zeros(idx.shape[0], dtype=t.int64, device=idx.device)
    for m, s in enumerate(strides):
        if m != mode:
            key += idx[:, m] * int(s)
    return key


def build_store(dims, idx, vals, mode, row_lo=0, row_hi=None):
    """idx: (nnz, N) int64 CUDA tensor of global coordinates, vals: (nnz,) fp64."""
    t = torch()
    dims = tuple(int(d) for d in dims)
    row_hi = dims[mode] if row_hi is None else int(row_hi)
    dev = idx.device
    n = idx.shape[0]
    if n == 0:
        z = t.zeros(0, dtype=t.int64, device=dev)
        return DeviceStore(dims, mode, row_lo, row_hi, z, t.zeros(1, dtype=t.int64, device=dev),
                           t.zeros(0, dtype=t.int32, device=dev),
                           t.zeros(0, dtype=t.float64, device=dev), 0)
    rows = idx[:, mode]
    if int(rows.min()) < row_lo or int(rows.max()) >= row_hi:
        raise ValueError("entry rows outside block [%d, %d)" % (row_lo, row_hi))
    key = column_keys_dev(idx, dims, mode)
    # (key, row) order: stable sort by row, then stable sort by key
    o1 = t.sort(rows, stable=True).indices
    o2 = t.sort(key[o1], stable=True).indices
    order = o1[o2]
    del o1, o2
    skeys = key[order]
    del key
    ukeys, counts = t.unique_consecutive(skeys, return_counts=True)
    del skeys
    colptr = t.zeros(ukeys.shape[0] + 1, dtype=t.int64, device=dev)
    t.cumsum(counts, 0, out=colptr[1:])
    max_col = int(counts.max()) if counts.numel() else 0
    lrows = (rows[order] - row_lo).to(t.int32)
    lvals = vals[order].to(t.float64).contiguous()
    return DeviceStore(dims, mode, row_lo, row_hi, ukeys.contiguous(), colptr, lrows.contiguous(),
                       lvals, max_col)
