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
    # (key, row) order: stable radix sort by row, then by key (csrc/sort.cu)
    span = 1
    for m, d in enumerate(dims):
        if m != mode:
            span *= d
    rows = rows.contiguous()
    from .ops import ops_for
    order = ops_for(dev).order_by_key_row(key, rows, span - 1, dims[mode] - 1)
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


def build_store_chunks(dims, chunks, mode, row_lo=0, row_hi=None, buckets=16):
    """Mode-`mode` store from a list of device COO chunks (idx int32/int64 [n, N], vals):
    the device-ingest path for tensors whose int64 COO would not fit (C4/C5).  Entries are
    bucketed by column-key range (a column never straddles two buckets), each bucket is
    ordered by (key, row) with two stable sorts and written at its offset, so the working
    set beyond the store itself is one bucket.  Same layout as build_store."""
    t = torch()
    dims = tuple(int(d) for d in dims)
    N = len(dims)
    row_hi = dims[mode] if row_hi is None else int(row_hi)
    strides, exact = off_mode_strides(dims, mode)
    if not exact:
        raise ValueError("off-mode key space of mode %d exceeds 2^62" % mode)
    span = 1
    for m in range(N):
        if m != mode:
            span *= dims[m]
    dev = chunks[0][0].device if chunks else t.device("cuda", 0)
    B = max(1, int(buckets))
    from .ops import ops_for
    _ops = ops_for(dev)

    def keyed(idx, vals):
        rows = idx[:, mode].long()
        sel = (rows >= row_lo) & (rows < row_hi)
        fk = t.zeros(idx.shape[0], dtype=t.int64, device=dev)
        for m in range(N):
            if m != mode:
                fk += idx[:, m].long() * int(strides[m])
        return fk, rows, sel

    counts = t.zeros(B, dtype=t.int64, device=dev)
    for idx, vals in chunks:
        fk, rows, sel = keyed(idx, vals)
        counts += t.bincount((fk[sel] * B) // span, minlength=B)
        del fk, rows, sel
    total = int(counts.sum())
    out_rows = t.empty(total, dtype=t.int32, device=dev)
    out_vals = t.empty(total, dtype=t.float64, device=dev)
    keys_l, cnt_l = [], []
    off = 0
    max_col = 0
    for b in range(B):
        parts = []
        for idx, vals in chunks:
            fk, rows, sel = keyed(idx, vals)
            sel &= (fk * B) // span == b
            parts.append((fk[sel], rows[sel], vals[sel]))
            del fk, rows, sel
        fk = t.cat([p[0] for p in parts])
        rows = t.cat([p[1] for p in parts])
        vals = t.cat([p[2] for p in parts])
        del parts
        n = fk.numel()
        if n == 0:
            continue
        order = _ops.order_by_key_row(fk, rows.contiguous(), span - 1, dims[mode] - 1)
        out_rows[off:off + n] = (rows[order] - row_lo).to(t.int32)
        out_vals[off:off + n] = vals[order]
        uk, c = t.unique_consecutive(fk[order], return_counts=True)
        del order, fk, rows, vals
        keys_l.append(uk)
        cnt_l.append(c)
        max_col = max(max_col, int(c.max()))
        off += n
    if keys_l:
        keys = t.cat(keys_l)
        cnts = t.cat(cnt_l)
    else:
        keys = t.zeros(0, dtype=t.int64, device=dev)
        cnts = t.zeros(0, dtype=t.int64, device=dev)
    del keys_l, cnt_l
    colptr = t.zeros(keys.numel() + 1, dtype=t.int64, device=dev)
    t.cumsum(cnts, 0, out=colptr[1:])
    return DeviceStore(dims, mode, row_lo, row_hi, keys.contiguous(), colptr, out_rows, out_vals,
                       max_col)
