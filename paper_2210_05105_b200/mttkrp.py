"""Sampled-nonzero gather and downsampled MTTKRP -- drop-ins for the reference's
mttkrp.py (ref mttkrp.py:111-189), on the GPU.

`gather_sampled_nonzeros_to_csr` returns exactly the reference's CSR (with sample
multiplicity, rows ascending, sample ids ascending inside a row).  `downsampled_mttkrp`
is the CSR segmented SpMM kernel.  The ALS engine does not materialise this CSR: it runs
the fused, deduplicated pipeline `rcp_sampled_mttkrp` directly from the sample matrix.
"""

from __future__ import annotations

import numpy as np

from .device import require_cuda, to_dev, to_host, torch
from .matricization import Matricization
from .ops import ops_for


class SampledCsr:
    """(ref mttkrp.py:111-128)"""

    def __init__(self, row_ptr, col_idx, vals, n_rows, n_cols):
        self.row_ptr = row_ptr
        self.col_idx = col_idx
        self.vals = vals
        self.n_rows = int(n_rows)
        self.n_cols = int(n_cols)

    @property
    def nnz(self):
        return self.vals.size


def _x_dev(X, dev):
    t = torch()
    Xh = np.ascontiguousarray(np.asarray(X, dtype=np.int64).T)   # mode-major (N, J)
    return to_dev(Xh, dev, t.int64)


def gather_sampled_nonzeros_to_csr(mat: Matricization, X, k) -> SampledCsr:
    """(ref mttkrp.py:131-155)"""
    if mat.mode != k:
        raise ValueError("matricization is for mode %d, expected %d" % (mat.mode, k))
    X = np.asarray(X)
    J = X.shape[0]
    n_rows = mat.n_rows
    if J == 0 or mat.nnz == 0:
        return SampledCsr(np.zeros(n_rows + 1, dtype=np.int64), np.empty(0, dtype=np.int64),
                          np.empty(0), n_rows, J)
    dev = require_cuda()
    t = torch()
    ops = ops_for(dev)
    st = mat.store
    Xd = _x_dev(X, dev)
    lo = t.empty(J, dtype=t.int64, device=dev)
    cnt = t.empty(J, dtype=t.int64, device=dev)
    ops.fiber_lookup(st, Xd, k, lo, cnt)
    off = t.zeros(J + 1, dtype=t.int64, device=dev)
    t.cumsum(cnt, 0, out=off[1:])
    nnz = int(off[-1].item())
    if nnz == 0:
        return SampledCsr(np.zeros(n_rows + 1, dtype=np.int64), np.empty(0, dtype=np.int64),
                          np.empty(0), n_rows, J)
    ro = t.empty(nnz, dtype=t.int64, device=dev)
    co = t.empty(nnz, dtype=t.int64, device=dev)
    vo = t.empty(nnz, dtype=t.float64, device=dev)
    ops.fiber_expand(lo, off, st, ro, co, vo)
    order = ops.order_by_key_row(None, ro, 0, n_rows - 1)   # the counting-sort "sparse transpose"
    ro = ro[order]
    rp = t.zeros(n_rows + 1, dtype=t.int64, device=dev)
    t.cumsum(t.bincount(ro, minlength=n_rows), 0, out=rp[1:])
    return SampledCsr(to_host(rp), to_host(co[order]), to_host(vo[order]), n_rows, J)


def downsampled_mttkrp(csr: SampledCsr, H_rows, weights, workers=1):
    """out[i,:] = sum_s (w_s csr[i,s]) (w_s H[s,:]) (ref mttkrp.py:158-189)."""
    H_rows = np.asarray(H_rows, dtype=np.float64)
    weights = np.asarray(weights, dtype=np.float64)
    if H_rows.shape[0] != csr.n_cols or weights.shape != (csr.n_cols,):
        raise ValueError("H_rows/weights do not match the %d sampled columns" % csr.n_cols)
    R = H_rows.shape[1]
    if csr.nnz == 0 or csr.n_rows == 0:
        return np.zeros((csr.n_rows, R))
    dev = require_cuda()
    t = torch()
    ops = ops_for(dev)
    w = to_dev(weights, dev, t.float64)
    out = t.empty((csr.n_rows, R), dtype=t.float64, device=dev)
    ops.csr_spmm(to_dev(csr.row_ptr, dev, t.int64), to_dev(csr.col_idx, dev, t.int64),
                 to_dev(csr.vals, dev, t.float64), to_dev(H_rows, dev, t.float64), w * w, out)
    return to_host(out)


def mttkrp_exact(mat: Matricization, factors, offsets=None, workers=1):
    """Exact local MTTKRP (ref mttkrp.py:65-108): out[i_j - row_lo] += v * prod of the
    other factors' rows.  Device gathers + index_add (outside the sampled hot path)."""
    j = mat.mode
    R = next(f.shape[1] for i, f in enumerate(factors) if i != j and f is not None)
    if offsets is None:
        offsets = [0] * len(factors)
    for i, f in enumerate(factors):
        if i == j or f is None:
            continue
        lo_need = mat.idx[:, i].min(initial=offsets[i])
        hi_need = mat.idx[:, i].max(initial=offsets[i] - 1) + 1
        if lo_need < offsets[i] or hi_need > offsets[i] + f.shape[0]:
            raise ValueError("mode-%d rows [%d, %d) not covered by gathered block"
                             % (i, lo_need, hi_need))
    if mat.nnz == 0:
        return np.zeros((mat.n_rows, R))
    dev = require_cuda()
    t = torch()
    facs = [to_dev(np.ascontiguousarray(f, dtype=np.float64), dev, t.float64)
            if (i != j and f is not None) else None for i, f in enumerate(factors)]
    out = t.empty((mat.n_rows, R), dtype=t.float64, device=dev)
    ops_for(dev).exact_mttkrp(mat.store, facs, offsets, out)
    return to_host(out)


def set_mttkrp_mode(deterministic):
    """Select the fused sampled MTTKRP's mode for subsequent solves (process-wide):
    deterministic=True runs the row-tile x fiber pair path, whose every output row is
    summed in a fixed order (bit-identical results run to run, like the reference's
    worker-count invariance, ref tests/test_mttkrp.py:60-67,163-172); False the faster
    row-transpose path.  Returns the previous setting (C ABI rcp_set_mttkrp_mode)."""
    from . import _lib
    return bool(_lib.lib().rcp_set_mttkrp_mode(1 if deterministic else 0))


class deterministic_mttkrp:
    """Context manager: deterministic sampled MTTKRP inside the block."""

    def __init__(self, on=True):
        self.on = on

    def __enter__(self):
        self.prev = set_mttkrp_mode(self.on)
        return self

    def __exit__(self, *exc):
        set_mttkrp_mode(self.prev)
        return False
