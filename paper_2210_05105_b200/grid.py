"""Rank layout and factor-row ownership for the accumulator-stationary schedule.

Mirrors the ownership semantics of the reference processor grid (ref grid.py:32-156):
P ranks in a Cartesian grid P_1 x ... x P_N; mode j's rows are cut into P_j near-equal
chunks, and each chunk is re-cut among the ranks sharing that chunk coordinate, in rank
order.  CP-ARLS-LEV draws at P > 1 depend on this map (per-rank streams, rank-order
gather), so parity runs must use it verbatim.  The simulated collectives and the ledger
of the reference are not reproduced -- real collectives run over NCCL (dist.py); only
the closed-form traffic model is kept so measured bytes can be checked against it.
"""

from __future__ import annotations

import itertools

import numpy as np


def balanced_offsets(n, parts):
    """Cut range(n) into `parts` contiguous pieces whose sizes differ by at most one,
    larger pieces first (ref grid.py:32-39)."""
    n, parts = int(n), int(parts)
    q, extra = divmod(n, parts)
    return np.array([i * q + min(i, extra) for i in range(parts + 1)], dtype=np.int64)


def weighted_offsets(w, parts):
    """Cut range(len(w)) into `parts` contiguous pieces minimising the largest piece weight
    (binary search on the bound, greedy longest pieces; an nnz-balanced alternative to
    balanced_offsets for performance runs).  Pieces may be empty."""
    w = np.asarray(w, dtype=np.float64)
    n, parts = int(w.size), int(parts)
    cum = np.concatenate([[0.0], np.cumsum(w)])
    if n == 0 or cum[-1] <= 0.0 or parts <= 1:
        return balanced_offsets(n, parts)

    def cut(L):
        off = [0]
        for _ in range(parts - 1):
            s = off[-1]
            e = int(np.searchsorted(cum, cum[s] + L, side="right")) - 1
            off.append(min(max(e, s), n))
        off.append(n)
        return off, cum[n] - cum[off[-2]] <= L

    lo, hi = float(w.max()), float(cum[-1])
    for _ in range(60):
        mid = 0.5 * (lo + hi)
        if cut(mid)[1]:
            hi = mid
        else:
            lo = mid
    return np.array(cut(hi)[0], dtype=np.int64)


class ProcessorGrid:
    """Ownership map only: per mode and rank, the global row block [lo, hi).

    row_weights (optional, one array of per-row weights per mode, e.g. nonzeros per row):
    cut every mode's chunks and slice-group blocks at equal weight instead of equal row
    counts (Zipf head rows cannot move under the AS schedule, so equal-row
    blocks leave one GPU with ~1.5x its share at C4).  Parity runs use the reference's
    equal-row cuts (row_weights=None); CP-ARLS-LEV draws at P > 1 depend on them."""

    def __init__(self, tensor_dims, grid_dims, warning=False, row_weights=None):
        self.tensor_dims = tuple(int(d) for d in tensor_dims)
        self.grid_dims = tuple(int(g) for g in grid_dims)
        if len(self.tensor_dims) != len(self.grid_dims):
            raise ValueError("grid has %d dims, tensor has %d"
                             % (len(self.grid_dims), len(self.tensor_dims)))
        if min(self.grid_dims) < 1:
            raise ValueError("grid dims must be positive: %s" % (self.grid_dims,))
        self.N = len(self.grid_dims)
        self.P = int(np.prod(self.grid_dims))
        self.warning = warning
        # rank -> grid coordinates, row-major (last mode fastest)
        self._coord = np.array(list(itertools.product(*[range(g) for g in self.grid_dims])),
                               dtype=np.int64).reshape(self.P, self.N)
        self.weighted = row_weights is not None
        if self.weighted:
            row_weights = [np.asarray(w, dtype=np.float64) for w in row_weights]
            if [w.size for w in row_weights] != list(self.tensor_dims):
                raise ValueError("row_weights must hold one weight per row of every mode")
            self.chunk_offsets = [weighted_offsets(w, g) for w, g in zip(row_weights,
                                                                          self.grid_dims)]
        else:
            self.chunk_offsets = [balanced_offsets(I, g) for I, g in zip(self.tensor_dims,
                                                                            self.grid_dims)]
        self._lo = np.empty((self.N, self.P), dtype=np.int64)
        self._hi = np.empty((self.N, self.P), dtype=np.int64)
        for j in range(self.N):
            for c in range(self.grid_dims[j]):
                group = np.nonzero(self._coord[:, j] == c)[0]        # ascending rank ids
                base = int(self.chunk_offsets[j][c])
                end = int(self.chunk_offsets[j][c + 1])
                if self.weighted:
                    cut = weighted_offsets(row_weights[j][base:end], len(group))
                else:
                    cut = balanced_offsets(end - base, len(group))
                self._lo[j, group] = base + cut[:-1]
                self._hi[j, group] = base + cut[1:]
        # ranks in global row order per mode (ties by rank id); empty blocks excluded from
        # the owner lookup so block ends stay monotone
        self._order = [np.array(sorted(range(self.P), key=lambda p: (self._lo[j, p], p)),
                                dtype=np.int64) for j in range(self.N)]
        self._owner_ends = []
        self._owner_ids = []
        for j in range(self.N):
            live = [p for p in self._order[j] if self._hi[j, p] > self._lo[j, p]]
            self._owner_ids.append(np.array(live, dtype=np.int64))
            self._owner_ends.append(self._hi[j, live].astype(np.int64))

    def coords(self, p):
        return tuple(int(c) for c in self._coord[p])

    def block_range(self, j, p):
        return int(self._lo[j, p]), int(self._hi[j, p])

    def block_ranges(self, j):
        return self._lo[j].copy(), self._hi[j].copy()

    def row_order(self, j):
        return self._order[j].copy()

    def row_owner(self, j, rows):
        idx = np.searchsorted(self._owner_ends[j], np.asarray(rows), side="right")
        return self._owner_ids[j][idx]

    def slice_group(self, j, c):
        return np.nonzero(self._coord[:, j] == c)[0]


def _ordered_factorizations(P, N):
    if N == 1:
        yield (P,)
        return
    for d in range(1, P + 1):
        if P % d == 0:
            for tail in _ordered_factorizations(P // d, N - 1):
                yield (d,) + tail


def optimal_grid(tensor_dims, P, row_weights=None) -> ProcessorGrid:
    """Grid minimising sum_k I_k / P_k over ordered factorizations of P; grids with every
    P_k <= I_k win over infeasible ones; ties go to the lexicographically smallest tuple
    (ref grid.py:131-156)."""
    if P < 1:
        raise ValueError("P must be >= 1")
    dims = tuple(int(d) for d in tensor_dims)
    cands = [(sum(I / p for I, p in zip(dims, f)), f) for f in _ordered_factorizations(int(P), len(dims))]
    feasible = [c for c in cands if all(p <= I for p, I in zip(c[1], dims))]
    if feasible:
        return ProcessorGrid(dims, min(feasible)[1], warning=False, row_weights=row_weights)
    return ProcessorGrid(dims, min(cands)[1], warning=True, row_weights=row_weights)


def nnz_row_weights(dims, idx):
    """Nonzeros per row of every mode (numpy), for ProcessorGrid(row_weights=...).
    idx: (nnz, N) int64 numpy array or torch tensor, or a list of (idx, vals) chunks."""
    if isinstance(idx, (list, tuple)):
        parts = [nnz_row_weights(dims, ch[0]) for ch in idx]
        return [sum(p[j] for p in parts) for j in range(len(dims))]
    out = []
    for j, d in enumerate(dims):
        col = idx[:, j]
        if type(col).__module__.startswith("torch"):   # torch: count on its device
            import torch
            out.append(torch.bincount(col, minlength=int(d)).cpu().numpy())
        else:
            out.append(np.bincount(np.asarray(col), minlength=int(d)))
    return out


def as_gather_words_total_per_solve(J, R, N, P, sampler) -> int:
    """Words (8 B) all ranks receive in one accumulator-stationary solve's sampled-row
    all-gather: (P-1) J (N-1) (R+2) for STS, (P-1) J (N-1) R for CP-ARLS-LEV
    (ref grid.py:370-376)."""
    w = R + 2 if sampler == "sts" else R
    return (P - 1) * J * (N - 1) * w
