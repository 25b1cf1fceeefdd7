"""Host-side tensor input and result output (rows F3/F4 of SURVEY.md 8(f); not on the
sampled hot path): FROSTT `.tns` parsing with the reference's validation and
duplicate/log semantics (ref load_frostt tensor.py:86-149, sum_duplicates :72-83), the
binary matrix files (ref write_matrix/read_matrix tensor.py:213-225) and the per-trial
output directory of `randcp decompose --out` (ref cli.py:78-108).
"""

from __future__ import annotations

import os

import numpy as np

from .coo import BoundsError, SparseTensorCOO


class ParseError(ValueError):
    """Malformed tensor file (ref tensor.py:14-15)."""


def sum_duplicates(idx, vals):
    """Collapse repeated coordinates, summing their values (ref tensor.py:72-83): entries
    come back in lexicographic coordinate order, each duplicate run summed in file order."""
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    vals = np.ascontiguousarray(vals, dtype=np.float64)
    if idx.shape[0] == 0:
        return idx, vals
    order = np.lexsort(idx.T[::-1])
    s_idx, s_vals = idx[order], vals[order]
    first = np.ones(s_idx.shape[0], dtype=bool)
    first[1:] = np.any(s_idx[1:] != s_idx[:-1], axis=1)
    starts = np.flatnonzero(first)
    return np.ascontiguousarray(s_idx[starts]), np.add.reduceat(s_vals, starts)


def _data_lines(path):
    with open(path, "r") as fh:
        for no, line in enumerate(fh, 1):
            text = line.strip()
            if text and not text.startswith("#"):
                yield no, text


def load_frostt(path, *, log_transform=False, dedup=True, dims=None) -> SparseTensorCOO:
    """FROSTT `.tns` reader: N 1-based integer indices and a value per non-comment line
    (ref tensor.py:86-149, same errors: ParseError for malformed lines / non-integer
    indices / too few columns, BoundsError for indices < 1 or beyond `dims`)."""
    lines = list(_data_lines(path))
    if not lines:
        raise ParseError("%s: no tensor entries found" % path)
    width = len(lines[0][1].split())
    rows = []
    for no, text in lines:
        parts = text.split()
        if len(parts) != width:
            raise ParseError("%s: line %d: expected %d columns, got %d"
                             % (path, no, width, len(parts)))
        try:
            rows.append([float(x) for x in parts])
        except ValueError:
            raise ParseError("%s: line %d: unparsable number" % (path, no)) from None
    table = np.asarray(rows, dtype=np.float64)
    if table.shape[1] < 4:
        raise ParseError("%s: need at least 3 index columns and a value, got %d columns"
                         % (path, table.shape[1]))
    n_modes = table.shape[1] - 1
    idx_f = table[:, :n_modes]
    idx = idx_f.astype(np.int64)
    line_no = np.array([no for no, _ in lines])
    bad = np.flatnonzero((idx != idx_f).any(axis=1))
    if bad.size:
        raise ParseError("%s: line %d: non-integer index" % (path, line_no[bad[0]]))
    bad = np.flatnonzero((idx < 1).any(axis=1))
    if bad.size:
        raise BoundsError("%s: line %d: indices are 1-based and must be >= 1"
                          % (path, line_no[bad[0]]))
    idx -= 1
    vals = np.ascontiguousarray(table[:, n_modes])
    if dims is not None:
        dims = tuple(int(d) for d in dims)
        if len(dims) != n_modes:
            raise ParseError("%s: file has %d modes but %d dims declared"
                             % (path, n_modes, len(dims)))
        bad = np.flatnonzero((idx >= np.asarray(dims)).any(axis=1))
        if bad.size:
            raise BoundsError("%s: line %d: index exceeds declared dims %s"
                              % (path, line_no[bad[0]], dims))
    else:
        dims = tuple(int(m) + 1 for m in idx.max(axis=0))
    if dedup:
        idx, vals = sum_duplicates(idx, vals)
    if log_transform:
        vals = np.log1p(vals)
    return SparseTensorCOO(dims, idx, vals)


def write_matrix(path, M):
    """Little-endian int64 (rows, cols) header, then row-major float64 (ref tensor.py:213-220);
    a vector is written as one column."""
    M = np.ascontiguousarray(M, dtype=np.float64)
    if M.ndim == 1:
        M = M[:, None]
    with open(path, "wb") as fh:
        np.asarray(M.shape, dtype="<i8").tofile(fh)
        M.astype("<f8").tofile(fh)


def read_matrix(path):
    with open(path, "rb") as fh:
        shape = np.fromfile(fh, dtype="<i8", count=2)
        if shape.size != 2:
            raise ParseError("%s: truncated matrix header" % path)
        data = np.fromfile(fh, dtype="<f8")
    if data.size != int(shape[0]) * int(shape[1]):
        raise ParseError("%s: expected %d values, found %d"
                         % (path, int(shape[0]) * int(shape[1]), data.size))
    return data.reshape(int(shape[0]), int(shape[1]))


def write_results(results, out_dir):
    """One directory per trial (ref cli.py:93-104): factor_mode<j>.bin (rows in the input
    tensor's index order), sigma.bin, summary.txt."""
    os.makedirs(out_dir, exist_ok=True)
    for t, res in enumerate(results):
        tdir = os.path.join(out_dir, "trial%d" % t)
        os.makedirs(tdir, exist_ok=True)
        for j, U in enumerate(res.factors):
            write_matrix(os.path.join(tdir, "factor_mode%d.bin" % j), U)
        write_matrix(os.path.join(tdir, "sigma.bin"), res.sigma)
        with open(os.path.join(tdir, "summary.txt"), "w") as fh:
            fh.write(res.summary() + "\n")
