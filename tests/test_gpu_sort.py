"""Stable (key, row) orderings (csrc/sort.cu) against numpy's lexsort / stable argsort, the
orderings the reference's store and CSR transpose rely on (ref matricization.py:56-77,
mttkrp.py:131-155): duplicates keep their input order, keys beyond 2^32, empty input."""

import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]


def _ops():
    import torch
    from paper_2210_05105_b200.ops import ops_for
    dev = torch.device("cuda", 0)
    return torch, dev, ops_for(dev)


@pytest.mark.parametrize("n,key_max,row_max", [
    (0, 10, 10), (1, 0, 0), (1000, 7, 3), (50_000, (1 << 45) + 12345, 28817),
    (300_001, 1_000_003, (1 << 31) - 2), (4097, (1 << 62) - 1, 1)])
def test_order_by_key_row_matches_lexsort(n, key_max, row_max):
    torch, dev, ops = _ops()
    rng = np.random.default_rng(n + 7)
    # few distinct keys and rows among many entries: ties everywhere
    kpool = rng.integers(0, key_max + 1, size=max(1, n // 50), dtype=np.int64)
    key = kpool[rng.integers(0, kpool.size, size=n)] if n else np.zeros(0, dtype=np.int64)
    row = rng.integers(0, min(row_max, 40) + 1, size=n, dtype=np.int64)
    if n:
        key[0], row[0] = key_max, row_max          # the extremes are present
    got = ops.order_by_key_row(torch.as_tensor(key, device=dev), torch.as_tensor(row, device=dev),
                               key_max, row_max).cpu().numpy()
    want = np.lexsort((row, key))                   # stable: equal (key, row) keep input order
    assert got.dtype == np.int64
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("n,row_max", [(0, 5), (17, 0), (200_000, 12091)])
def test_order_by_row_alone_matches_stable_argsort(n, row_max):
    torch, dev, ops = _ops()
    rng = np.random.default_rng(n + 3)
    row = rng.integers(0, row_max + 1, size=n, dtype=np.int64)
    got = ops.order_by_key_row(None, torch.as_tensor(row, device=dev), 0, row_max).cpu().numpy()
    np.testing.assert_array_equal(got, np.argsort(row, kind="stable"))


def test_store_build_unchanged_by_native_ordering():
    """build_store on shuffled COO input with repeated (key, row) cells absent: the store
    equals the numpy lexsort layout entry for entry."""
    torch, dev, ops = _ops()
    from paper_2210_05105_b200.store import build_store
    rng = np.random.default_rng(11)
    dims = (37, 19, 23)
    cells = rng.choice(np.prod(dims), size=5000, replace=False)
    idx = np.stack(np.unravel_index(cells, dims), axis=1).astype(np.int64)
    vals = rng.standard_normal(idx.shape[0])
    for mode in range(3):
        st = build_store(dims, torch.as_tensor(idx, device=dev), torch.as_tensor(vals, device=dev), mode)
        strides = [int(x) for x in st.strides]
        key = sum(idx[:, m] * strides[m] for m in range(3) if m != mode)
        order = np.lexsort((idx[:, mode], key))
        np.testing.assert_array_equal(st.rows.cpu().numpy(), idx[order, mode].astype(np.int32))
        np.testing.assert_array_equal(st.vals.cpu().numpy(), vals[order])
        uk, cnt = np.unique(key[order], return_counts=True)
        np.testing.assert_array_equal(st.keys.cpu().numpy(), uk)
        np.testing.assert_array_equal(st.colptr.cpu().numpy(), np.concatenate([[0], np.cumsum(cnt)]))
