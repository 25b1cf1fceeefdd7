"""Device ingest (row F2, ingest.cu): counter-based Zipf draws reproduce the splitmix
stream of synth.zipf_tensor exactly, duplicates are summed (ref sum_duplicates
tensor.py:72-83), the per-mode permutation is applied (ref permute_modes tensor.py:182-210),
and stores built bucket by bucket from the chunks equal the single-pass build."""

import math

import numpy as np
import pytest

from conftest import cuda_ok
from paper_2210_05105_b200 import synth

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]


def torch_reference(dims, nbatch, bits, s, seed, values, sigma):
    """All distinct cells of `nbatch` chunks of 2^bits draws, with torch ops only (the
    inner loop of synth.zipf_tensor), values summed per cell in float64."""
    import torch
    dev = torch.device("cuda", 0)
    N = len(dims)
    strides = [1] * N
    for m in range(N - 2, -1, -1):
        strides[m] = strides[m + 1] * dims[m + 1]
    cdfs = [torch.as_tensor(synth.zipf_cdf(d, s), device=dev) for d in dims]
    batch = 1 << bits
    keys, vals = [], []
    for rnd in range(nbatch):
        lin = torch.zeros(batch, dtype=torch.int64, device=dev)
        for m in range(N):
            u = synth._splitmix_uniform(torch, seed * 1000 + rnd, batch, m + 1, dev)
            lin += torch.searchsorted(cdfs[m], u, right=True).clamp_(max=dims[m] - 1) * strides[m]
        u1 = synth._splitmix_uniform(torch, seed * 1000 + rnd, batch, 101, dev)
        if values == "lognormal":
            u2 = synth._splitmix_uniform(torch, seed * 1000 + rnd, batch, 102, dev)
            z = torch.sqrt(-2.0 * torch.log1p(-u1)) * torch.cos(2.0 * math.pi * u2)
            v = torch.exp(sigma * z)
        else:
            v = synth._poisson3(torch, u1)
        keys.append(lin)
        vals.append(v)
    keys = torch.cat(keys)
    vals = torch.cat(vals)
    uk, inv = torch.unique(keys, return_inverse=True)
    tot = torch.zeros(uk.numel(), dtype=torch.float64, device=dev).index_add_(0, inv, vals)
    if values == "log1p_poisson":
        tot = torch.log1p(tot)
    idx = torch.empty((uk.numel(), N), dtype=torch.int64, device=dev)
    rem = uk.clone()
    for m in range(N):
        idx[:, m] = rem // strides[m]
        rem = rem % strides[m]
    return idx.cpu().numpy(), tot.cpu().numpy()


def canon(idx, vals):
    o = np.lexsort(idx.T[::-1])
    return idx[o], vals[o]


@pytest.mark.parametrize("values,parts", [("lognormal", 1), ("lognormal", 4),
                                          ("log1p_poisson", 8)])
def test_zipf_chunks_match_torch_stream(values, parts):
    dims = (300, 50, 700)
    bits = 14
    ridx, rv = torch_reference(dims, 3, bits, 1.1, 7, values, 1.5)
    chunks = synth.zipf_chunks(dims, 3 << bits, 1.1, seed=7, values=values, sigma=1.5, parts=parts,
                               chunk_bits=bits)
    gidx = np.concatenate([c[0].cpu().numpy() for c in chunks]).astype(np.int64)
    gv = np.concatenate([c[1].cpu().numpy() for c in chunks])
    assert gidx.shape == ridx.shape
    a, av = canon(gidx, gv)
    b, bv = canon(ridx, rv)
    assert np.array_equal(a, b)
    assert np.allclose(av, bv, rtol=1e-12, atol=0)


def test_zipf_chunks_permutation_and_capacity_retry():
    """Permutations map every coordinate; a partition that overflows its first buffer
    guess is redrawn with the exact size (all draws of a 2-cell tensor hit one part)."""
    import torch
    dims = (40, 30, 20)
    perms = [np.random.default_rng(j).permutation(d) for j, d in enumerate(dims)]
    plain = synth.zipf_chunks(dims, 1 << 13, 1.3, seed=3, parts=2, chunk_bits=12)
    perm = synth.zipf_chunks(dims, 1 << 13, 1.3, seed=3, parts=2, chunk_bits=12, perms=perms)
    for (a, va), (b, vb) in zip(plain, perm):
        a = a.cpu().numpy()
        b = b.cpu().numpy()
        for m in range(3):
            assert np.array_equal(perms[m][a[:, m]], b[:, m])
        assert torch.equal(va, vb)
    tiny = synth.zipf_chunks((2, 1, 1), 5000, 1.0, seed=1, parts=4, chunk_bits=10)
    assert sum(c[0].shape[0] for c in tiny) == 2


@pytest.mark.parametrize("buckets", [1, 3, 16])
def test_store_chunks_equal_single_pass(buckets):
    import torch
    from paper_2210_05105_b200.store import build_store, build_store_chunks
    dims = (90, 40, 60)
    chunks = synth.zipf_chunks(dims, 1 << 15, 1.05, seed=2, parts=4, chunk_bits=13)
    idx = torch.cat([c[0] for c in chunks]).long()
    vals = torch.cat([c[1] for c in chunks])
    for j, (lo, hi) in enumerate([(0, 90), (10, 30), (0, 60)]):
        sel = (idx[:, j] >= lo) & (idx[:, j] < hi)
        a = build_store(dims, idx[sel], vals[sel], j, lo, hi)
        b = build_store_chunks(dims, chunks, j, lo, hi, buckets=buckets)
        for name in ("keys", "colptr", "rows", "vals"):
            assert torch.equal(getattr(a, name), getattr(b, name)), (j, name)
        assert a.max_col == b.max_col


def test_engine_on_chunks_matches_coo_engine():
    """A cluster built from ingest chunks runs the same rounds as one built from the
    equivalent COO (same samples, same factors)."""
    import torch
    from paper_2210_05105_b200.engine import make_local_cluster
    dims = (60, 45, 50)
    chunks = synth.zipf_chunks(dims, 1 << 14, 1.1, seed=4, parts=2, chunk_bits=12)
    idx = torch.cat([c[0] for c in chunks]).long()
    vals = torch.cat([c[1] for c in chunks])
    a = make_local_cluster(dims, idx, vals, 6, 300, "sts", 1)
    b = make_local_cluster(dims, chunks, None, 6, 300, "sts", 1)
    for rnd in (1, 2):
        a.round(rnd)
        b.round(rnd)
    assert torch.equal(a.ranks[0].X, b.ranks[0].X)
    for j in range(3):
        assert torch.allclose(a.ranks[0].U[j], b.ranks[0].U[j], rtol=1e-12, atol=1e-14)


def test_zipf_chunks_keep_only_rank_blocks():
    """Per-rank ingest: with keep=<a rank's block ranges>, every partition keeps exactly the
    cells of the full ingest that have at least one mode index in the rank's blocks
    (ref matricization.py:187-198); the ranks' stores built from their kept cells equal the
    stores built from the whole tensor."""
    from paper_2210_05105_b200.grid import optimal_grid
    from paper_2210_05105_b200.store import build_store_chunks
    dims = (300, 200, 250)
    perms = [np.random.default_rng(j).permutation(d) for j, d in enumerate(dims)]
    full = synth.zipf_chunks(dims, 1 << 15, 1.2, seed=5, parts=4, chunk_bits=13, perms=perms)
    w = synth.zipf_expected_row_weights(dims, 1.2, perms)
    assert all(abs(x.sum() - 1.0) < 1e-12 for x in w)
    g = optimal_grid(dims, 4, row_weights=w)
    fidx = np.concatenate([c[0].cpu().numpy() for c in full]).astype(np.int64)
    for p in range(4):
        keep = [g.block_range(j, p) for j in range(3)]
        mine = synth.zipf_chunks(dims, 1 << 15, 1.2, seed=5, parts=4, chunk_bits=13, perms=perms,
                                 keep=keep)
        midx = np.concatenate([c[0].cpu().numpy() for c in mine]).astype(np.int64)
        sel = np.zeros(len(fidx), dtype=bool)
        for j, (lo, hi) in enumerate(keep):
            sel |= (fidx[:, j] >= lo) & (fidx[:, j] < hi)
        assert np.array_equal(canon(midx, np.zeros(len(midx)))[0],
                              canon(fidx[sel], np.zeros(int(sel.sum())))[0])
        for j, (lo, hi) in enumerate(keep):
            a = build_store_chunks(dims, mine, j, lo, hi)
            b = build_store_chunks(dims, full, j, lo, hi)
            assert a.nnz == b.nnz
            assert torch_equal(a.keys, b.keys) and torch_equal(a.rows, b.rows)
            assert torch_equal(a.vals, b.vals)


def torch_equal(x, y):
    import torch
    return bool(torch.equal(x, y))
