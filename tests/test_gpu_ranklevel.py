"""Rank-level (P > 1) STS kernels through the C ABI: the packed rank tree, the run-grouped
rank walk against the per-sample rank walk, the local flat search of the first constant
mode against the oracle's leaf search, and the exchange pack/unpack kernels
(ref samplers.py:239-275, :423-451, :313-345; schedules.py:239-247)."""

import numpy as np
import pytest

from conftest import cuda_ok

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]


@pytest.fixture(scope="module")
def env():
    import torch
    from paper_2210_05105_b200.device import require_cuda
    from paper_2210_05105_b200.ops import ops_for
    dev = require_cuda()
    return torch, dev, ops_for(dev)


def _spd(rng, R, n):
    A = rng.standard_normal((n, R))
    return A.T @ A


def _full_rank_tree(blocks, order, width):
    """Level-major full R x R node Grams (the per-sample kernel's layout)."""
    P, R, _ = blocks.shape
    lv = np.zeros((width, R, R))
    lv[:P] = blocks[order]
    levels = [lv]
    while levels[0].shape[0] > 1:
        levels.insert(0, levels[0].reshape(-1, 2, R, R).sum(axis=1))
    return np.concatenate([x.reshape(-1) for x in levels])


@pytest.mark.parametrize("P,R,groups", [(2, 5, 1), (3, 8, 7), (4, 50, 300), (8, 25, 2000),
                                        (5, 70, 50), (8, 50, 1), (37, 100, 1)])
def test_grouped_rank_walk_matches_per_sample_walk(env, P, R, groups):
    t, dev, ops = env
    rng = np.random.default_rng(P * 100 + R)
    J = 4096
    depth = int(np.ceil(np.log2(P)))
    width = 1 << depth
    blocks = np.stack([_spd(rng, R, 3 * R) for _ in range(P)])
    order = rng.permutation(P).astype(np.int64)
    leaf_rank = np.full(width, -1, dtype=np.int32)
    leaf_rank[:P] = order
    M = _spd(rng, R, 2 * R)
    # samples of one group share their Hadamard row (equal keys <=> equal rows)
    gid = rng.integers(0, groups, J)
    Hg = rng.uniform(0.2, 1.5, (groups, R))
    H = Hg[gid] if groups > 1 else np.ones((J, R))
    d = lambda a: t.as_tensor(np.ascontiguousarray(a), device=dev)  # noqa: E731
    bg, Md, Hd = d(blocks), d(M), d(H)
    hkey = d(gid.astype(np.int64))
    key = (0x1234567, 0x89abcdef)
    # per-sample kernel on full node Grams
    own_a = t.zeros(J, dtype=t.int32, device=dev)
    r_a = t.zeros(J, dtype=t.float64, device=dev)
    p_a = t.ones(J, dtype=t.float64, device=dev)
    ops.sts_rank_walk(d(_full_rank_tree(blocks, order, width)), depth, P, d(leaf_rank), Md, Hd, J,
                      key, None, own_a, r_a, p_a)
    # grouped kernel on the packed tree
    tree = ops.sts_rank_tree(bg, d(order))
    own_b = t.full((J,), -7, dtype=t.int32, device=dev)
    r_b = t.zeros(J, dtype=t.float64, device=dev)
    p_b = t.ones(J, dtype=t.float64, device=dev)
    kb = max(1, int(groups - 1).bit_length() + 1)
    # one group: H_in = None takes the node-masses-once kernel (rcp_sts_rank_walk_ones), an
    # explicit all-ones H_in the run-grouped walk with its single-group shortcut (no sort)
    variants = [(Hd, hkey)] if groups > 1 else [(None, None), (Hd, None)]
    for Hv, kv in variants:
        own_b.fill_(-7)
        ops.sts_rank_walk_grouped(tree, P, d(leaf_rank), Md, Hv, J, key, None, own_b, r_b, p_b,
                                  hkey=kv, key_bits=kb)
        ops.status.check("rank walks")
        a, b = own_a.cpu().numpy(), own_b.cpu().numpy()
        assert np.array_equal(a, b)
        assert set(np.unique(b)) <= set(order.tolist())
        assert np.allclose(p_a.cpu().numpy(), p_b.cpu().numpy(), rtol=1e-11, atol=0)
        assert np.allclose(r_a.cpu().numpy(), r_b.cpu().numpy(), rtol=0, atol=1e-9)


def test_rank_tree_levels_are_pairwise_sums(env):
    t, dev, ops = env
    rng = np.random.default_rng(3)
    P, R = 5, 6
    blocks = np.stack([_spd(rng, R, 10) for _ in range(P)])
    order = np.array([3, 0, 4, 1, 2], dtype=np.int64)
    tree = ops.sts_rank_tree(t.as_tensor(blocks, device=dev), t.as_tensor(order, device=dev))
    Rs = (R * (R + 1) // 2 + 1) & ~1
    tr = tree.cpu().numpy().reshape(-1, Rs)
    iu = np.triu_indices(R)
    width = 8
    leaves = np.zeros((width, R, R))
    leaves[:P] = blocks[order]
    lvl = leaves
    base = width - 1
    while True:
        for v in range(lvl.shape[0]):
            assert np.array_equal(tr[base + v, :len(iu[0])], lvl[v][iu])
            assert np.all(tr[base + v, len(iu[0]):] == 0.0)
        if lvl.shape[0] == 1:
            break
        lvl = lvl.reshape(-1, 2, R, R).sum(axis=1)
        base = lvl.shape[0] - 1


def test_flat_local_search_matches_oracle_leaf_search(env):
    """Samples routed to a rank invert that rank's row-mass CDF at their residual."""
    t, dev, ops = env
    rng = np.random.default_rng(11)
    n, R, J = 777, 9, 3000
    U = rng.standard_normal((n, R))
    M = _spd(rng, R, 3 * R)
    r = rng.random(J)
    sel = rng.integers(0, 3, J).astype(np.int32)
    d = lambda a: t.as_tensor(np.ascontiguousarray(a), device=dev)  # noqa: E731
    Ud, Md = d(U), d(M)
    dist = t.zeros(n, dtype=t.float64, device=dev)
    cdf = t.zeros(n, dtype=t.float64, device=dev)
    mass = t.zeros(1, dtype=t.float64, device=dev)
    ops.arls_build(Ud, Md, dist, cdf, mass)
    X = t.full((J,), -5, dtype=t.int64, device=dev)
    pmp = t.full((J,), 0.5, dtype=t.float64, device=dev)
    resid = t.full((J,), -1.0, dtype=t.float64, device=dev)
    ops.sts_flat_local(cdf, dist, 100, mass, d(r), d(sel), 1, J, X, pmp, resid)
    ops.status.check("flat local")
    m = np.maximum(np.einsum("qa,ab,qb->q", U, M, U), 0.0)
    c = np.cumsum(m)
    mine = sel == 1
    exp = np.minimum(np.searchsorted(c, r * c[-1], side="right"), n - 1)
    got = X.cpu().numpy()
    # a uniform within rounding of a CDF boundary may fall on either side
    near = np.abs(r * c[-1] - c[np.minimum(exp, n - 1)]) < 1e-9 * c[-1]
    near |= np.abs(r * c[-1] - np.where(exp > 0, c[exp - 1], 0.0)) < 1e-9 * c[-1]
    ok = (got[mine] == 100 + exp[mine]) | near[mine]
    assert ok.all()
    assert np.all(got[~mine] == -5)
    pg = pmp.cpu().numpy()
    assert np.allclose(pg[mine & ~near], 0.5 * m[exp[mine & ~near]] / c[-1], rtol=1e-11)
    assert np.all(pg[~mine] == 0.5)
    rg = resid.cpu().numpy()
    assert np.all((rg[mine] >= 0.0) & (rg[mine] < 1.0)) and np.all(rg[~mine] == -1.0)
    below = np.where(exp > 0, c[exp - 1], 0.0)
    want = (r * c[-1] - below) / np.maximum(m[exp], 1e-300)
    sel_ok = mine & ~near & (m[exp] > 1e-6 * c[-1])
    assert np.allclose(rg[sel_ok], want[sel_ok], atol=1e-6)


def test_flat_local_search_zero_mass_rank_raises(env):
    t, dev, ops = env
    from paper_2210_05105_b200 import DegenerateWalkError
    J = 8
    z = t.zeros(4, dtype=t.float64, device=dev)
    mass = t.zeros(1, dtype=t.float64, device=dev)
    X = t.zeros(J, dtype=t.int64, device=dev)
    pmp = t.ones(J, dtype=t.float64, device=dev)
    ops.sts_flat_local(z, z, 0, mass, t.full((J,), 0.3, dtype=t.float64, device=dev),
                       t.zeros(J, dtype=t.int32, device=dev), 0, J, X, pmp, None)
    with pytest.raises(DegenerateWalkError):
        ops.status.check("flat local on an empty rank")
    ops.status.reset()


@pytest.mark.parametrize("R", [4, 50, 75])
def test_exchange_pack_unpack(env, R):
    t, dev, ops = env
    rng = np.random.default_rng(R)
    J, n, lo, rank = 1000, 300, 5000, 2
    U = t.as_tensor(rng.standard_normal((n, R)), device=dev)
    owner = t.as_tensor(rng.integers(0, 4, J).astype(np.int32), device=dev)
    X = t.as_tensor(rng.integers(lo, lo + n, J), device=dev)
    X[::17] = -1                                   # degenerate samples contribute nothing
    pmp = t.as_tensor(rng.random(J), device=dev)
    resid = t.as_tensor(rng.random(J), device=dev)
    buf = t.full((J, R + 3), 9.0, dtype=t.float64, device=dev)
    ops.exchange_pack(X, pmp, resid, U, lo, owner, rank, buf)
    mine = (owner == rank) & (X >= lo)
    exp = t.zeros_like(buf)
    exp[mine, 0] = X[mine].to(t.float64)
    exp[mine, 1] = pmp[mine]
    exp[mine, 2] = resid[mine]
    exp[mine, 3:] = U[(X[mine] - lo)]
    assert t.equal(buf, exp)
    H = t.as_tensor(rng.random((J, R)), device=dev)
    H0 = H.clone()
    X2 = t.zeros(J, dtype=t.int64, device=dev)
    p2 = t.zeros(J, dtype=t.float64, device=dev)
    r2 = t.zeros(J, dtype=t.float64, device=dev)
    ops.exchange_unpack(buf, False, X2, p2, r2, H)
    assert t.equal(X2, exp[:, 0].to(t.int64)) and t.equal(p2, exp[:, 1]) and t.equal(r2, exp[:, 2])
    assert t.equal(H, H0 * exp[:, 3:])
    ops.exchange_unpack(buf, True, X2, p2, r2, H)
    assert t.equal(H, exp[:, 3:])
