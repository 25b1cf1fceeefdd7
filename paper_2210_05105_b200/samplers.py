"""Leverage-score samplers -- drop-ins for the reference's samplers.py, run on the GPU.

Same names, signatures, return types and exceptions as the reference (ref
samplers.py:34-478).  Inputs/outputs are numpy arrays; the work runs in the sm_100a
kernels of librandcp_b200.so:

* CP-ARLS-LEV: per-row leverage + ordered mass + normalised cdf on the device
  (`rcp_arls_build`), inverse-CDF draws on the LOCAL_DRAW Philox streams
  (`rcp_arls_draw`), SHUFFLE permutation and Hadamard fold (`rcp_batch_fold`).
  The P-sized multinomial split stays on the host with numpy, as in the reference.
* STS-CP: per-block binary tree of packed node Grams (`rcp_sts_build`), the rank-level
  shared levels (`rcp_sts_rank_walk`) and the per-owner tree walk + leaf inverse-CDF
  (`rcp_sts_walk`).  The reference's flat leaf-block scan is replaced by a full tree
  walk; both are the inverse CDF of the same uniform over rows in global order, so draws
  agree except where a uniform lies within rounding of a CDF boundary (the reference
  itself relies on this invariance across leaf sizes and rank counts,
  ref tests/test_samplers.py:223-233).
"""

from __future__ import annotations

import math

import numpy as np

from . import rng
from .device import DegenerateWalkError, require_cuda, to_dev, to_host, torch
from .engine import default_leaf
from .linalg import FactorBlocks
from .ops import ops_for

ORACLE_GUARD = 10 ** 6          # ref samplers.py:30

__all__ = ["DegenerateWalkError", "SampleBatch", "sample_weights", "ArlsLevState",
           "arls_lev_build", "consistent_multinomial", "arls_lev_sample", "LeverageTree",
           "sts_build", "sts_sample", "local_sts_leaf_search", "krp_leverage_scores",
           "exact_krp_leverage_oracle"]


class SampleBatch:
    """J sampled design rows for one mode-k solve (ref samplers.py:65-86)."""

    def __init__(self, X, H, per_mode_prob, prob, residual=None, owner=None):
        self.X = X
        self.H = H
        self.per_mode_prob = per_mode_prob
        self.prob = prob
        self.residual = residual
        self.owner = owner
        self.weights = None

    @property
    def J(self):
        return self.X.shape[0]


def _empty_batch(N, R):
    return SampleBatch(np.full((0, N), -1, dtype=np.int64), np.ones((0, R)), np.ones((0, N)),
                       np.ones(0), residual=np.ones(0))


def sample_weights(batch: SampleBatch, J=None):
    """w_s = 1/sqrt(J p_s) (ref samplers.py:89-96)."""
    if J is None:
        J = batch.J
    if batch.J == 0:
        batch.weights = np.empty(0)
        return batch.weights
    dev = require_cuda()
    t = torch()
    ops = ops_for(dev)
    p = to_dev(np.asarray(batch.prob, dtype=np.float64), dev, t.float64)
    if int(J) == batch.J:
        w = t.empty_like(p)
        ops.weights(p.reshape(1, -1), None, w)
        ops.status.check("in sample_weights")
    else:
        if bool((p <= 0).any()):
            raise ValueError("sample with zero probability cannot have been drawn")
        w = 1.0 / t.sqrt(float(J) * p)
    batch.weights = to_host(w)
    return batch.weights


def _prod_rows(pmp):
    p = pmp[0].clone()
    for m in range(1, pmp.shape[0]):
        p *= pmp[m]
    return p


# ----------------------------------------------------------------- CP-ARLS-LEV
class ArlsLevState:
    """Per-mode leverage distributions and masses (ref samplers.py:104-119); `dev` holds
    the device (U, dist, cdf) of each block."""

    def __init__(self, mode, dists, C, lows, his, gram_matrix, gram_pinv, dev=None):
        self.mode = mode
        self.dists = dists
        self.C = C
        self.lows = lows
        self.his = his
        self.gram = gram_matrix
        self.gram_pinv = gram_pinv
        self.dev = dev


def arls_lev_build(blocks: FactorBlocks, ledger=None, round_id=0) -> ArlsLevState:
    """(ref samplers.py:122-135)"""
    dev = require_cuda()
    t = torch()
    ops = ops_for(dev)
    R = blocks.R
    Us = [to_dev(B, dev, t.float64) for B in blocks.blocks]
    G = t.zeros((R, R), dtype=t.float64, device=dev)
    for U in Us:
        if U.shape[0]:
            G += ops.gram(U)
    Gp = ops.pinv(G)
    ops.status.check("in arls_lev_build")
    dists, C, devs = [], np.zeros(blocks.n_blocks), []
    for p, U in enumerate(Us):
        n = U.shape[0]
        dist = t.zeros(n, dtype=t.float64, device=dev)
        cdf = t.zeros(n, dtype=t.float64, device=dev)
        mass = t.zeros(1, dtype=t.float64, device=dev)
        if n:
            ops.arls_build(U, Gp, dist, cdf, mass)
        C[p] = float(mass.item())
        dists.append(to_host(dist))
        devs.append((U, dist, cdf))
    return ArlsLevState(blocks.mode, dists, C, blocks.lows.copy(), blocks.his.copy(),
                        to_host(G), to_host(Gp), dev=devs)


def consistent_multinomial(masses, J, seed, round_id, k, mode):
    """Rank sample counts from the shared MULTINOMIAL stream (ref samplers.py:138-145)."""
    masses = np.asarray(masses, dtype=np.float64)
    total = masses.sum()
    if total <= 0.0:
        raise ValueError("all rank masses are zero; nothing to sample from")
    return rng.stream(seed, rng.MULTINOMIAL, round_id, k, mode).multinomial(int(J), masses / total)


def arls_lev_sample(states, k, J, factors_full, seed, round_id=0, ledger=None) -> SampleBatch:
    """(ref samplers.py:148-191)"""
    N = len(states)
    R = next(f.shape[1] for f in factors_full if f is not None)
    if J == 0:
        return _empty_batch(N, R)
    dev = require_cuda()
    t = torch()
    ops = ops_for(dev)
    X = t.full((N, J), -1, dtype=t.int64, device=dev)
    pmp = t.ones((N, J), dtype=t.float64, device=dev)
    H = t.ones((J, R), dtype=t.float64, device=dev)
    rows = t.empty(J, dtype=t.int64, device=dev)
    probs = t.empty(J, dtype=t.float64, device=dev)
    first = True
    for i in range(N):
        if i == k:
            continue
        st = states[i]
        W = float(st.C.sum())
        if W <= 0.0:
            raise ValueError("mode %d has zero total leverage mass" % i)
        split = consistent_multinomial(st.C, J, seed, round_id, k, i)
        off = 0
        for p in range(len(st.dists)):
            q = int(split[p])
            if q == 0:
                continue
            U, dist, cdf = st.dev[p]
            key = rng.stream_key(seed, rng.LOCAL_DRAW, round_id, k, i, p)
            ops.arls_draw(cdf, dist, int(st.lows[p]), float(st.C[p] / W), None, key, q, off,
                          rows, probs)
            off += q
        perm = to_dev(rng.permutation(rng.stream_key(seed, rng.SHUFFLE, round_id, k, i), J), dev,
                      t.int64)
        Ui = to_dev(factors_full[i], dev, t.float64)
        ops.batch_fold(perm, rows, probs, Ui, 0, None, first, X[i], pmp[i], H)
        first = False
    ops.status.check("in arls_lev_sample")
    return SampleBatch(to_host(X.T.contiguous()), to_host(H), to_host(pmp.T.contiguous()),
                       to_host(_prod_rows(pmp)), owner=None)


# ----------------------------------------------------------------------- STS-CP
class LeverageTree:
    """Leverage tree of one factor (ref samplers.py:194-221).

    `node_grams[lev]` is the rank-level padded tree (host, (2^lev, R, R)), exactly the
    reference's structure; below it every rank block carries a device binary tree of
    packed node Grams over leaves of `leaf_sizes[p]` rows (`row_trees[p]`)."""

    def __init__(self, mode, node_grams, leaf_rank, block_lo, block_hi, leaf_offsets,
                 leaf_grams, leaf_block_size, dev=None):
        self.mode = mode
        self.node_grams = node_grams
        self.leaf_rank = leaf_rank
        self.block_lo = block_lo
        self.block_hi = block_hi
        self.leaf_offsets = leaf_offsets
        self.leaf_grams = leaf_grams
        self.leaf_block_size = leaf_block_size
        self.dev = dev

    @property
    def depth(self):
        return len(self.node_grams) - 1

    @property
    def root_gram(self):
        return self.node_grams[0][0]


def sts_build(blocks: FactorBlocks, grid=None, ledger=None, round_id=0,
              leaf_block_size=None) -> LeverageTree:
    """(ref samplers.py:224-288)"""
    dev = require_cuda()
    t = torch()
    ops = ops_for(dev)
    R = blocks.R
    P = blocks.n_blocks
    if grid is not None:
        order = np.asarray(grid.row_order(blocks.mode), dtype=np.int64)
    else:
        order = np.lexsort((np.arange(P), blocks.lows))
    depth = max(int(math.ceil(math.log2(P))), 0) if P > 1 else 0
    width = 1 << depth
    Us, trees, leaves, offsets = [], [], [], []
    rank_g = t.zeros((P, R, R), dtype=t.float64, device=dev)
    for p, B in enumerate(blocks.blocks):
        U = to_dev(B, dev, t.float64)
        n = U.shape[0]
        L = int(leaf_block_size) if leaf_block_size else default_leaf(max(n, 1), R)
        L = max(1, min(64, L))
        Us.append(U)
        leaves.append(L)
        if n:
            trees.append(ops.sts_build(U, L))
            rank_g[p] = ops.gram(U)
            nl = int(math.ceil(n / L))
            offsets.append(np.minimum(np.arange(nl + 1, dtype=np.int64) * L, n))
        else:
            trees.append(None)
            offsets.append(np.zeros(1, dtype=np.int64))
    leaf_rank = np.full(width, -1, dtype=np.int64)
    leaf_rank[:P] = order
    lv = t.zeros((width, R, R), dtype=t.float64, device=dev)
    lv[:P] = rank_g[t.as_tensor(order, device=dev)]
    levels = [None] * (depth + 1)
    levels[depth] = lv
    for lev in range(depth - 1, -1, -1):
        levels[lev] = levels[lev + 1].reshape(-1, 2, R, R).sum(dim=1)
    node_dev = t.cat([x.reshape(-1) for x in levels]).contiguous()
    devstate = dict(U=Us, trees=trees, leaves=leaves, node_grams=node_dev,
                    rank_tree=ops.sts_rank_tree(rank_g, t.as_tensor(order, device=dev)),
                    leaf_rank=t.as_tensor(leaf_rank.astype(np.int32), device=dev))
    return LeverageTree(blocks.mode, [to_host(x) for x in levels], leaf_rank, blocks.lows.copy(),
                        blocks.his.copy(), offsets, None, leaf_block_size, dev=devstate)


def sts_sample(trees, k, J, gram_chain_pinv, grams, blocks_per_mode, seed, round_id=0,
               grid=None, ledger=None, uniform_override=None) -> SampleBatch:
    """(ref samplers.py:379-468)"""
    N = len(grams)
    R = np.asarray(gram_chain_pinv).shape[0]
    if J == 0:
        return _empty_batch(N, R)
    dev = require_cuda()
    t = torch()
    ops = ops_for(dev)
    first_i = next(i for i in range(N) if i != k and trees[i] is not None)
    P = len(trees[first_i].block_lo)
    cp = to_dev(gram_chain_pinv, dev, t.float64)
    G = to_dev(np.stack([np.asarray(g, dtype=np.float64) for g in grams]), dev, t.float64)
    X = t.full((N, J), -1, dtype=t.int64, device=dev)
    pmp = t.ones((N, J), dtype=t.float64, device=dev)
    H = t.ones((J, R), dtype=t.float64, device=dev)
    urow = t.zeros((J, R), dtype=t.float64, device=dev)
    resid = t.zeros(J, dtype=t.float64, device=dev)
    owner = t.as_tensor((np.arange(J, dtype=np.int64) * P) // J, device=dev).to(t.int32)
    rtop = t.zeros(J, dtype=t.float64, device=dev)
    M = t.zeros((R, R), dtype=t.float64, device=dev)
    ones = t.ones((J, R), dtype=t.float64, device=dev)
    hkey = t.zeros(J, dtype=t.int64, device=dev)
    ov_all = None
    if uniform_override is not None:
        ov_all = to_dev(np.asarray(uniform_override, dtype=np.float64).T.copy(), dev, t.float64)
    first = True
    for i in range(N):
        if i == k:
            continue
        tr = trees[i].dev
        ops.sts_cond(cp, G, i, k, M)
        key = rng.stream_key(seed, rng.WALK_UNIFORM, round_id, k, i)
        ov = ov_all[i] if ov_all is not None else None
        H_in = None if first else H
        dims = [int(tt.block_hi.max()) if tt is not None else 1 for tt in trees]
        hk, kb = ops.walk_key(X, dims, k, i, hkey)
        depth = trees[i].depth
        if P > 1 and depth > 0:
            ops.sts_rank_walk_grouped(tr["rank_tree"], P, tr["leaf_rank"], M, H_in, J, key, ov,
                                      owner, rtop, pmp[i], hkey=hk, key_bits=kb)
            for p in range(P):
                if tr["trees"][p] is None:
                    continue
                Up = tr["U"][p]
                if first:   # H = ones for every sample: a flat inverse CDF per rank
                    n = Up.shape[0]
                    dist = t.zeros(n, dtype=t.float64, device=dev)
                    cdf = t.zeros(n, dtype=t.float64, device=dev)
                    mass = t.zeros(1, dtype=t.float64, device=dev)
                    ops.arls_build(Up, M, dist, cdf, mass)
                    ops.sts_flat_local(cdf, dist, int(trees[i].block_lo[p]), mass, rtop, owner, p,
                                       J, X[i], pmp[i], resid)
                    continue
                ops.sts_walk(tr["trees"][p], Up, tr["leaves"][p], int(trees[i].block_lo[p]),
                             M, H_in, J, key, None, rtop, owner, p, X[i], pmp[i], resid, hkey=hk,
                             key_bits=kb)
            # samples routed to a rank without rows (ref samplers.py:341-342)
            ops.status.check("in sts_sample")
            if bool((X[i] < 0).any()):
                raise DegenerateWalkError("walk reached a rank with no rows")
            for p in range(P):
                if tr["trees"][p] is not None:
                    ops.fold_rows(urow, tr["U"][p], int(trees[i].block_lo[p]), X[i], True,
                                  owner, p)
        else:
            p = int(trees[i].leaf_rank[0]) if P > 1 else 0
            owner.fill_(p)
            if tr["trees"][p] is None:
                raise DegenerateWalkError("walk reached a rank with no rows")
            ops.sts_walk(tr["trees"][p], tr["U"][p], tr["leaves"][p], int(trees[i].block_lo[p]), M,
                         H_in, J, key, ov, None, None, 0, X[i], pmp[i], resid, hkey=hk,
                         key_bits=kb)
            ops.fold_rows(urow, tr["U"][p], int(trees[i].block_lo[p]), X[i], True)
        ops.hadamard_rows(H, urow, init=first)
        first = False
    ops.status.check("in sts_sample")
    return SampleBatch(to_host(X.T.contiguous()), to_host(H), to_host(pmp.T.contiguous()),
                       to_host(_prod_rows(pmp)), residual=to_host(resid), owner=to_host(owner).astype(np.int64))


def local_sts_leaf_search(h, block_rows, leaf_grams, leaf_offsets, cond, r, row_offset=0):
    """Finish one sample's search over a rank's local rows (ref samplers.py:348-358):
    returns the global row whose CDF segment (row masses (u_q . h)^T cond (u_q . h), rows
    in order) contains r.  `leaf_grams`/`leaf_offsets` describe the reference's flat leaf
    blocks; the device search builds its own tree over `block_rows`."""
    dev = require_cuda()
    t = torch()
    ops = ops_for(dev)
    W = to_dev(np.asarray(block_rows, dtype=np.float64), dev, t.float64)
    if W.shape[0] == 0:
        raise DegenerateWalkError("walk reached a rank with no rows")
    R = W.shape[1]
    offs = np.asarray(leaf_offsets)
    L = int(offs[1] - offs[0]) if offs.size > 1 else W.shape[0]
    L = max(1, min(64, L))
    tree = ops.sts_build(W, L)
    Mt = to_dev(np.asarray(cond, dtype=np.float64), dev, t.float64)
    Hh = to_dev(np.asarray(h, dtype=np.float64).reshape(1, R), dev, t.float64)
    ov = t.full((1,), float(r), dtype=t.float64, device=dev)
    X = t.full((1,), -1, dtype=t.int64, device=dev)
    pm = t.ones(1, dtype=t.float64, device=dev)
    rs = t.zeros(1, dtype=t.float64, device=dev)
    ur = t.zeros((1, R), dtype=t.float64, device=dev)
    ops.sts_walk(tree, W, L, 0, Mt, Hh, 1, (0, 0), ov, None, None, 0, X, pm, rs)
    ops.status.check("in local_sts_leaf_search")
    return int(row_offset + int(X.item()))


def krp_leverage_scores(factors, skip=None):
    """Brute-force KRP leverage scores (test-scale oracle, ref samplers.py:43-52)."""
    size = 1
    for i, U in enumerate(factors):
        if i != skip and U is not None:
            size *= U.shape[0]
    if size > ORACLE_GUARD:
        raise ValueError("oracle guard exceeded: %d rows > %d" % (size, ORACLE_GUARD))
    from .linalg import khatri_rao, pseudo_inverse
    dev = require_cuda()
    t = torch()
    A = to_dev(khatri_rao(factors, skip=skip), dev, t.float64)
    Gp = to_dev(pseudo_inverse(to_host(A.T @ A)), dev, t.float64)
    return to_host(t.clamp(((A @ Gp) * A).sum(dim=1), min=0.0))


def exact_krp_leverage_oracle(factors, skip=None):
    """(ref samplers.py:55-62)"""
    scores = krp_leverage_scores(factors, skip=skip)
    total = scores.sum()
    if total <= 0.0:
        raise ValueError("all leverage scores are zero")
    return scores / total
