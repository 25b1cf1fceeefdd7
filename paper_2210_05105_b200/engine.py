"""Device-resident accumulator-stationary sketched ALS (the hot path, B200-native).

One `RankState` per GPU rank holds that rank's factor row blocks, per-mode sorted
nonzero stores, sampler structures and batch buffers -- all in HBM.  The round is written
bulk-synchronously over a list of rank states and a communicator:

* SPMD (`dist.TorchComm`, one process per GPU, NCCL): the list holds one rank state;
* simulation (`LocalComm`, one process, P virtual ranks): the list holds all P states and
  collectives are list operations -- the reference's own execution model (ref grid.py:1-20),
  used to check CP-ARLS-LEV parity at P > 1 on a single GPU.

Schedule of one mode-k solve (ref schedules.py:227-258, als.py:196-208):
  sampling  -> STS walk (rank-level levels replicated, local tree per owner) or CP-ARLS-LEV
               draws, then the sampled-row all-gather (J (N-1) (R+2) / R words)
  weights   -> w = 1/sqrt(J p)
  Gs        -> (H.w)^T (H.w), pinv           (replicated, no collective)
  mttkrp    -> local sampled MTTKRP into the stationary row block (no collective)
  update    -> U_k = M Gs^+, column sums of squares (R-word reduction), renormalise
  rebuild   -> per-rank block Gram (R x R all-gather), tree / leverage rebuild
"""

from __future__ import annotations

import math
import os
import time

import numpy as np

from . import rng
from .device import torch
from .grid import ProcessorGrid, optimal_grid
from .ops import ops_for
from .store import build_store, build_store_chunks

# Sampled-MTTKRP entry capacity above which the workspace is sized from the observed
# gathered-entry counts (checked after each call, grown and re-run on overflow) instead
# of the worst case min(nnz, J * longest fiber).
CAP_LIMIT = 1 << 28

PHASES = ("sampling", "gather", "mttkrp", "reduction", "postprocess", "rebuild")


def default_leaf(n, R, budget_bytes=4 << 30, walkers=None):
    """Rows per tree leaf: 8, doubled (<= 64) until the padded tree fits the budget and has
    at most 8 nodes per walking sample.  A leaf costs L row masses (L R^2/2 each) per
    walking run, a level one pair of node masses, so small leaves win (measured on C3:
    L = 8 beats 16 and 4) until the per-walk G (.) M pass over every node and the rebuild
    grow: with P ranks a rank walks about J / P samples, and a tree with many more nodes
    than walkers spends its time conditioning nodes nobody visits (C4 at P = 8: 0.46 ms
    per walk for the 1.5 GB tree of L = 8, 0.06 ms at L = 64)."""
    Rt = R * (R + 1) // 2
    L = 8
    while L < 64:
        nl = max(1, math.ceil(n / L))
        nodes = 2 * (1 << max(0, math.ceil(math.log2(nl)))) - 1
        if nodes * Rt * 8 <= budget_bytes and (walkers is None or nodes <= 8 * max(walkers, 1)):
            break
        L *= 2
    return L


class ShufflePrefetch:
    """Generator.permutation(J) of the CP-ARLS-LEV SHUFFLE streams (ref samplers.py:183-185)
    computed ahead on the host.  The permutation is a sequential rejection-sampling chain
    (host native code, ~1 ms for J = 65536); it depends only on (seed, round, k, i), so a
    background thread makes each upcoming round's N(N-1) permutations with one native
    call (`rcp_permutations_host`, several threads, one release of the interpreter lock)
    into a pinned (N, N, J) buffer while the GPU runs the current round; the eager path
    uploads them asynchronously and recycles the buffer once its copies completed."""

    def __init__(self, seed, J, N, ahead=2):
        import threading
        from concurrent.futures import ThreadPoolExecutor
        self.seed, self.J, self.N = int(seed), int(J), int(N)
        self.ahead = int(ahead)   # rounds requested beyond the one being consumed
        self.pool = ThreadPoolExecutor(max_workers=1)
        self.futs = {}            # round -> future of its pinned (N, N, J) buffer
        self.left = {}            # round -> pairs not yet copied out
        self.free = []            # recycled pinned buffers
        self.lock = threading.Lock()
        self.inflight = []        # (event, buffer) until the uploads are done

    def _buffer(self):
        with self.lock:
            if self.free:
                return self.free.pop()
        t = torch()
        return t.empty((self.N, self.N, self.J), dtype=t.int64, pin_memory=True)

    def fill(self, rnd, buf):
        """Write round rnd's permutations into buf[k, i] (k != i)."""
        pairs = [(k, i) for k in range(self.N) for i in range(self.N) if i != k]
        keys = [rng.stream_key(self.seed, rng.SHUFFLE, rnd, k, i) for k, i in pairs]
        rng.permutations_into(keys, self.J, [buf[k, i] for k, i in pairs],
                              threads=len(pairs))
        return buf

    def _request(self, rnd):
        for r in range(rnd, rnd + self.ahead + 1):
            if r not in self.futs:
                self.futs[r] = self.pool.submit(self.fill, r, self._buffer())
                self.left[r] = self.N * (self.N - 1)

    def copy_to(self, dst, rnd, k, i):
        t = torch()
        self._request(rnd)
        buf = self.futs[rnd].result()
        dst.copy_(buf[k, i], non_blocking=True)
        self.left[rnd] -= 1
        if self.left[rnd] == 0:   # every pair uploaded: recycle after the copies finish
            ev = t.cuda.Event()
            ev.record()
            self.inflight.append((ev, buf))
            self.futs.pop(rnd)
            self.left.pop(rnd)
        while self.inflight and self.inflight[0][0].query():
            with self.lock:
                self.free.append(self.inflight.pop(0)[1])
        for r in [q for q in self.futs if q < rnd]:   # rounds that will not come back
            self.futs.pop(r)
            self.left.pop(r, None)

class LocalComm:
    """P virtual ranks in one process (list collectives, rank order)."""

    def __init__(self, P):
        self.P = int(P)
        self.ranks = list(range(self.P))

    def all_gather(self, local):            # local: list (one per local rank) of tensors
        return list(local)

    def all_gather_v(self, local, counts):  # counts known to all ranks
        return list(local)

    def all_gather_obj(self, local):
        return list(local)

    def all_reduce_sum(self, local):
        """Sum over the virtual ranks in rank order; every rank gets the total."""
        tot = local[0].clone()
        for x in local[1:]:
            tot.add_(x)
        return [tot if p == 0 else tot.clone() for p in range(len(local))]

    def barrier(self):
        pass


class RankState:
    def __init__(self, rank, grid: ProcessorGrid, dev, dims, R, J, sampler, seed, leaf=None):
        t = torch()
        self.t = t
        self.rank = int(rank)
        self.grid = grid
        self.P = grid.P
        self.dev = dev
        self.dims = tuple(int(d) for d in dims)
        self.N = len(self.dims)
        self.R, self.J = int(R), int(J)
        self.sampler = sampler
        self.seed = int(seed)
        self.ops = ops_for(dev)
        N, R, J = self.N, self.R, self.J
        self.lo = [grid.block_range(j, rank)[0] for j in range(N)]
        self.n = [grid.block_range(j, rank)[1] - self.lo[j] for j in range(N)]
        self.leaf_cfg = leaf
        self.leaf = [None] * N
        f64 = dict(dtype=t.float64, device=dev)
        self.U = [t.zeros((self.n[j], R), **f64) for j in range(N)]
        self.grams = t.zeros((N, R, R), **f64)
        self.block_grams = [None] * N          # (P, R, R) per mode (P > 1)
        self.trees = [None] * N
        self.tree_stale = [True] * N
        self.tree_ev = [None] * N              # pending side-stream tree build per mode
        self._tree_stream = None
        self.rank_tree = [None] * N            # (node_grams, leaf_rank, depth) per mode
        self.dist = [None] * N
        self.cdf = [None] * N
        self.mass = [t.zeros(1, **f64) for _ in range(N)]
        self.C_host = [None] * N               # P rank masses per mode (ARLS)
        self.stores = [None] * N
        self.X = t.full((N, J), -1, dtype=t.int64, device=dev)
        self.pmp = t.ones((N, J), **f64)
        self.prob = t.ones(J, **f64)
        self.w = t.ones(J, **f64)
        self.resid = t.zeros(J, **f64)
        self.H = t.ones((J, R), **f64)
        self.H_alt = t.zeros((J, R), **f64)      # walk output buffer (swapped with H)
        self.owner = t.zeros(J, dtype=t.int32, device=dev)
        self.rtop = t.zeros(J, **f64)
        self.rows_tmp = t.zeros(J, dtype=t.int64, device=dev)
        self.prob_tmp = t.zeros(J, **f64)
        self.urow_tmp = t.zeros((J, R), **f64) if self.P > 1 else None
        self.perm = t.zeros(J, dtype=t.int64, device=dev)
        self.shuffles = None   # ShufflePrefetch, created on the first CP-ARLS-LEV fold
        self.hkey = t.zeros(J, dtype=t.int64, device=dev)
        self.flat_dist = self.flat_cdf = self.flat_mass = None
        self.chain_pinv = t.zeros((R, R), **f64)
        self.M = t.zeros((R, R), **f64)
        self.M_pre = t.zeros((R, R), **f64)    # conditioning matrix of the prefetched walk
        self.walk_ws = None                    # this rank's walk workspace (holds G (.) M')
        self.gm_ev = None                      # (mode, event) of a prefetched conditioning pass
        self.Gs = t.zeros((R, R), **f64)
        self.Gsp = t.zeros((R, R), **f64)
        self.Gp = t.zeros((R, R), **f64)
        self.colsq = t.zeros(R, **f64)
        self.sigma = t.ones(R, **f64)
        self.Mout = t.zeros((max(self.n) if N else 0, R), **f64)
        self.stats = t.zeros(8, dtype=t.int64, device=dev)
        self.mt_cap = {}
        self.dkeys = None        # (N, N, 2) stream keys of the round's draws (graph mode)
        self._rank_order = {}    # mode -> (rank row order, padded leaf ranks) on the device
        self.gperm = None        # (N, N, J) SHUFFLE permutations of the round (graph mode)
        self.block_gram_buf = t.zeros((R, R), **f64)

    # -------------------------------------------------------------- set-up
    def load_factor_blocks(self, full_factors):
        """full_factors: list of host (I_j x R) arrays; keep this rank's block."""
        t = self.t
        for j in range(self.N):
            blk = np.ascontiguousarray(full_factors[j][self.lo[j]:self.lo[j] + self.n[j]],
                                       dtype=np.float64)
            self.U[j].copy_(t.from_numpy(blk))

    def build_stores(self, idx, vals):
        """idx/vals: device COO of the whole tensor (or a superset); keeps, per mode, the
        nonzeros whose mode-j row lies in this rank's block (ref matricization.py:187-198)."""
        if isinstance(idx, list):   # device-ingest chunks (C4/C5): bucketed build
            for j in range(self.N):
                self.stores[j] = build_store_chunks(self.dims, idx, j, self.lo[j],
                                                    self.lo[j] + self.n[j])
            return
        for j in range(self.N):
            rows = idx[:, j]
            sel = (rows >= self.lo[j]) & (rows < self.lo[j] + self.n[j])
            if self.P == 1:
                self.stores[j] = build_store(self.dims, idx, vals, j, self.lo[j], self.lo[j] + self.n[j])
            else:
                self.stores[j] = build_store(self.dims, idx[sel], vals[sel], j, self.lo[j],
                                             self.lo[j] + self.n[j])

    def leaf_of(self, j):
        if self.leaf[j] is None:
            if self.leaf_cfg is not None:
                self.leaf[j] = int(max(1, min(64, int(self.leaf_cfg))))
            else:
                self.leaf[j] = default_leaf(max(self.n[j], 1), self.R,
                                            walkers=max(1, self.J // self.P))
        return self.leaf[j]

    # ------------------------------------------------------------- rebuild
    def block_gram(self, k):
        return self.ops.gram(self.U[k], out=self.block_gram_buf)

    def set_gram(self, k, blocks):
        """blocks: list of P (R x R) tensors in rank order -> ordered sum (ref grid.py:295-297)."""
        if self.P == 1:
            self.grams[k].copy_(blocks[0])
            return
        bg = self.block_grams[k]   # persistent per mode: a graph replay reads its address
        if bg is None:
            bg = self.block_grams[k] = self.t.empty((self.P, self.R, self.R),
                                                    dtype=self.t.float64, device=self.dev)
        self.t.stack(list(blocks), out=bg)
        self.ops.ordered_sum(bg, self.grams[k])

    def build_tree(self, k):
        """Mark the local tree of mode k stale (it is rebuilt on its first walk: at P = 1 the
        first constant mode draws from a flat CDF, so mode 0's tree is never walked there)
        and rebuild the small rank-level tree."""
        self.tree_stale[k] = True
        if self.P > 1:
            self._build_rank_tree(k)

    def prefetch_trees(self, modes):
        """Build the stale trees of `modes` on a side stream: they depend only on the
        factors, so they overlap the chain pseudo-inverse, the conditioning and the first
        constant mode's flat draw; the walk that reads a tree waits for its event."""
        t = self.t
        pend = [i for i in modes if self.tree_stale[i] and self.n[i] > 0]
        if not pend:
            return
        main = t.cuda.current_stream()
        if self._tree_stream is None:
            self._tree_stream = t.cuda.Stream(device=main.device)
        s = self._tree_stream
        s.wait_stream(main)
        with t.cuda.stream(s):
            for i in pend:
                self.trees[i] = self.ops.sts_build(self.U[i], self.leaf_of(i), self.trees[i])
                self.tree_stale[i] = False
                ev = t.cuda.Event()
                ev.record()
                self.tree_ev[i] = ev

    def prefetch_gm(self, i, k):
        """The conditioning pass of the first walked mode (G (.) M' for every node of its
        tree) on the tree stream: it needs only the chain pseudo-inverse and the tree, so
        it overlaps the first constant mode's draw; the walk waits for its event."""
        if self.n[i] == 0:
            return
        t = self.t
        main = t.cuda.current_stream()
        if self._tree_stream is None:
            self._tree_stream = t.cuda.Stream(device=main.device)
        s = self._tree_stream
        n, leaf = self.n[i], self.leaf_of(i)
        self.walk_ws = self.ops.sts_walk_ws(self.J, n, leaf, self.R, self.walk_ws, owned=True)
        s.wait_stream(main)   # the chain pseudo-inverse; the previous solve's walk
        with t.cuda.stream(s):
            tree = self.local_tree(i)
            self.ops.sts_cond(self.chain_pinv, self.grams, i, k, self.M_pre)
            self.ops.sts_walk_gm(tree, n, leaf, self.M_pre, self.J, self.walk_ws)
            ev = t.cuda.Event()
            ev.record()
        self.gm_ev = (i, ev)

    def local_tree(self, k):
        if self.tree_ev[k] is not None:
            self.t.cuda.current_stream().wait_event(self.tree_ev[k])
            self.tree_ev[k] = None
        if self.tree_stale[k] and self.n[k] > 0:
            self.trees[k] = self.ops.sts_build(self.U[k], self.leaf_of(k), self.trees[k])
        self.tree_stale[k] = False
        return self.trees[k]

    def _build_rank_tree(self, k):
        """Padded complete tree over ranks in global row order (ref samplers.py:239-275)."""
        t = self.t
        P, R = self.P, self.R
        depth = int(math.ceil(math.log2(P))) if P > 1 else 0
        width = 1 << depth
        idx = self._rank_order.get(k)
        if idx is None:   # fixed by the grid: uploaded once (no host copies inside a capture)
            order = self.grid.row_order(k)
            leaf_rank = np.full(width, -1, dtype=np.int32)
            leaf_rank[:P] = order
            idx = self._rank_order[k] = (
                t.as_tensor(np.asarray(order, dtype=np.int64), device=self.dev),
                t.as_tensor(leaf_rank, device=self.dev))
        old = self.rank_tree[k]   # one buffer per mode, rewritten in place (graph replays)
        tree = self.ops.sts_rank_tree(self.block_grams[k], idx[0], old[0] if old else None)
        self.rank_tree[k] = (tree, idx[1], depth)

    def arls_local(self, k):
        """Local leverage distribution of mode k given the replicated Gram (ref
        samplers.py:122-135); returns the device mass scalar."""
        ops = self.ops
        ops.pinv(self.grams[k], out=self.Gp)
        n = self.n[k]
        if self.dist[k] is None or self.dist[k].shape[0] != n:
            self.dist[k] = self.t.zeros(n, dtype=self.t.float64, device=self.dev)
            self.cdf[k] = self.t.zeros(n, dtype=self.t.float64, device=self.dev)
        if n > 0:
            ops.arls_build(self.U[k], self.Gp, self.dist[k], self.cdf[k], self.mass[k])
        else:
            self.mass[k].zero_()
        return self.mass[k]

    # ------------------------------------------------------------ sampling
    def chain(self, k):
        self.ops.pinv(self.grams, n_chain=self.N, skip=k, out=self.chain_pinv)

    def sts_mode(self, i, k, rnd, first, override=None):
        """Walk all samples for constant mode i; this rank completes the samples whose
        leaf lies in its block (all of them when P == 1)."""
        ops = self.ops
        gm_ready = self.gm_ev is not None and self.gm_ev[0] == i
        if gm_ready:   # conditioning matrix and G (.) M' made ahead on the tree stream
            self.t.cuda.current_stream().wait_event(self.gm_ev[1])
            self.gm_ev = None
            M = self.M_pre
        else:
            M = self.M
            ops.sts_cond(self.chain_pinv, self.grams, i, k, M)
        if self.dkeys is not None:   # graph-replayed round: the key is read on the device
            key = self.dkeys[k, i]
        else:
            key = rng.stream_key(self.seed, rng.WALK_UNIFORM, rnd, k, i)
        H_in = None if first else self.H
        hk, kb = ops.walk_key(self.X, self.dims, k, i, self.hkey)
        if self.P > 1:
            # the rank-level levels, replicated: every rank learns every sample's owner
            rtree, leaf_rank, _ = self.rank_tree[i]
            ops.sts_rank_walk_grouped(rtree, self.P, leaf_rank, M, H_in, self.J, key, override,
                                      self.owner, self.rtop, self.pmp[i], hkey=hk, key_bits=kb)
            sel, rin = self.owner, self.rtop
        else:   # the walk / flat draw sets every sample's probability (no rank-level factor)
            sel, rin = None, None
        if first and (self.P > 1 or (override is None and self.n[i] > 0)):
            # every sample shares H = ones: one inverse CDF over the local rows' masses
            # u M u^T -- all J draws at P = 1, the residuals of the samples routed to this
            # rank at P > 1 (ref _leaf_search_batch samplers.py:313-345)
            t = self.t
            n = self.n[i]
            if self.flat_dist is None or self.flat_dist.shape[0] < n:
                self.flat_dist = t.zeros(max(self.n), dtype=t.float64, device=self.dev)
                self.flat_cdf = t.zeros(max(self.n), dtype=t.float64, device=self.dev)
                self.flat_mass = t.zeros(1, dtype=t.float64, device=self.dev)
            if n > 0:
                ops.arls_build(self.U[i], M, self.flat_dist[:n], self.flat_cdf[:n],
                               self.flat_mass)
            else:
                self.flat_mass.zero_()
            if self.P > 1:
                ops.sts_flat_local(self.flat_cdf[:n], self.flat_dist[:n], self.lo[i],
                                   self.flat_mass, rin, sel, self.rank, self.J, self.X[i],
                                   self.pmp[i], self.resid)
                return
            ops.sts_flat_draw(self.flat_cdf[:n], self.flat_dist[:n], self.lo[i], self.flat_mass,
                              key, self.J, self.X[i], self.pmp[i])
            ops.fold_rows(self.H, self.U[i], self.lo[i], self.X[i], init=True)
            return
        if self.n[i] > 0:
            fused = self.P == 1   # the walk folds U rows into the Hadamard rows itself
            self.walk_ws = ops.sts_walk_ws(self.J, self.n[i], self.leaf_of(i), self.R, self.walk_ws,
                                            owned=True)
            ops.sts_walk(self.local_tree(i), self.U[i], self.leaf_of(i), self.lo[i], M, H_in,
                         self.J, key, override if self.P == 1 else None, rin, sel, self.rank,
                         self.X[i], self.pmp[i], self.resid, hkey=hk, key_bits=kb,
                         H_out=self.H_alt if fused else None, ws=self.walk_ws, gm_ready=gm_ready)
            if fused:
                self.H, self.H_alt = self.H_alt, self.H

    def _ones_H(self):
        if not hasattr(self, "_H1"):
            self._H1 = self.t.ones((self.J, self.R), dtype=self.t.float64, device=self.dev)
        return self._H1

    def arls_draw(self, i, k, rnd, quota, W):
        """This rank's quota of draws for constant mode i (ref samplers.py:169-181);
        staged in rows_tmp/prob_tmp (and urow_tmp when P > 1)."""
        q = int(quota[self.rank]) if self.P > 1 else self.J
        if q == 0:
            return 0
        if self.dkeys is not None:   # graph-replayed round: the key is read on the device
            key = self.dkeys[k, i]
        else:
            key = rng.stream_key(self.seed, rng.LOCAL_DRAW, rnd, k, i, self.rank)
        if self.P > 1:
            ratio = float(self.C_host[i][self.rank]) / W
            tmass = None
        else:
            ratio = 1.0
            tmass = self.mass[i]
        self.ops.arls_draw(self.cdf[i], self.dist[i], self.lo[i], ratio, tmass, key, q, 0,
                           self.rows_tmp, self.prob_tmp,
                           U=self.U[i] if self.P > 1 else None,
                           urow_out=self.urow_tmp if self.P > 1 else None)
        return q

    def arls_fold(self, i, k, rnd, first, rows, probs, urows):
        if self.gperm is not None:   # graph-replayed round: permutations uploaded beforehand
            perm = self.gperm[k, i]
        else:
            if self.shuffles is None:
                self.shuffles = ShufflePrefetch(self.seed, self.J, self.N)
            self.shuffles.copy_to(self.perm, rnd, k, i)
            perm = self.perm
        self.ops.batch_fold(perm, rows, probs, self.U[i] if urows is None else None,
                            self.lo[i], urows, first, self.X[i], self.pmp[i], self.H)

    # --------------------------------------------------------------- solve
    def weights(self):
        self.ops.weights(self.pmp, self.prob, self.w)

    def sketched_system(self):
        """Gs = (H.w)^T (H.w) and its pseudo-inverse (ref schedules.py:104-109, :258)."""
        self.ops.gram(self.H, scale=self.w, out=self.Gs)
        self.ops.pinv(self.Gs, out=self.Gsp)

    def mttkrp(self, k):
        n = self.n[k]
        out = self.Mout[:n]
        if n > 0:
            st = self.stores[k]
            worst = st.capacity(self.J)
            if worst <= CAP_LIMIT:
                self.ops.sampled_mttkrp(st, self.X, k, self.H, self.w, out, self.stats, cap=worst)
                return out
            # bounded workspace: the call is idempotent (reads X, H, w; writes out), so an
            # overflowing call is repeated with the exact requirement
            cap = self.mt_cap.get(k, CAP_LIMIT)
            stats0 = self.stats.clone()
            while True:
                need, have = self.ops.sampled_mttkrp(st, self.X, k, self.H, self.w, out,
                                                     self.stats, cap=cap, need=True)
                if need <= have:
                    break
                self.ops.status.clear_flag(_lib_capacity())
                self.stats.copy_(stats0)
                cap = min(worst, int(need * 1.25) + (1 << 20))
            self.mt_cap[k] = cap
        return out

    def update(self, k):
        n = self.n[k]
        if n > 0:
            self.ops.update(self.Mout[:n], self.Gsp, self.U[k], self.colsq)
        else:
            self.colsq.zero_()
        return self.colsq

    def stage_colsq(self, parts):
        """parts: the P ranks' column sums of squares in rank order (P > 1)."""
        if getattr(self, "colsq_parts", None) is None:
            self.colsq_parts = self.t.empty((self.P, self.R), dtype=self.t.float64, device=self.dev)
        self.t.stack(list(parts), out=self.colsq_parts)

    def renormalize(self, k):
        """colsq: this rank's sums (P = 1) or the rank-ordered total of the staged parts."""
        if self.P > 1:
            self.ops.ordered_sum(self.colsq_parts, self.colsq)
        if self.n[k] > 0:
            self.ops.renormalize(self.U[k], self.colsq, self.sigma)
        else:
            self.sigma.copy_(self.t.sqrt(self.colsq))


class Cluster:
    """Bulk-synchronous driver over the rank states of this process."""

    def __init__(self, ranks, comm, sampler, J, seed):
        self.ranks = ranks
        self.comm = comm
        self.sampler = sampler
        self.J = int(J)
        self.seed = int(seed)
        self.N = ranks[0].N
        self.P = ranks[0].P
        self.timings = {p: 0.0 for p in PHASES}
        self.timed = False
        self.phase_events = None
        self._side = None
        self._nvtx_open = False

    def _tick(self, phase, t0):
        if not self.timed:
            return t0
        torch().cuda.synchronize()
        t1 = time.perf_counter()
        self.timings[phase] += t1 - t0
        return t1

    # ------------------------------------------------------------ rebuild
    def rebuild(self, k):
        """(ref als.py:114-126)"""
        blocks = self.comm.all_gather([r.block_gram(k) for r in self.ranks])
        for r in self.ranks:
            r.set_gram(k, [b for b in blocks])
        if self.sampler == "sts":
            for r in self.ranks:
                r.build_tree(k)
        else:
            masses = [r.arls_local(k) for r in self.ranks]
            if self.P > 1:
                allm = self.comm.all_gather(masses)
                # the P rank masses feed the host multinomial (numpy's binomial chain is part
                # of the reference's random-stream contract): one device-to-host read
                C = torch().cat([m.reshape(-1)[:1] for m in allm]).cpu().numpy().astype(np.float64)
                for r in self.ranks:
                    r.C_host[k] = C

    # ------------------------------------------------------------ sampling
    def sample(self, k, rnd, override=None):
        N = self.N
        for r in self.ranks:
            r.X[k].fill_(-1)
            r.pmp[k].fill_(1.0)
        if self.sampler == "sts":
            walked = [i for i in range(N) if i != k]
            if self.P > 1 or override is None:
                walked = walked[1:]   # the first constant mode is a flat draw / flat local search
            for r in self.ranks:
                r.prefetch_trees(walked)
                r.chain(k)
                if walked:
                    r.prefetch_gm(walked[0], k)
            first = True
            for i in range(N):
                if i == k:
                    continue
                ov = None
                if override is not None:
                    ov = override[i]
                for r in self.ranks:
                    r.sts_mode(i, k, rnd, first, override=ov)
                if self.P > 1:
                    self._exchange_walk(i, first)
                first = False
        else:
            first = True
            for i in range(N):
                if i == k:
                    continue
                quota, W = self._arls_quota(i, k, rnd)
                for r in self.ranks:
                    r.arls_draw(i, k, rnd, quota, W)
                if self.P > 1:
                    cat_rows, cat_probs, cat_urows = self._gather_arls_draws(quota)
                    for r in self.ranks:
                        r.arls_fold(i, k, rnd, first, cat_rows.to(r.dev), cat_probs.to(r.dev),
                                    cat_urows.to(r.dev))
                else:
                    for r in self.ranks:
                        r.arls_fold(i, k, rnd, first, r.rows_tmp, r.prob_tmp, None)
                first = False
        for r in self.ranks:
            r.weights()

    def _gather_arls_draws(self, quota):
        """Concatenate every rank's local draws in rank order (ref samplers.py:181-182):
        one all-gather-v of [row, probability, factor row] per draw (R+2 words)."""
        t = torch()
        counts = [int(q) for q in quota]
        packs = []
        for r in self.ranks:
            q = counts[r.rank]
            packs.append(t.cat([r.rows_tmp[:q].to(t.float64).unsqueeze(1),
                                r.prob_tmp[:q].unsqueeze(1), r.urow_tmp[:q]], dim=1).contiguous())
        got = self.comm.all_gather_v(packs, counts)
        cat = t.cat([got[p][:counts[p]] for p in range(self.P)])
        return (cat[:, 0].to(t.int64).contiguous(), cat[:, 1].contiguous(),
                cat[:, 2:].contiguous())

    def _arls_quota(self, i, k, rnd):
        """Consistent multinomial split of J over rank masses (ref samplers.py:138-145);
        trivial at P = 1 (zero-mass is raised on the device)."""
        if self.P == 1:
            return np.array([self.J]), 1.0
        C = self.ranks[0].C_host[i]
        W = float(C.sum())
        if W <= 0.0:
            raise ValueError("mode %d has zero total leverage mass" % i)
        gen = rng.stream(self.seed, rng.MULTINOMIAL, rnd, k, i)
        return gen.multinomial(self.J, C / W), W

    def _exchange_walk(self, i, first):
        """After the local walks, every rank holds the finished samples it owns; move
        (row, step probability, residual, factor row) of every sample to all ranks
        (ref schedules.py:239-247: R+2 words per sample per constant mode, plus the
        residual here).  Every rank knows every sample's owner (the rank-level walk is
        replicated), so the exchange is one fixed-size J x (R+3) sum all-reduce of disjoint
        contributions: each slot has exactly one nonzero contributor, the sum is exact,
        and nothing depends on host-side counts (no host synchronisation; capturable in a
        CUDA graph)."""
        t = torch()
        bufs = []
        for r in self.ranks:
            buf = getattr(r, "xbuf", None)
            if buf is None or buf.shape != (r.J, r.R + 3):
                buf = r.xbuf = t.empty((r.J, r.R + 3), dtype=t.float64, device=r.dev)
            r.ops.exchange_pack(r.X[i], r.pmp[i], r.resid, r.U[i], r.lo[i], r.owner, r.rank, buf)
            bufs.append(buf)
        got = self.comm.all_reduce_sum(bufs)
        for r, g in zip(self.ranks, got):
            r.ops.exchange_unpack(g, first, r.X[i], r.pmp[i], r.resid, r.H)

    # -------------------------------------------------------------- solve
    def _ev(self, phase):
        """Phase boundary: closes the previous NVTX range and opens `phase` (ranges are
        named after the reference's ctx.timings phases, ref schedules.py:227-258; visible
        in nsys/ncu --nvtx), and records a CUDA event on the current stream when
        profiling."""
        nv = torch().cuda.nvtx
        if self._nvtx_open:
            nv.range_pop()
            self._nvtx_open = False
        if phase != "end":
            nv.range_push("rcp:" + phase)
            self._nvtx_open = True
        if self.phase_events is None:
            return
        e = torch().cuda.Event(enable_timing=True)
        e.record()
        self.phase_events.append((phase, e))

    def solve(self, k, rnd, override=None, injected=None, check=False):
        """One mode-k solve.  check=True synchronises after the sampler and raises its
        errors there, where the reference raises them (ref samplers.py:34-35,93-94,
        142-143): not usable inside a CUDA-graph capture."""
        t0 = time.perf_counter()
        self._ev("sampling")
        if injected is None:
            self.sample(k, rnd, override=override)
        else:
            for r in self.ranks:
                injected(r)
        if check:
            self.check("after round %d mode %d sampling" % (rnd, k))
        t0 = self._tick("sampling", t0)
        # Gs = (H w)^T (H w) and its pseudo-inverse depend only on the batch: they run on a
        # side stream, overlapped with the sampled MTTKRP, and join before the update
        self._ev("gram+pinv")
        t = torch()
        main = t.cuda.current_stream()
        if self._side is None:
            self._side = t.cuda.Stream(device=main.device)
        self._side.wait_stream(main)
        with t.cuda.stream(self._side):
            for r in self.ranks:
                r.sketched_system()
        self._ev("mttkrp")
        for r in self.ranks:
            r.mttkrp(k)
        main.wait_stream(self._side)
        t0 = self._tick("mttkrp", t0)
        self._ev("update")
        parts = self.comm.all_gather([r.update(k) for r in self.ranks])
        if self.P > 1:   # every rank reads all parts before any rank overwrites its own
            for r in self.ranks:
                r.stage_colsq(parts)
        for r in self.ranks:
            r.renormalize(k)
        t0 = self._tick("postprocess", t0)
        self._ev("rebuild")
        self.rebuild(k)
        self._tick("rebuild", t0)
        self._ev("end")

    # ------------------------------------------------------------ exact fit (F1)
    def full_factor(self, j):
        """Full mode-j factor on each local rank's device: the row blocks all-gathered and
        placed at their global offsets.  Returns one tensor per local rank."""
        t = torch()
        grid = self.ranks[0].grid
        counts = [grid.block_range(j, p)[1] - grid.block_range(j, p)[0] for p in range(self.P)]
        blocks = self.comm.all_gather_v([r.U[j] for r in self.ranks], counts)
        outs = []
        for r in self.ranks:
            full = t.empty((r.dims[j], r.R), dtype=t.float64, device=r.dev)
            for p, blk in enumerate(blocks):
                lo = grid.block_range(j, p)[0]
                if counts[p]:
                    full[lo:lo + counts[p]].copy_(blk[:counts[p]])
            outs.append(full)
        return outs

    def fit(self):
        """Exact fit 1 - ||T - T_hat||_F / ||T||_F of the current model (ref compute_fit
        linalg.py:130-151), computed on the devices from the last-mode stores: every rank
        adds v <sigma (.) prod U_m[i_m], U_last[row]> over its nonzeros, ||T||^2 over the
        same store (cached), ||T_hat||^2 = sigma^T (Hadamard of the Grams) sigma.  One
        all-gather of two scalars per rank at P > 1; nothing is copied to the host but the
        three scalars."""
        t = torch()
        N = self.N
        last = N - 1
        fulls = [self.full_factor(j) if j != last else None for j in range(N)]
        parts = []
        for q, r in enumerate(self.ranks):
            st = r.stores[last]
            v = t.zeros(3, dtype=t.float64, device=r.dev)
            if getattr(r, "norm_sq", None) is None:
                r.norm_sq = t.zeros(1, dtype=t.float64, device=r.dev)
                r.ops.sum_squares(st.vals, r.norm_sq)
            v[0:1].copy_(r.norm_sq)
            if st.nnz:
                facs = [fulls[m][q] if m != last else None for m in range(N)]
                r.ops.fit_cross(st, facs, [0] * N, r.U[last], r.sigma, v[1:2])
            parts.append(v)
        allp = self.comm.all_gather(parts)
        tot = allp[0].clone()
        for p in allp[1:]:
            tot += p.to(tot.device)
        r0 = self.ranks[0]
        model = t.zeros(1, dtype=t.float64, device=r0.dev)
        r0.ops.model_norm(r0.grams, r0.sigma, model)
        norm_sq, cross = (float(x) for x in tot[:2].cpu())
        model_sq = float(model.cpu())
        if norm_sq == 0.0:
            raise ValueError("fit is undefined for an all-zero tensor")
        resid_sq = max(norm_sq - 2.0 * cross + model_sq, 0.0)
        return 1.0 - math.sqrt(resid_sq) / math.sqrt(norm_sq)

    def phase_breakdown(self):
        """ms per phase from the recorded events (after synchronisation)."""
        out = {}
        ev = self.phase_events or []
        for (name, a), (_, b) in zip(ev, ev[1:]):
            if name == "end":
                continue
            out[name] = out.get(name, 0.0) + a.elapsed_time(b)
        return out

    def check(self, where=""):
        for r in self.ranks:
            r.ops.status.check(where)

    def round(self, rnd, check=True, on_solved=None):
        """One ALS round; on_solved(k) is called (host side, stream-ordered) once factor k
        is final for the round (after its update and renormalisation)."""
        for k in range(self.N):
            self.solve(k, rnd)
            if on_solved is not None:
                on_solved(k)
            if check:
                self.check("after round %d mode %d solve" % (rnd, k))

    # ------------------------------------------------------------ CUDA-graph rounds
    def graph_ok(self):
        """A round is replayable from a CUDA graph when nothing in it depends on the host
        between launches: its per-round host inputs (the draw keys and, for CP-ARLS-LEV,
        the SHUFFLE permutations) move to device memory before the replay, and workspaces
        are sized up front (no bounded-capacity MTTKRP, which checks its entry count on
        the host).  P > 1: STS-CP rounds only (CP-ARLS-LEV splits J over the rank masses
        with a host multinomial, ref samplers.py:138-145), with the virtual ranks of one
        process (LocalComm); SPMD rounds (NCCL collectives inside the capture) only with
        RCP_GRAPH_SPMD=1."""
        if not all(st.capacity(self.J) <= CAP_LIMIT for r in self.ranks for st in r.stores):
            return False
        if self.P == 1:
            return True
        if self.sampler != "sts":
            return False
        return isinstance(self.comm, LocalComm) or os.environ.get("RCP_GRAPH_SPMD") == "1"

    def round_graph(self, rnd, on_solved=None, join=(), tag="round"):
        """One ALS round replayed from a CUDA graph (captured on the first call, after at
        least one eager round has sized every workspace).  The round's draw keys (and
        CP-ARLS-LEV's SHUFFLE permutations) are uploaded to device memory before each
        replay, from pinned staging filled while the previous replay runs; the replay
        issues the same kernels with the same arguments as an eager round
        (tests/test_gpu_graph.py).
        on_solved/join: as in round(), with the side streams its work forks into (joined
        before the capture ends); one graph is kept per `tag`."""
        t = torch()
        if not self.graph_ok():
            raise RuntimeError("this cluster's rounds cannot be replayed from a graph")
        r = self.ranks[0]
        N = self.N
        arls = self.sampler != "sts"
        if r.dkeys is None:
            for q in self.ranks:   # STS keys are rank-independent; ARLS graphs are P = 1
                q.dkeys = t.zeros((N, N, 2), dtype=t.int64, device=q.dev)
            self._gkeys = [t.zeros((N, N, 2), dtype=t.int64, pin_memory=True) for _ in range(2)]
            if arls:
                r.gperm = t.zeros((N, N, self.J), dtype=t.int64, device=r.dev)
                self._gperm = [t.zeros((N, N, self.J), dtype=t.int64, pin_memory=True)
                               for _ in range(2)]
                if r.shuffles is None:
                    r.shuffles = ShufflePrefetch(self.seed, self.J, N)
            self._gkey_ev = [None, None]
            self._gready = {}   # round -> staging slot holding its inputs
        slot = self._gready.pop(rnd, None)
        self._gready.clear()   # inputs staged for any other round are stale
        if slot is None:
            slot = self._graph_stage(rnd, 0)
        for q in self.ranks:
            q.dkeys.copy_(self._gkeys[slot], non_blocking=True)
        if arls:
            r.gperm.copy_(self._gperm[slot], non_blocking=True)
        ev = t.cuda.Event()
        ev.record()
        self._gkey_ev[slot] = ev
        if not hasattr(self, "_graphs"):
            self._graphs = {}
        g = self._graphs.get(tag)
        if g is None:
            from . import _lib
            lib = _lib.lib()
            g = t.cuda.CUDAGraph()
            n0 = lib.rcp_launch_count()
            with t.cuda.graph(g):
                self.round(rnd, check=False, on_solved=on_solved)
                cap = t.cuda.current_stream()
                for st in join:
                    cap.wait_stream(st)
            self.graph_kernels = lib.rcp_launch_count() - n0
            self._graphs[tag] = g
        g.replay()
        # the next round's inputs are staged in the other slot while the GPU runs this one
        self._gready[rnd + 1] = self._graph_stage(rnd + 1, 1 - slot)

    def _graph_stage(self, rnd, slot):
        """Write round rnd's draw keys (and permutations) into pinned staging slot `slot`."""
        r = self.ranks[0]
        N = self.N
        if self._gkey_ev[slot] is not None:
            self._gkey_ev[slot].synchronize()   # the slot's previous upload is done
        host = np.zeros((N, N, 2), dtype=np.uint64)
        for k in range(N):
            for i in range(N):
                if i == k:
                    continue
                if self.sampler == "sts":
                    host[k, i] = rng.stream_key(self.seed, rng.WALK_UNIFORM, rnd, k, i)
                else:
                    host[k, i] = rng.stream_key(self.seed, rng.LOCAL_DRAW, rnd, k, i, r.rank)
        if self.sampler != "sts":   # native threads, straight into the pinned slot
            r.shuffles.fill(rnd, self._gperm[slot])
        self._gkeys[slot].numpy()[...] = host.view(np.int64)
        return slot


def _lib_capacity():
    from . import _lib
    return _lib.ST_CAPACITY


def make_grid(dims, P, grid_dims, idx, balance="rows"):
    """The AS processor grid: reference equal-row blocks, or nnz-balanced blocks."""
    from .grid import nnz_row_weights
    if balance not in ("rows", "nnz"):
        raise ValueError("balance must be 'rows' or 'nnz'")
    rw = nnz_row_weights(dims, idx) if balance == "nnz" else None
    if grid_dims is not None:
        return ProcessorGrid(dims, grid_dims, row_weights=rw)
    return optimal_grid(dims, P, row_weights=rw)


def make_local_cluster(dims, idx, vals, R, J, sampler, seed, P=1, grid_dims=None, leaf=None,
                       factors=None, trial=0, balance="rows"):
    """Single-process cluster (P virtual ranks on the current device).  idx/vals are CUDA
    tensors; factors default to the reference initialisation (ref als.py:99-105).
    balance="rows": the reference's equal-row blocks (parity); "nnz": nnz-balanced blocks
    (grid.ProcessorGrid row_weights; performance runs)."""
    from .device import require_cuda
    dev = require_cuda()
    grid = make_grid(dims, P, grid_dims, idx, balance)
    if factors is None:
        from .linalg import init_factors
        factors, _ = init_factors(dims, R, seed, trial)
    ranks = []
    for p in range(grid.P):
        r = RankState(p, grid, dev, dims, R, J, sampler, seed, leaf=leaf)
        r.load_factor_blocks(factors)
        r.build_stores(idx, vals)
        ranks.append(r)
    cl = Cluster(ranks, LocalComm(grid.P), sampler, J, seed)
    for j in range(len(dims)):
        cl.rebuild(j)
    return cl
