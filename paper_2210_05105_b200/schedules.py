"""One mode-k least-squares solve under the accumulator-stationary schedule -- drop-in for
ref schedules.py (SolveContext, draw_batch, solve_mode_accumulator_stationary,
solve_mode).  Host arrays in, host arrays out; every step runs on the GPU:
sampler kernels, weights, sketched Gram + pseudo-inverse, the fused sampled MTTKRP from
each rank's device store, and the update GEMM.

The tensor-stationary schedule (medium-grained, with a reduce-scatter of MTTKRP
accumulators) is outside this build's scope: the north star forbids a large reduction
collective on the hot path.  Requests for it raise ScheduleError.
"""

from __future__ import annotations

import time

import numpy as np

from .device import require_cuda, to_dev, to_host, torch
from .linalg import hadamard_gram_chain, pseudo_inverse
from .ops import ops_for
from .samplers import arls_lev_sample, sample_weights, sts_sample


class ScheduleError(ValueError):
    """Invalid schedule / sampler combination or missing state (ref schedules.py:31-32)."""


class SolveContext:
    """Everything one mode solve needs, shared across a run (ref schedules.py:35-61)."""

    def __init__(self, grid, schedule, sampler, J, factors, grams, local, ledger, seed,
                 workers=1):
        self.grid = grid
        self.schedule = schedule
        self.sampler = sampler
        self.J = J
        self.factors = factors
        self.grams = grams
        self.local = local
        self.ledger = ledger
        self.seed = seed
        self.workers = workers
        self.round_id = 0
        self.arls_states = [None] * len(factors)
        self.trees = [None] * len(factors)
        self.timings = {"sampling": 0.0, "gather": 0.0, "mttkrp": 0.0, "reduction": 0.0,
                        "postprocess": 0.0}
        self.stats = {"sampled_nnz": 0, "sampled_nnz_distinct": 0}

    def tick(self, phase, t0):
        t1 = time.perf_counter()
        self.timings[phase] += t1 - t0
        return t1


def draw_batch(ctx: SolveContext, k: int):
    """(ref schedules.py:86-101)"""
    t0 = time.perf_counter()
    if ctx.sampler == "arls-lev":
        full = [fb.assemble() for fb in ctx.factors]
        batch = arls_lev_sample(ctx.arls_states, k, ctx.J, full, ctx.seed, round_id=ctx.round_id)
    elif ctx.sampler == "sts":
        chain_pinv = pseudo_inverse(hadamard_gram_chain(ctx.grams, skip=k))
        batch = sts_sample(ctx.trees, k, ctx.J, chain_pinv, ctx.grams, ctx.factors, ctx.seed,
                           round_id=ctx.round_id, grid=ctx.grid)
    else:
        raise ScheduleError("no sampler configured (sampler=%r)" % ctx.sampler)
    ctx.tick("sampling", t0)
    return batch


def solve_mode_accumulator_stationary(ctx: SolveContext, k: int, injected_batch=None):
    """Replicated sampled rows, local sampled MTTKRP into each rank's stationary block,
    no reduction (ref schedules.py:227-258)."""
    if ctx.sampler == "exact" and injected_batch is None:
        raise ScheduleError("accumulator-stationary schedule requires a sampler; "
                            "exact solves must use tensor-stationary")
    if ctx.local.schedule != "accumulator-stationary":
        raise ScheduleError("context partition is %r" % ctx.local.schedule)
    batch = injected_batch if injected_batch is not None else draw_batch(ctx, k)
    if batch.weights is None:
        sample_weights(batch)
    t0 = time.perf_counter()
    dev = require_cuda()
    t = torch()
    ops = ops_for(dev)
    J = batch.J
    R = ctx.factors[0].R
    grid = ctx.grid
    H = to_dev(batch.H, dev, t.float64)
    w = to_dev(batch.weights, dev, t.float64)
    X = to_dev(np.ascontiguousarray(np.asarray(batch.X, dtype=np.int64).T), dev, t.int64)
    t0 = ctx.tick("gather", t0)
    Gs = ops.gram(H, scale=w) if J else t.zeros((R, R), dtype=t.float64, device=dev)
    Gsp = ops.pinv(Gs)
    stats = t.zeros(8, dtype=t.int64, device=dev)
    new_blocks = []
    for p in range(grid.P):
        mat = ctx.local.local(p, k)
        n = mat.n_rows
        out = t.zeros((n, R), dtype=t.float64, device=dev)
        if n and J and mat.nnz:
            st = mat.store
            ops.sampled_mttkrp(st, X, k, H, w, out, stats, cap=st.capacity(J))
        Unew = t.zeros((n, R), dtype=t.float64, device=dev)
        if n:
            colsq = t.zeros(R, dtype=t.float64, device=dev)
            ops.update(out, Gsp, Unew, colsq)
        new_blocks.append(Unew)
    ops.status.check("in solve_mode_accumulator_stationary")
    st_h = to_host(stats)
    ctx.stats["sampled_nnz"] += int(st_h[3])
    ctx.stats["sampled_nnz_distinct"] += int(st_h[2])
    t0 = ctx.tick("mttkrp", t0)
    ctx.factors[k].blocks = [np.ascontiguousarray(to_host(b)) for b in new_blocks]
    ctx.tick("postprocess", t0)
    return batch


def solve_mode(ctx: SolveContext, k: int, injected_batch=None):
    if ctx.schedule == "accumulator-stationary":
        return solve_mode_accumulator_stationary(ctx, k, injected_batch)
    if ctx.schedule == "tensor-stationary":
        raise ScheduleError("tensor-stationary schedule is not part of this build")
    raise ScheduleError("unknown schedule %r" % ctx.schedule)
