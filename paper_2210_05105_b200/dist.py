"""Multi-GPU accumulator-stationary runs: one process per GPU, torch.distributed (NCCL over
NVLink/NVSwitch) for the plumbing.

The engine's bulk-synchronous round (engine.Cluster) is written against a communicator
with list semantics; `TorchComm` implements it for SPMD processes, each holding exactly
one rank state.  Collectives on the hot path (ref schedules.py:227-258 and SURVEY.md 8(e)):

* sampled rows: per STS constant mode, (row, step probability, residual, factor row) of
  every sample, as one fixed-size sum all-reduce of disjoint owner contributions (no
  host-side counts); per CP-ARLS-LEV mode, an all-gather-v of (row, probability, factor row)
  in rank order -- O(J (N-1) R) words per solve, independent of the tensor size;
* R x R block Grams (all-gather, summed in rank order -- also yields the STS rank tree);
* R column sums of squares for renormalisation; P rank masses for CP-ARLS-LEV.

There is no reduction of MTTKRP output: every rank writes its stationary row block.
"""

from __future__ import annotations

import os

from .device import torch


class TorchComm:
    """List-semantics collectives over torch.distributed (one local rank per process)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.P = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.ranks = [self.rank]
        self.words = 0      # 8-byte words this rank handed to sum all-reduces (exchange volume)

    def all_gather(self, local):
        """local: [tensor] (this rank's) -> list of P tensors, rank order."""
        (x,) = local
        x = x.contiguous()
        out = [torch().empty_like(x) for _ in range(self.P)]
        self.dist.all_gather(out, x, group=self.group)
        return out

    def all_gather_v(self, local, counts):
        """Variable leading sizes known to every rank: pad to the maximum count."""
        (x,) = local
        t = torch()
        m = max(int(c) for c in counts) if counts else 0
        shape = (max(m, 1),) + tuple(x.shape[1:])
        buf = t.zeros(shape, dtype=x.dtype, device=x.device)
        c = int(counts[self.rank])
        if c:
            buf[:c] = x[:c]
        out = [t.empty_like(buf) for _ in range(self.P)]
        self.dist.all_gather(out, buf, group=self.group)
        return [o[:int(counts[p])] for p, o in enumerate(out)]

    def all_reduce_sum(self, local):
        """In-place sum all-reduce of this rank's tensor; returns [tensor]."""
        (x,) = local
        self.words += x.numel()
        self.dist.all_reduce(x, op=self.dist.ReduceOp.SUM, group=self.group)
        return [x]

    def all_gather_obj(self, local):
        (x,) = local
        out = [None] * self.P
        self.dist.all_gather_object(out, x, group=self.group)
        return out

    def barrier(self):
        self.dist.barrier(group=self.group)


def comm_words_per_solve(J, R, N, P, sampler):
    """Sampled-row all-gather volume per solve summed over ranks (words), as the
    reference's closed form (ref grid.py:370-376)."""
    from .grid import as_gather_words_total_per_solve
    return as_gather_words_total_per_solve(J, R, N, P, sampler)


def make_spmd_cluster(dims, idx, vals, R, J, sampler, seed, grid_dims=None, leaf=None,
                      factors=None, trial=0, balance="rows", grid=None):
    """This process's rank of a P-GPU accumulator-stationary cluster.  idx/vals: the
    tensor's COO on this GPU (every rank may hold all of it; only the rows of its blocks
    are kept in its stores).  Ownership follows the reference processor grid."""
    import torch.distributed as dist
    from .device import require_cuda
    from .engine import Cluster, RankState
    from .grid import ProcessorGrid, optimal_grid
    from .linalg import init_factors
    dev = require_cuda()
    P = dist.get_world_size()
    rank = dist.get_rank()
    from .engine import make_grid
    if grid is None:   # (a caller that ingested only its blocks passes the grid it used)
        grid = make_grid(dims, P, grid_dims, idx, balance)
    if grid.P != P:
        raise ValueError("grid %s has %d ranks, world size is %d" % (grid.grid_dims, grid.P, P))
    if factors is None:
        factors, _ = init_factors(dims, R, seed, trial)
    st = RankState(rank, grid, dev, dims, R, J, sampler, seed, leaf=leaf)
    st.load_factor_blocks(factors)
    st.build_stores(idx, vals)
    cl = Cluster([st], TorchComm(), sampler, J, seed)
    for j in range(len(dims)):
        cl.rebuild(j)
    return cl


def env_rank():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))
