"""Multi-rank host logic on CPU: world_size 2 over gloo (127.0.0.1).

Covers the product communicator (dist.TorchComm) and the engine's real exchange steps --
the STS sampled-row all-gather-v (owner-packed rows scattered back into sample order) and
the CP-ARLS-LEV rank-order concatenation -- with rank states that carry only the arrays
those steps touch.  The CUDA kernels around them are exercised by the GPU tests."""

import os
import socket
import types

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2210_05105_b200 import grid as G
from paper_2210_05105_b200.dist import TorchComm, comm_words_per_solve
from paper_2210_05105_b200.engine import Cluster


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class _HostOps:
    """Test double for the two exchange kernels (rcp_exchange_pack / rcp_exchange_unpack,
    include/randcp_b200.h) so that the Cluster's exchange logic runs on CPU tensors; the
    kernels themselves are checked against the same semantics in tests/test_gpu_engine.py."""

    @staticmethod
    def exchange_pack(Xi, pmp_i, resid, U, row_lo, owner, rank, buf):
        row = Xi - row_lo
        mine = (owner == rank) & (row >= 0) & (row < U.shape[0])
        buf.zero_()
        buf[mine, 0] = Xi[mine].to(torch.float64)
        buf[mine, 1] = pmp_i[mine]
        buf[mine, 2] = resid[mine]
        buf[mine, 3:] = U[row[mine]]

    @staticmethod
    def exchange_unpack(buf, init, Xi, pmp_i, resid, H):
        Xi.copy_(buf[:, 0].to(torch.int64))
        pmp_i.copy_(buf[:, 1])
        resid.copy_(buf[:, 2])
        if init:
            H.copy_(buf[:, 3:])
        else:
            H.mul_(buf[:, 3:])


def _fake_rank(rank, P, N, J, R):
    t = torch
    return types.SimpleNamespace(
        rank=rank, P=P, N=N, J=J, R=R, dev=t.device("cpu"), ops=_HostOps(),
        owner=t.tensor([s % P for s in range(J)], dtype=t.int32),
        X=t.full((N, J), -1, dtype=t.int64), pmp=t.ones((N, J), dtype=t.float64),
        resid=t.zeros(J, dtype=t.float64), H=t.full((J, R), 2.0, dtype=t.float64),
        lo=[1000 * rank] * N,
        U=[(t.arange(J, dtype=t.float64) + 0.1 * rank).unsqueeze(1).repeat(1, R) for _ in range(N)],
        rows_tmp=t.zeros(J, dtype=t.int64), prob_tmp=t.zeros(J, dtype=t.float64),
        urow_tmp=t.zeros((J, R), dtype=t.float64))


def _worker(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = TorchComm()
        assert comm.P == world and comm.rank == rank
        # all_gather: rank order
        got = comm.all_gather([torch.full((3, 2), float(rank))])
        assert [float(g[0, 0]) for g in got] == [float(p) for p in range(world)]
        # all_gather_v: uneven counts (one rank may contribute nothing)
        counts = [2, 0] if world == 2 else [2] * world
        x = torch.arange(10 * 3, dtype=torch.float64).reshape(10, 3) + 100 * rank
        got = comm.all_gather_v([x], counts)
        for p in range(world):
            assert got[p].shape[0] == counts[p]
            if counts[p]:
                assert float(got[p][0, 0]) == 100.0 * p
        # STS exchange: each rank finished the samples it owns
        N, J, R, i = 3, 11, 4, 1
        r = _fake_rank(rank, world, N, J, R)
        mine = (r.owner == rank).nonzero().squeeze(1)
        r.X[i][mine] = 1000 * rank + mine
        r.pmp[i][mine] = 0.5 + rank
        r.resid[mine] = 0.25 * rank
        cl = Cluster([r], comm, "sts", J, 0)
        cl._exchange_walk(i, True)          # first constant mode: H = the sampled rows
        s = torch.arange(J)
        own = s % world
        rowv = s.to(torch.float64) + 0.1 * own.to(torch.float64)
        assert torch.equal(r.X[i], 1000 * own + s)
        assert torch.equal(r.pmp[i], 0.5 + own.to(torch.float64))
        assert torch.equal(r.resid, 0.25 * own.to(torch.float64))
        assert torch.equal(r.H[:, 0], rowv) and torch.equal(r.H[:, R - 1], rowv)
        r.X[i].fill_(-1)
        r.X[i][mine] = 1000 * rank + mine
        cl._exchange_walk(i, False)         # later modes multiply the running rows
        assert torch.equal(r.H[:, 0], rowv * rowv)
        # CP-ARLS-LEV: rank-order concatenation of local draws
        quota = np.array([3, 4][:world] if world == 2 else [2] * world)
        q = int(quota[rank])
        r.rows_tmp[:q] = torch.arange(q) + 10 * rank
        r.prob_tmp[:q] = 0.1 * (rank + 1)
        r.urow_tmp[:q] = float(rank)
        rows, probs, urows = cl._gather_arls_draws(quota)
        exp = torch.cat([torch.arange(int(quota[p])) + 10 * p for p in range(world)])
        assert torch.equal(rows, exp)
        assert probs.shape[0] == int(quota.sum()) and urows.shape == (int(quota.sum()), R)
        assert float(urows[-1, 0]) == float(world - 1)
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_collectives_and_exchanges():
    mp.spawn(_worker, args=(2, _port()), nprocs=2, join=True)


def test_comm_volume_matches_reference_closed_form():
    # ref grid.py:370-376: (P-1) J (N-1) (R+2) for STS, R words for CP-ARLS-LEV
    assert comm_words_per_solve(65536, 50, 3, 8, "sts") == 7 * 65536 * 2 * 52
    assert comm_words_per_solve(65536, 50, 3, 8, "arls-lev") == 7 * 65536 * 2 * 50
    assert comm_words_per_solve(4096, 8, 3, 1, "sts") == 0


@pytest.mark.parametrize("dims,P", [((2000, 1500, 1000), 4), ((183, 24, 1140, 1717), 8),
                                    ((12092, 9184, 28818), 8), ((8, 6, 5), 4), ((3, 3, 3), 32)])
def test_grid_ownership_matches_oracle(dims, P):
    from oracle import randcp_oracle as O
    g = G.optimal_grid(dims, P)
    o = O.best_grid(dims, P)
    assert g.grid_dims == o.gdims
    for j in range(len(dims)):
        lo, hi = g.block_ranges(j)
        assert np.array_equal(lo, o.lo[j]) and np.array_equal(hi, o.hi[j])
        assert np.array_equal(g.row_order(j), o.order[j])
        rows = np.arange(dims[j])
        assert np.array_equal(g.row_owner(j, rows), o.owner(j, rows))


def test_nnz_balanced_blocks():
    """ProcessorGrid(row_weights=...) cuts every mode into contiguous blocks minimising the
    largest block's nonzeros: never worse than the reference's equal-row cuts, within one
    row's weight of the ideal share, and the default (no weights) stays the reference map."""
    dims = (3000, 2000, 1500)
    rng = np.random.default_rng(1)
    idx = np.stack([np.minimum(rng.zipf(1.2, 300000) - 1, d - 1) for d in dims], axis=1)
    idx = np.stack([rng.permutation(d)[idx[:, j]] for j, d in enumerate(dims)], axis=1)
    w = G.nnz_row_weights(dims, idx)
    for P in (2, 4, 8):
        ref = G.optimal_grid(dims, P)
        bal = G.optimal_grid(dims, P, row_weights=w)
        assert bal.grid_dims == ref.grid_dims
        for j in range(3):
            lr = [w[j][slice(*ref.block_range(j, p))].sum() for p in range(P)]
            lb = [w[j][slice(*bal.block_range(j, p))].sum() for p in range(P)]
            assert sum(lb) == sum(lr) == len(idx)
            assert max(lb) <= max(lr)
            # blocks are contiguous, cover the mode, and ownership is consistent
            rows = np.arange(dims[j])
            own = bal.row_owner(j, rows)
            for p in range(P):
                lo, hi = bal.block_range(j, p)
                assert np.all(own[lo:hi] == p)
    # weighted cuts of one sequence: the optimum of the min-max contiguous partition
    ww = np.array([5, 1, 1, 1, 1, 1, 5, 1], dtype=float)
    off = G.weighted_offsets(ww, 3)
    assert off[0] == 0 and off[-1] == ww.size
    assert max(ww[off[i]:off[i + 1]].sum() for i in range(3)) == 6.0
