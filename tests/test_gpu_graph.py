"""Rounds replayed from a CUDA graph (draw keys and SHUFFLE permutations in device memory)
draw the same samples and produce the same factors as eager rounds."""

import numpy as np
import pytest

from conftest import cuda_ok
from paper_2210_05105_b200 import synth

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]


@pytest.mark.parametrize("dims,sampler", [((60, 50, 40), "sts"), ((30, 8, 25, 20), "sts"),
                                          ((60, 50, 40), "arls-lev"),
                                          ((30, 8, 25, 20), "arls-lev")])
def test_graph_rounds_match_eager(dims, sampler):
    import torch
    from paper_2210_05105_b200.engine import make_local_cluster
    idx, vals = synth.small_random(dims, 4000, seed=6)
    dev = torch.device("cuda", 0)
    ti, tv = torch.as_tensor(idx, device=dev), torch.as_tensor(vals, device=dev)
    a = make_local_cluster(dims, ti, tv, 7, 512, sampler, 3)
    b = make_local_cluster(dims, ti, tv, 7, 512, sampler, 3)
    assert b.graph_ok()
    a.round(1)
    b.round(1)
    for rnd in range(2, 6):
        a.round(rnd)
        b.round_graph(rnd)
        torch.cuda.synchronize()
        b.check("graph round %d" % rnd)
        assert torch.equal(a.ranks[0].X, b.ranks[0].X), rnd
    assert b.graph_kernels > 10 * len(dims)
    for j in range(len(dims)):
        ua, ub = a.ranks[0].U[j], b.ranks[0].U[j]
        # the transpose's atomic order perturbs a round by ~1 ulp; four rounds amplify it
        assert float((ua - ub).abs().max() / ua.abs().max()) < 1e-10
    np.testing.assert_allclose(a.ranks[0].sigma.cpu().numpy(), b.ranks[0].sigma.cpu().numpy(),
                               rtol=1e-10)
    assert abs(a.fit() - b.fit()) < 1e-10


@pytest.mark.parametrize("dims,grid", [((60, 50, 40), (2, 1, 1)), ((60, 50, 40), (2, 2, 1)),
                                       ((30, 8, 25, 20), (1, 1, 2, 2)),
                                       ((30, 8, 25, 20), (2, 1, 1, 2))])
def test_graph_rounds_match_eager_multi_rank(dims, grid):
    """STS-CP at P > 1 (virtual ranks): the rank-level walk reads its key from device
    memory, the rank-tree indices are uploaded once, the walk exchange is a device-side
    sum -- the replayed round equals the eager one."""
    import torch
    from paper_2210_05105_b200.engine import make_local_cluster
    idx, vals = synth.small_random(dims, 4000, seed=6)
    dev = torch.device("cuda", 0)
    ti, tv = torch.as_tensor(idx, device=dev), torch.as_tensor(vals, device=dev)
    a = make_local_cluster(dims, ti, tv, 7, 512, "sts", 3, grid_dims=grid)
    b = make_local_cluster(dims, ti, tv, 7, 512, "sts", 3, grid_dims=grid)
    assert b.P > 1 and b.graph_ok()
    a.round(1)
    b.round(1)
    for rnd in range(2, 5):
        a.round(rnd)
        b.round_graph(rnd)
        torch.cuda.synchronize()
        b.check("graph round %d" % rnd)
        for ra, rb in zip(a.ranks, b.ranks):
            assert torch.equal(ra.X, rb.X), rnd
    for ra, rb in zip(a.ranks, b.ranks):
        for j in range(len(dims)):
            ua, ub = ra.U[j], rb.U[j]
            if ua.numel():
                assert float((ua - ub).abs().max() / ua.abs().max()) < 1e-10
    assert abs(a.fit() - b.fit()) < 1e-10


def test_graph_not_offered_for_host_dependent_rounds():
    import torch
    from paper_2210_05105_b200.engine import make_local_cluster
    dims = (20, 15, 10)
    idx, vals = synth.small_random(dims, 500, seed=1)
    dev = torch.device("cuda", 0)
    ti, tv = torch.as_tensor(idx, device=dev), torch.as_tensor(vals, device=dev)
    # CP-ARLS-LEV at P > 1 splits J over the rank masses on the host
    multi = make_local_cluster(dims, ti, tv, 4, 64, "arls-lev", 1, grid_dims=(2, 1, 1))
    assert not multi.graph_ok()
    with pytest.raises(RuntimeError):
        multi.round_graph(1)
