"""The torch.distributed (NCCL) SPMD engine at world size 1 runs the same solves as the
single-process engine: same samples, same factors to rounding (the multi-GPU plumbing on
one GPU)."""

import os

import numpy as np
import pytest

from conftest import cuda_ok
from paper_2210_05105_b200 import synth

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]


@pytest.fixture(scope="module")
def nccl_world1():
    import torch
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29531")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("sampler", ["sts", "arls-lev"])
def test_spmd_world1_matches_local(nccl_world1, sampler):
    import torch
    from paper_2210_05105_b200.dist import make_spmd_cluster
    from paper_2210_05105_b200.engine import make_local_cluster
    dims = (50, 40, 30)
    idx, vals = synth.small_random(dims, 4000, seed=3)
    dev = torch.device("cuda", 0)
    ti, tv = torch.as_tensor(idx, device=dev), torch.as_tensor(vals, device=dev)
    a = make_local_cluster(dims, ti, tv, 6, 400, sampler, 2)
    b = make_spmd_cluster(dims, ti, tv, 6, 400, sampler, 2)
    for rnd in (1, 2, 3):
        a.round(rnd)
        b.round(rnd)
        assert torch.equal(a.ranks[0].X, b.ranks[0].X), rnd
    for j in range(3):   # the transpose's row order is atomic-order dependent: ~1 ulp
        ua, ub = a.ranks[0].U[j], b.ranks[0].U[j]
        assert float((ua - ub).abs().max() / ua.abs().max()) < 1e-12
    assert abs(a.fit() - b.fit()) < 1e-10
