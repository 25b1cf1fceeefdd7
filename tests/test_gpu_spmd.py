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


# ---------------------------------------------------------------- two processes
def _two_proc_worker(rank, world, port, sampler, out):
    import torch
    import torch.distributed as dist
    from paper_2210_05105_b200.dist import make_spmd_cluster
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    # gloo: two ranks share the one GPU of a test box (NCCL needs a GPU per rank); the
    # collectives stage through the host, no kernel waits on another process
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dims = (50, 40, 30)
        idx, vals = synth.small_random(dims, 4000, seed=3)
        dev = torch.device("cuda", 0)
        ti, tv = torch.as_tensor(idx, device=dev), torch.as_tensor(vals, device=dev)
        cl = make_spmd_cluster(dims, ti, tv, 6, 400, sampler, 2)
        comm = cl.comm
        words = []
        for rnd in (1, 2):
            w0 = comm.words
            cl.round(rnd)
            words.append(comm.words - w0)
        me = cl.ranks[0]
        np.savez(out % rank, X=me.X.cpu().numpy(), sigma=me.sigma.cpu().numpy(),
                 words=np.array(words), lo=np.array(me.lo), fit=np.array([cl.fit()]),
                 **{"U%d" % j: me.U[j].cpu().numpy() for j in range(3)})
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("sampler", ["sts", "arls-lev"])
def test_two_process_round_matches_local_p2(sampler, tmp_path):
    """Two SPMD processes (real RankState, real Cluster.round, TorchComm) reproduce the
    single-process P=2 cluster (LocalComm): identical samples, factors to 1e-12.  The STS
    exchange volume is the fixed J (R+3) words per constant mode per process (the
    reference's closed form counts (P-1) J (N-1) (R+2) received words, ref
    grid.py:370-376; here every process contributes its owned rows to one sum
    all-reduce, and the residual rides along)."""
    import socket
    import torch
    import torch.multiprocessing as mp
    from paper_2210_05105_b200.engine import make_local_cluster
    from paper_2210_05105_b200.grid import as_gather_words_total_per_solve
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = str(tmp_path / ("r%d_" + sampler + ".npz"))
    mp.start_processes(_two_proc_worker, args=(2, port, sampler, out), nprocs=2,
                       start_method="spawn")
    dims = (50, 40, 30)
    idx, vals = synth.small_random(dims, 4000, seed=3)
    dev = torch.device("cuda", 0)
    ti, tv = torch.as_tensor(idx, device=dev), torch.as_tensor(vals, device=dev)
    a = make_local_cluster(dims, ti, tv, 6, 400, sampler, 2, P=2)
    for rnd in (1, 2):
        a.round(rnd)
    J, R, N = 400, 6, 3
    for p in range(2):
        got = np.load(out % p)
        ref = a.ranks[p]
        assert np.array_equal(got["X"], ref.X.cpu().numpy())
        for j in range(N):
            u = ref.U[j].cpu().numpy()
            assert np.abs(got["U%d" % j] - u).max() <= 1e-12 * max(np.abs(u).max(), 1e-300)
        assert np.allclose(got["sigma"], ref.sigma.cpu().numpy(), rtol=1e-12, atol=0)
        assert abs(float(got["fit"][0]) - a.fit()) < 1e-10
        if sampler == "sts":
            # per round: N solves x (N-1) constant modes x J (R+3) words
            assert list(got["words"]) == [N * (N - 1) * J * (R + 3)] * 2
            closed = as_gather_words_total_per_solve(J, R, N, 2, "sts")
            assert closed == (2 - 1) * J * (N - 1) * (R + 2)
