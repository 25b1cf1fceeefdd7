"""Exact fit and exact MTTKRP on the GPU (row F1, fit.cu) against the CPU oracle
(ref compute_fit linalg.py:130-151, mttkrp_exact mttkrp.py:65-108)."""

import numpy as np
import pytest

from conftest import cuda_ok
from oracle import randcp_oracle as O
from paper_2210_05105_b200 import synth

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]


def rel_err(a, b):
    scale = max(np.abs(b).max(), 1e-300)
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / scale)


def random_model(dims, R, seed):
    rs = np.random.default_rng(seed)
    facs = [O.unit_columns(rs.standard_normal((d, R)))[0] for d in dims]
    sigma = rs.uniform(0.5, 2.0, R)
    return facs, sigma


@pytest.mark.parametrize("dims,nnz,R", [((40, 30, 20), 3000, 7), ((9, 5, 7, 6), 900, 33),
                                        ((300, 2, 150), 5000, 70)])
def test_exact_mttkrp_matches_oracle(dims, nnz, R):
    import paper_2210_05105_b200 as P
    idx, vals = synth.small_random(dims, nnz, seed=11)
    facs, _ = random_model(dims, R, 2)
    for j in range(len(dims)):
        mat = P.Matricization(dims, idx, vals, j)
        got = P.mttkrp_exact(mat, facs)
        ref = O.exact_mttkrp(O.Store(dims, idx, vals, j), facs)
        assert rel_err(got, ref) < 1e-12, j


def test_exact_mttkrp_block_offsets():
    """A row block of mode j with factor row windows (offsets) of the other modes."""
    import paper_2210_05105_b200 as P
    dims = (50, 40, 30)
    idx, vals = synth.small_random(dims, 2000, seed=4)
    facs, _ = random_model(dims, 6, 3)
    sel = (idx[:, 0] >= 10) & (idx[:, 0] < 30)
    mat = P.Matricization(dims, idx[sel], vals[sel], 0, row_lo=10, row_hi=30)
    lo1 = int(idx[sel, 1].min())
    lo2 = int(idx[sel, 2].min())
    got = P.mttkrp_exact(mat, [None, facs[1][lo1:], facs[2][lo2:]], offsets=[0, lo1, lo2])
    ref = O.exact_mttkrp(O.Store(dims, idx, vals, 0), facs)[10:30]
    assert rel_err(got, ref) < 1e-12


@pytest.mark.parametrize("dims,nnz,R", [((40, 30, 20), 3000, 7), ((9, 5, 7, 6), 900, 12)])
def test_compute_fit_matches_oracle(dims, nnz, R):
    import paper_2210_05105_b200 as P
    idx, vals = synth.small_random(dims, nnz, seed=7)
    facs, sigma = random_model(dims, R, 5)
    t = P.SparseTensorCOO(dims, idx, vals)
    got = P.compute_fit(t, facs, sigma)
    last = len(dims) - 1
    ref = O.fit_value(float(np.sum(vals * vals)), facs, sigma, O.Store(dims, idx, vals, last))
    assert abs(got - ref) < 1e-12
    mat = P.Matricization(dims, idx, vals, last)
    assert P.compute_fit(t, facs, sigma, mode_mat=mat) == got   # cached store, same kernels
    with pytest.raises(ValueError):
        P.compute_fit(t, facs, sigma, mode_mat=P.Matricization(dims, idx, vals, 0))
    with pytest.raises(ValueError):
        P.compute_fit(P.SparseTensorCOO(dims, idx, np.zeros_like(vals)), facs, sigma)


@pytest.mark.parametrize("procs", [1, 3])
def test_cluster_fit_matches_oracle(procs):
    """Device fit of the engine state after two rounds (virtual ranks at P = 3) equals the
    oracle fit of the same factors, and is bit-reproducible."""
    import torch
    from paper_2210_05105_b200.als import gather_factors
    from paper_2210_05105_b200.engine import make_local_cluster
    dims = (30, 25, 20)
    idx, vals = synth.small_random(dims, 2500, seed=9)
    dev = torch.device("cuda", 0)
    cl = make_local_cluster(dims, torch.as_tensor(idx, device=dev), torch.as_tensor(vals, device=dev),
                            5, 256, "sts", 1, grid_dims=None if procs == 1 else (3, 1, 1))
    for rnd in (1, 2):
        cl.round(rnd)
    f1 = cl.fit()
    f2 = cl.fit()
    assert f1 == f2
    facs = gather_factors(cl)
    sigma = cl.ranks[0].sigma.cpu().numpy()
    ref = O.fit_value(float(np.sum(vals * vals)), facs, sigma, O.Store(dims, idx, vals, 2))
    assert abs(f1 - ref) < 1e-10
