"""Engine edge cases on the GPU against the CPU oracle: 4-mode tensors, rank exceeding a
mode dimension, processor grids with empty blocks, several rank counts, empty batches,
unsupported configurations, determinism.  Mirrors the reference's edge-case suite
(ref tests/test_edge_cases.py, tests/test_als.py)."""

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


@pytest.fixture(scope="module")
def P():
    import paper_2210_05105_b200 as pkg
    return pkg


def run_both(P, dims, nnz, R, sampler, J, rounds, procs=1, gdims=None, seed=5):
    idx, vals = synth.small_random(dims, nnz, seed=seed)
    t = P.SparseTensorCOO(dims, idx, vals)
    cfg = P.AlsConfig(rank=R, rounds=rounds, sampler=sampler, samples=J,
                      schedule="accumulator-stationary", procs=procs, grid_dims=gdims, seed=seed,
                      fit_every=rounds, record_samples=True, permute=False)
    res = P.run_als(cfg, tensor=t)
    st, fits = O.run_as(dims, idx, vals, R, sampler, J, rounds, seed=seed, P=procs,
                        gdims=gdims)
    return res, st, fits


@pytest.mark.parametrize("sampler", ["sts", "arls-lev"])
@pytest.mark.parametrize("procs", [1, 2])
def test_four_mode_als_matches_oracle(P, sampler, procs):
    res, st, fits = run_both(P, (12, 9, 7, 5), 900, 4, sampler, 300, 3, procs=procs)
    for a, b in zip(res.sample_log, st.sample_log):
        assert np.array_equal(a, b)
    for j in range(4):
        assert rel_err(res.factors[j], st.full(j)) < 1e-9
    assert abs(res.final_fit - fits[-1]) < 1e-6


def horizon(dims, nnz, R, sampler, J, rounds, procs, seed=5):
    """First solve whose samples the reference algorithm itself changes under one-ulp
    perturbations of its floating-point inputs (numerical ties, e.g. leverage scores that
    are all exactly 1 when R exceeds a mode's size, whose rank masses then feed numpy's
    binomial an exact p = 0.5); len(log) when it never does.  Probes: tensor values and
    initial factors moved by one ulp, and the per-rank leverage masses of CP-ARLS-LEV's
    multinomial moved by one ulp."""
    idx, vals = synth.small_random(dims, nnz, seed=seed)
    base, _ = O.run_as(dims, idx, vals, R, sampler, J, rounds, seed=seed, P=procs, fit=False)
    h = len(base.sample_log)
    probes = [(vals * (1 + e), 1.0, None) for e in (2.0 ** -52, -2.0 ** -52)]
    probes += [(vals, 1 + e, None) for e in (2.0 ** -52, -2.0 ** -52)]
    probes += [(vals, 1.0, d) for d in (np.inf, -np.inf)]
    split = O.lev_split
    try:
        for v, scale, direction in probes:
            if direction is not None:
                O.lev_split = (lambda C, *a, _d=direction:
                               split(np.where(np.asarray(C) > 0, np.nextafter(C, _d), C), *a))
            st, _ = O.run_as(dims, idx, v, R, sampler, J, rounds, seed=seed, P=procs, fit=False,
                             init_scale=scale)
            O.lev_split = split
            d = [i for i, (a, b) in enumerate(zip(st.sample_log, base.sample_log))
                 if not np.array_equal(a, b)]
            if d:
                h = min(h, d[0])
    finally:
        O.lev_split = split
    return h


@pytest.mark.parametrize("procs", [1, 4])
@pytest.mark.parametrize("sampler", ["sts", "arls-lev"])
def test_rank_exceeding_mode_dimension(P, sampler, procs):
    # overcomplete factor on the short mode => rank-deficient Gram chain (Jacobi pinv path)
    res, st, fits = run_both(P, (20, 3, 15), 250, 6, sampler, 256, 5, procs=procs)
    assert np.isfinite(res.final_fit)
    assert res.factors[1].shape == (3, 6)
    h = horizon((20, 3, 15), 250, 6, sampler, 256, 5, procs)
    for a, b in list(zip(res.sample_log, st.sample_log))[:h]:
        assert np.array_equal(a, b)
    if h == len(st.sample_log):
        for j in range(3):
            assert rel_err(res.factors[j], st.full(j)) < 1e-9


def test_grid_dimension_exceeding_mode_dimension(P):
    # explicit grid with P_1 > I_1 leaves some row blocks empty
    res, st, fits = run_both(P, (6, 3, 5), 60, 2, "sts", 64, 4, gdims=(1, 4, 1))
    assert np.isfinite(res.final_fit)
    for a, b in zip(res.sample_log, st.sample_log):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("procs", [3, 8])
def test_sts_rank_count_invariance(P, procs):
    """STS draws do not depend on the processor grid (ref tests/test_samplers.py:223-233)."""
    r1, _, _ = run_both(P, (16, 12, 10), 800, 3, "sts", 200, 2, procs=1)
    rp, _, _ = run_both(P, (16, 12, 10), 800, 3, "sts", 200, 2, procs=procs)
    for a, b in zip(r1.sample_log, rp.sample_log):
        assert np.array_equal(a, b)


def test_determinism_same_seed_same_samples(P):
    a, _, _ = run_both(P, (15, 11, 9), 600, 3, "sts", 256, 3)
    b, _, _ = run_both(P, (15, 11, 9), 600, 3, "sts", 256, 3)
    for x, y in zip(a.sample_log, b.sample_log):
        assert np.array_equal(x, y)
    for j in range(3):
        assert rel_err(a.factors[j], b.factors[j]) < 1e-12


def test_unsupported_configurations_raise(P):
    idx, vals = synth.small_random((5, 4, 3), 20, seed=1)
    t = P.SparseTensorCOO((5, 4, 3), idx, vals)
    with pytest.raises(P.ScheduleError):
        P.run_als(P.AlsConfig(rank=2, rounds=1, sampler="exact",
                              schedule="accumulator-stationary"), tensor=t)
    with pytest.raises(P.ScheduleError):
        P.run_als(P.AlsConfig(rank=2, rounds=1, sampler="sts", samples=8,
                              schedule="tensor-stationary"), tensor=t)
    with pytest.raises(ValueError):
        P.AlsConfig(rank=0, rounds=1).validate()


def test_empty_batch_paths(P):
    idx, vals = synth.small_random((5, 4, 3), 20, seed=10)
    t = P.SparseTensorCOO((5, 4, 3), idx, vals)
    m = P.matricize(t, 0)
    csr = P.gather_sampled_nonzeros_to_csr(m, np.full((0, 3), -1, dtype=np.int64), 0)
    assert csr.nnz == 0 and csr.n_cols == 0
    out = P.downsampled_mttkrp(csr, np.ones((0, 2)), np.ones(0))
    assert np.array_equal(out, np.zeros((5, 2)))
    with pytest.raises(ValueError):
        P.downsampled_mttkrp(csr, np.ones((3, 2)), np.ones(0))


def test_matricization_row_bounds_enforced(P):
    with pytest.raises(ValueError):
        P.Matricization((4, 2, 2), np.array([[0, 0, 0], [3, 0, 0]]), np.ones(2), 0,
                        row_lo=0, row_hi=2)


def test_all_ones_full_cover_reproduces_exact(P):
    """Every column sampled once with p = 1/n_cols: downsampled == exact MTTKRP
    (ref tests/test_mttkrp.py:118-146)."""
    idx, vals = synth.small_random((4, 3, 3), 25, seed=10)
    t = P.SparseTensorCOO((4, 3, 3), idx, vals)
    gen = np.random.default_rng(11)
    factors = [gen.standard_normal((d, 2)) for d in t.dims]
    m = P.matricize(t, 0)
    X = np.full((9, 3), -1, dtype=np.int64)
    s = 0
    for c in range(3):
        for b in range(3):
            X[s, 1], X[s, 2] = b, c
            s += 1
    H = factors[1][X[:, 1]] * factors[2][X[:, 2]]
    got = P.downsampled_mttkrp(P.gather_sampled_nonzeros_to_csr(m, X, 0), H, np.ones(9))
    ref = P.mttkrp_exact(m, factors)
    assert np.abs(got - ref).max() < 1e-12


@pytest.mark.parametrize("graph", [False, True])
def test_host_step_api_matches_device_round(P, graph):
    """AlsSession.step_host (pinned host factors in, overlapped transfers, factors and sigma
    out; eager or replayed from a CUDA graph) computes the same rounds as the
    device-resident engine."""
    import torch
    from paper_2210_05105_b200.als import AlsSession
    from paper_2210_05105_b200.engine import make_local_cluster
    dims = (300, 200, 150)
    idx, vals = synth.small_random(dims, 20000, seed=3)
    dev = torch.device("cuda")
    ti, tv = torch.as_tensor(idx, device=dev), torch.as_tensor(vals, device=dev)
    a = make_local_cluster(dims, ti, tv, 8, 1024, "sts", 7)
    b = make_local_cluster(dims, ti, tv, 8, 1024, "sts", 7)
    a.round(1)
    b.round(1)
    sess = AlsSession(a)
    host_in, host_out = sess.pinned_factors(), sess.pinned_factors()
    for rnd in (2, 3, 4):
        sess.step_host(host_in, host_out, rnd, graph=graph)
        for j in range(3):      # step_host re-uploads the host factors, then rebuilds
            b.ranks[0].U[j].copy_(host_in[j].to(dev))
            b.rebuild(j)
        b.round(rnd)
        assert torch.equal(a.ranks[0].X, b.ranks[0].X), rnd
        for j in range(3):
            got = host_out[j].numpy()
            ref = b.ranks[0].U[j].cpu().numpy()
            assert rel_err(got, ref) < 1e-12
        assert rel_err(sess.sigma.numpy(), b.ranks[0].sigma.cpu().numpy()) < 1e-12
        for j in range(3):      # the next step starts from this step's output
            host_in[j].copy_(host_out[j])


@pytest.mark.parametrize("sampler,R", [("sts", 70), ("arls-lev", 70), ("sts", 128)])
def test_rank_above_64(P, sampler, R):
    """R > 64: tensor-core tiles padded past 64 columns (leaf masses, leverage, update
    GEMM), two column pairs per lane in the SpMM, register GJ with 8x4 tiles; R = 128 is
    the largest supported rank (fewer walker warps fit in shared memory)."""
    dims = (120, 100, 90)
    res, st, fits = run_both(P, dims, 30000, R, sampler, 512, 2)
    h = horizon(dims, 30000, R, sampler, 512, 2, 1)
    for a, b in list(zip(res.sample_log, st.sample_log))[:h]:
        assert np.array_equal(a, b)
    if h == len(st.sample_log):
        for j in range(3):
            assert rel_err(res.factors[j], st.full(j)) < 1e-9


def test_tensor_path_trials_and_result_files(P, tmp_path):
    """run_trials from a FROSTT file (loaded and permuted once, ref als.py:141-237) and the
    `decompose --out` files (ref cli.py:93-104): factors in the file's index order."""
    from paper_2210_05105_b200.tensorio import read_matrix, write_results
    dims = (30, 20, 25)
    idx, vals = synth.small_random(dims, 1500, seed=2)
    path = tmp_path / "t.tns"
    with open(path, "w") as fh:
        for (a, b, c), v in zip(idx + 1, vals):
            fh.write("%d %d %d %.17g\n" % (a, b, c, v))
    cfg = P.AlsConfig(rank=4, rounds=2, tensor_path=str(path), sampler="sts", samples=200,
                      schedule="accumulator-stationary", seed=5, fit_every=1)
    res = P.run_trials(cfg, 2)
    t = P.load_frostt(str(path))
    tp, mp = P.permute_modes(t, 5)
    ref = P.run_als(cfg, tensor=tp, perms=mp)
    for j in range(3):
        assert rel_err(res[0].factors[j], ref.factors[j]) < 1e-12
        assert res[0].factors[j].shape == (t.dims[j], 4)
    assert np.isfinite(res[1].final_fit)
    write_results(res, str(tmp_path / "out"))
    for tr in range(2):
        d = tmp_path / "out" / ("trial%d" % tr)
        for j in range(3):
            assert np.array_equal(read_matrix(str(d / ("factor_mode%d.bin" % j))), res[tr].factors[j])
        assert read_matrix(str(d / "sigma.bin")).shape == (4, 1)
        assert "final_fit" in (d / "summary.txt").read_text()
