"""Pin the CPU oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py).  CPU only."""

import hashlib

import numpy as np
import pytest

from conftest import golden
from oracle import randcp_oracle as O
from paper_2210_05105_b200 import synth


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_rng_keys_and_draws():
    g = golden("rng.npz")
    for row, key, draws in zip(g["ctx"], g["keys"], g["draws"]):
        seed, purpose, n = int(row[0]), int(row[1]), int(row[2])
        ctx = [int(v) for v in row[3:3 + n]]
        assert np.array_equal(O.stream_key(seed, purpose, *ctx), key)
        assert np.array_equal(O.stream(seed, purpose, *ctx).random(13), draws)
    s, p, *ctx = [int(v) for v in g["perm_ctx"]]
    for J in (1, 2, 7, 1000, 4096):
        assert np.array_equal(O.stream(s, p, *ctx).permutation(J), g["perm_%d" % J])


def _blocks(g, factors, N):
    return [[factors[j][g.lo[j, p]:g.hi[j, p]] for p in range(g.P)] for j in range(N)]


@pytest.mark.parametrize("gd", [(1, 1, 1), (2, 2, 1), (4, 2, 1)])
def test_samplers_match_reference(gd):
    g0 = golden("samplers.npz")
    dims = tuple(int(d) for d in g0["dims"])
    factors = [g0["U%d" % j] for j in range(3)]
    g = O.Grid(dims, gd)
    blocks = _blocks(g, factors, 3)
    grams = [O.gram_blocks(b) for b in blocks]
    trees = [O.tree_build(blocks[j], g.lo[j], order=g.order[j]) for j in range(3)]
    tag = "x".join(map(str, gd))
    for k in range(3):
        cp = O.sym_pinv(O.hadamard_chain(grams, skip=k))
        b = O.tree_sample(trees, k, 512, cp, grams, blocks, seed=17, rnd=2)
        assert np.array_equal(b.X, g0["sts_%s_k%d_X" % (tag, k)])
        assert np.array_equal(b.prob, g0["sts_%s_k%d_prob" % (tag, k)])
        assert np.array_equal(b.H, g0["sts_%s_k%d_H" % (tag, k)])
        states = [O.lev_build(blocks[j], g.lo[j]) for j in range(3)]
        a = O.lev_sample(states, k, 512, factors, seed=19, rnd=3)
        assert np.array_equal(a.X, g0["arls_%s_k%d_X" % (tag, k)])
        assert np.array_equal(a.prob, g0["arls_%s_k%d_prob" % (tag, k)])
        assert np.array_equal(O.weights_for(a.prob, 512), g0["arls_%s_k%d_w" % (tag, k)])


def test_steered_walk_matches_reference():
    g0 = golden("walk.npz")
    factors = [g0["U%d" % j] for j in range(3)]
    dims = tuple(U.shape[0] for U in factors)
    g = O.Grid(dims, (1, 1, 1))
    blocks = _blocks(g, factors, 3)
    grams = [O.gram_blocks(b) for b in blocks]
    trees = [O.tree_build(blocks[j], g.lo[j], order=g.order[j], leaf=2) for j in range(3)]
    k = int(g0["k"])
    cp = O.sym_pinv(O.hadamard_chain(grams, skip=k))
    b = O.tree_sample(trees, k, g0["override"].shape[0], cp, grams, blocks, seed=0,
                      uniforms=g0["override"])
    assert np.array_equal(b.X, g0["X"])
    assert np.array_equal(b.prob, g0["prob"])


def test_mttkrp_matches_reference():
    g0 = golden("mttkrp.npz")
    st_idx, st_vals = g0["idx"], g0["vals"]
    for k in range(3):
        st = O.Store((9, 8, 7), st_idx, st_vals, k)
        csr = O.sampled_csr(st, g0["X%d" % k], k)
        assert np.array_equal(csr.row_ptr, g0["rp%d" % k])
        assert np.array_equal(csr.col_idx, g0["ci%d" % k])
        assert np.array_equal(csr.vals, g0["cv%d" % k])
        out = O.sketched_mttkrp(csr, g0["H%d" % k], g0["w%d" % k])
        assert np.array_equal(out, g0["out%d" % k])
        for workers in (2, 3):
            assert np.array_equal(O.sketched_mttkrp(csr, g0["H%d" % k], g0["w%d" % k], workers), out)


@pytest.mark.parametrize("sampler,P", [("sts", 1), ("sts", 4), ("arls-lev", 1),
                                       ("arls-lev", 2), ("arls-lev", 4)])
def test_c1_als_matches_reference(sampler, P):
    g0 = golden("als_c1.npz")
    idx, vals = synth.planted_c1(seed=0)
    assert sha(idx) == str(g0["idx_sha"]) and sha(vals) == str(g0["vals_sha"])
    st, fits = O.run_as((2000, 1500, 1000), idx, vals, 8, sampler, 4096, 10, seed=3, P=P)
    tag = "%s_p%d" % (sampler.replace("-", ""), P)
    hashes = [sha(X) for X in st.sample_log]
    assert hashes == [str(h) for h in g0[tag + "_hash"]]
    for j in range(3):
        assert np.array_equal(st.full(j), g0[tag + "_U%d" % j])
    assert np.array_equal(st.sigma, g0[tag + "_sigma"])
    assert np.allclose(fits, g0[tag + "_fits"], rtol=0, atol=1e-12)
