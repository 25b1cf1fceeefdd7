"""Generate golden vectors by running the REFERENCE implementation.

Runs only in the build container, where `/root/reference/pkg/src` (the
reference `randcp` package, pure numpy) is importable; the resulting
`.npz` fixtures are committed and travel with the repo.  Nothing on the GPU
box reads `/root/reference`.

    python tests/golden/make_golden.py

Fixtures (all under tests/golden/):
  rng.npz       -- Philox keys, first draws, uint32 draws, permutations for
                   several (seed, purpose, context) streams (ref rng.py:26-32)
  samplers.npz  -- STS / CP-ARLS-LEV batches (X, prob, per_mode_prob, H) on
                   small factors at several processor grids (ref samplers.py)
  walk.npz      -- uniform_override steered STS walks (ref samplers.py:379-419)
  mttkrp.npz    -- gathered CSR + downsampled MTTKRP on a small tensor
                   (ref mttkrp.py:131-189)
  als_c1.npz    -- C1 runs (10 rounds, R=8, J=4096): per-solve sample hashes
                   + heads, fits per round, final factors and sigma, for
                   STS P=1/4 and CP-ARLS-LEV P=1/2/4 (ref als.py:141-218)
"""

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import randcp  # noqa: E402  (the reference)
from randcp import grid as gridmod  # noqa: E402
from randcp import rng as rrng  # noqa: E402
from randcp.als import AlsConfig, run_als  # noqa: E402
from randcp.linalg import FactorBlocks, gram, hadamard_gram_chain, pseudo_inverse  # noqa: E402
from randcp.matricization import matricize  # noqa: E402
from randcp.mttkrp import downsampled_mttkrp, gather_sampled_nonzeros_to_csr  # noqa: E402
from randcp.samplers import (arls_lev_build, arls_lev_sample, sample_weights,  # noqa: E402
                             sts_build, sts_sample)
from randcp.tensor import SparseTensorCOO  # noqa: E402

from paper_2210_05105_b200 import synth  # noqa: E402  (pure numpy part)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def make_rng():
    out = {}
    cases = [(0, 5, (1, 0, 1)), (0, 5, (3, 2, 0)), (7, 3, (1, 0, 1, 0)), (7, 3, (2, 1, 2, 3)),
             (123456789, 4, (5, 1, 0)), (2 ** 40 + 3, 2, (1, 2, 1)), (0, 0, (0, 2)),
             (42, 6, ()), (42, 6, (2 ** 33 + 5,)), (0, 1, (0,))]
    keys, draws, u32, ctxs = [], [], [], []
    for seed, purpose, ctx in cases:
        g = rrng.stream(seed, purpose, *ctx)
        keys.append(np.array(g.bit_generator.state["state"]["key"], dtype=np.uint64))
        draws.append(g.random(13))
        g2 = rrng.stream(seed, purpose, *ctx)
        u32.append(g2.integers(0, 2 ** 32, size=9, dtype=np.uint64))  # not used for parity
        ctxs.append(np.array([seed & (2 ** 64 - 1), purpose, len(ctx)] + list(ctx) +
                             [0] * (4 - len(ctx)), dtype=np.uint64))
    out["ctx"] = np.stack(ctxs)
    out["keys"] = np.stack(keys)
    out["draws"] = np.stack(draws)
    for J in (1, 2, 7, 1000, 4096):
        out["perm_%d" % J] = rrng.stream(11, rrng.SHUFFLE, 3, 1, 2).permutation(J)
    out["perm_ctx"] = np.array([11, rrng.SHUFFLE, 3, 1, 2], dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "rng.npz"), **out)


def blocks_for(factors, g):
    return [FactorBlocks.from_global(U, g, j) for j, U in enumerate(factors)]


def make_samplers():
    out = {}
    gen = np.random.default_rng(16)
    dims = (40, 30, 25)
    R = 4
    factors = [gen.standard_normal((d, R)) for d in dims]
    out["dims"] = np.array(dims)
    for j, U in enumerate(factors):
        out["U%d" % j] = U
    for gd in ((1, 1, 1), (2, 2, 1), (4, 2, 1)):
        g = gridmod.ProcessorGrid(dims, gd)
        blocks = blocks_for(factors, g)
        grams = [gram(b) for b in blocks]
        trees = [sts_build(b, grid=g) for b in blocks]
        tag = "x".join(map(str, gd))
        for k in range(3):
            cp = pseudo_inverse(hadamard_gram_chain(grams, skip=k))
            b = sts_sample(trees, k, 512, cp, grams, blocks, seed=17, round_id=2, grid=g)
            for nm in ("X", "prob", "per_mode_prob", "H", "residual"):
                out["sts_%s_k%d_%s" % (tag, k, nm)] = getattr(b, nm)
            states = [arls_lev_build(bb) for bb in blocks]
            full = factors
            a = arls_lev_sample(states, k, 512, full, seed=19, round_id=3)
            for nm in ("X", "prob", "per_mode_prob", "H"):
                out["arls_%s_k%d_%s" % (tag, k, nm)] = getattr(a, nm)
            out["arls_%s_k%d_w" % (tag, k)] = sample_weights(a)
    np.savez_compressed(os.path.join(HERE, "samplers.npz"), **out)


def make_walk():
    """Steered walks: uniform_override sweeps (ref acceptance criterion 3 idea)."""
    out = {}
    gen = np.random.default_rng(5)
    dims = (6, 5, 7)
    R = 3
    factors = [gen.standard_normal((d, R)) for d in dims]
    for j, U in enumerate(factors):
        out["U%d" % j] = U
    g = gridmod.ProcessorGrid(dims, (1, 1, 1))
    blocks = blocks_for(factors, g)
    grams = [gram(b) for b in blocks]
    trees = [sts_build(b, grid=g, leaf_block_size=2) for b in blocks]
    k = 1
    cp = pseudo_inverse(hadamard_gram_chain(grams, skip=k))
    J = 2000
    ov = np.zeros((J, 3))
    ov[:, 0] = (np.arange(J) + 0.5) / J
    ov[:, 2] = gen.random(J)
    b = sts_sample(trees, k, J, cp, grams, blocks, seed=0, uniform_override=ov)
    out["override"] = ov
    out["X"] = b.X
    out["prob"] = b.prob
    out["k"] = np.array(k)
    np.savez_compressed(os.path.join(HERE, "walk.npz"), **out)


def make_mttkrp():
    out = {}
    idx, vals = synth.small_random((9, 8, 7), 250, seed=13)
    t = SparseTensorCOO((9, 8, 7), idx, vals)
    out["idx"], out["vals"] = idx, vals
    gen = np.random.default_rng(12)
    factors = [gen.standard_normal((d, 3)) for d in t.dims]
    for k in range(3):
        m = matricize(t, k)
        J = 40
        X = np.stack([gen.integers(0, d, J) for d in t.dims], 1).astype(np.int64)
        X[:, k] = -1
        X[5] = X[3]          # duplicated samples are kept with multiplicity
        X[9] = X[3]
        H = np.ones((J, 3))
        for i in range(3):
            if i != k:
                H *= factors[i][X[:, i]]
        w = gen.random(J) + 0.5
        w[5] = w[3]
        w[9] = w[3]
        csr = gather_sampled_nonzeros_to_csr(m, X, k)
        res = downsampled_mttkrp(csr, H, w)
        out["X%d" % k], out["H%d" % k], out["w%d" % k] = X, H, w
        out["rp%d" % k], out["ci%d" % k], out["cv%d" % k] = csr.row_ptr, csr.col_idx, csr.vals
        out["out%d" % k] = res
    np.savez_compressed(os.path.join(HERE, "mttkrp.npz"), **out)


def make_als_c1():
    out = {}
    idx, vals = synth.planted_c1(seed=0)
    dims = (2000, 1500, 1000)
    t = SparseTensorCOO(dims, idx, vals)
    out["idx_sha"] = np.array(sha(idx))
    out["vals_sha"] = np.array(sha(vals))
    runs = [("sts", 1), ("sts", 4), ("arls-lev", 1), ("arls-lev", 2), ("arls-lev", 4)]
    for sampler, P in runs:
        cfg = AlsConfig(rank=8, rounds=10, sampler=sampler, samples=4096,
                        schedule="accumulator-stationary", procs=P, seed=3,
                        fit_every=1, record_samples=True, permute=False)
        res = run_als(cfg, tensor=t)
        tag = "%s_p%d" % (sampler.replace("-", ""), P)
        out[tag + "_hash"] = np.array([sha(X) for X in res.sample_log])
        out[tag + "_head"] = np.stack([X[:16] for X in res.sample_log])
        out[tag + "_fits"] = np.array([f for _, f in res.fit_history])
        out[tag + "_sigma"] = res.sigma
        for j in range(3):
            out[tag + "_U%d" % j] = res.factors[j]
        print(tag, "final fit", res.final_fit, "grid", res.grid_dims, flush=True)
    np.savez_compressed(os.path.join(HERE, "als_c1.npz"), **out)


if __name__ == "__main__":
    print("reference randcp", randcp.__version__, "numpy", np.__version__)
    make_rng()
    make_samplers()
    make_walk()
    make_mttkrp()
    make_als_c1()
    print("done")
