"""Stress the multi-rank (P > 1) engine paths on the GPU box: run_als with P virtual ranks
against the oracle on the same processor grid over random small tensors -- 3 and 4 modes,
ranks 2..8 (incl. non-powers of two: padded rank trees, empty blocks), ranks R from 3 to
100, both samplers.  One JSON line per case: first differing sample batch, worst factor
error, fits.  (STS-CP draws are P-invariant; CP-ARLS-LEV is compared on the same grid.)"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import randcp_oracle as O  # noqa: E402
import paper_2210_05105_b200 as P  # noqa: E402
from paper_2210_05105_b200 import synth  # noqa: E402

seeds = int(os.environ.get("SEEDS", "6"))
out = open(os.environ.get("OUT", "gpurun_out/stress_multirank.jsonl"), "w")
gen = np.random.default_rng(2024)
bad = 0
for case in range(seeds * 6):
    N = int(gen.choice([3, 3, 4]))
    dims = tuple(int(x) for x in gen.integers(6, 140, N))
    procs = int(gen.choice([2, 3, 4, 5, 6, 8]))
    R = int(gen.choice([3, 8, 16, 25, 50, 70, 100]))
    sampler = str(gen.choice(["sts", "sts", "arls-lev"]))
    if sampler == "arls-lev":
        # R above a mode's size makes that mode's leverage scores exact ties (all 1): the
        # rank multinomial then sees exact p = 0.5 and the reference itself changes its
        # draws under one-ulp perturbations; keep R below every mode
        R = min(R, max(2, min(dims) - 1))
    J = int(gen.choice([200, 1000, 4096]))
    nnz = int(min(np.prod(dims) // 3, gen.integers(2000, 40000)))
    seed = 100 + case
    rec = {"case": case, "dims": dims, "P": procs, "R": R, "sampler": sampler, "J": J, "nnz": nnz}
    idx, vals = synth.small_random(dims, nnz, seed=seed)
    t = P.SparseTensorCOO(dims, idx, vals)
    cfg = P.AlsConfig(rank=R, rounds=2, sampler=sampler, samples=J,
                      schedule="accumulator-stationary", procs=procs, seed=seed, fit_every=2,
                      record_samples=True, permute=False)
    t0 = time.time()
    try:
        res = P.run_als(cfg, tensor=t)
        rec["gpu"] = "ok"
    except Exception as e:
        res = None
        rec["gpu"] = "%s: %s" % (type(e).__name__, str(e)[:120])
    try:
        st, fits = O.run_as(dims, idx, vals, R, sampler, J, 2, seed=seed, P=procs)
        rec["oracle"] = "ok"
    except Exception as e:
        st = None
        rec["oracle"] = "%s: %s" % (type(e).__name__, str(e)[:120])
    if res is not None and st is not None:
        same = [bool(np.array_equal(a, b)) for a, b in zip(res.sample_log, st.sample_log)]
        rec["first_sample_diff"] = same.index(False) if False in same else None
        rec["factor_err"] = max(float(np.abs(res.factors[j] - st.full(j)).max() /
                                      max(np.abs(st.full(j)).max(), 1e-300)) for j in range(N))
        rec["fit"] = [res.final_fit, fits[-1]]
        ok = rec["first_sample_diff"] is None and rec["factor_err"] < 1e-9
    else:   # both sides must agree on raising (e.g. a degenerate walk)
        ok = (res is None) == (st is None) and rec["gpu"][:10] == rec["oracle"][:10]
    rec["ok"] = bool(ok)
    bad += 0 if ok else 1
    rec["s"] = round(time.time() - t0, 2)
    print(json.dumps(rec), flush=True)
    out.write(json.dumps(rec) + "\n")
    out.flush()
print("cases %d, not ok %d" % (seeds * 6, bad))
