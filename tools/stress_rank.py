"""Stress the R > 64 engine paths on the GPU box: run_als (CUDA) against the oracle over
many seeds, ranks and both samplers; one JSON line per case with the first failing solve,
the device status flags of any error, and the sample/factor agreement.  Design probe for
the round-1 driver failure (test_rank_above_64[sts-70] non-finite factors)."""
import json
import os
import sys
import time
import traceback

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import randcp_oracle as O  # noqa: E402
import paper_2210_05105_b200 as P  # noqa: E402
from paper_2210_05105_b200 import synth  # noqa: E402

seeds = int(os.environ.get("SEEDS", "8"))
cases = [("sts", 70), ("arls-lev", 70), ("sts", 128), ("sts", 75), ("sts", 100), ("arls-lev", 100)]
dims = (120, 100, 90)
out = open(os.environ.get("OUT", "gpurun_out/stress_rank.jsonl"), "w")
for seed in range(5, 5 + seeds):
    for sampler, R in cases:
        rec = {"seed": seed, "sampler": sampler, "R": R}
        idx, vals = synth.small_random(dims, 30000, seed=seed)
        t = P.SparseTensorCOO(dims, idx, vals)
        cfg = P.AlsConfig(rank=R, rounds=2, sampler=sampler, samples=512,
                          schedule="accumulator-stationary", seed=seed, fit_every=2,
                          record_samples=True, permute=False)
        t0 = time.time()
        try:
            res = P.run_als(cfg, tensor=t)
            rec["gpu"] = "ok"
        except Exception as e:
            res = None
            rec["gpu"] = "%s: %s" % (type(e).__name__, e)
        try:
            st, fits = O.run_as(dims, idx, vals, R, sampler, 512, 2, seed=seed)
            rec["oracle"] = "ok"
        except Exception as e:
            st = None
            rec["oracle"] = "%s: %s" % (type(e).__name__, e)
        if res is not None and st is not None:
            same = [bool(np.array_equal(a, b)) for a, b in zip(res.sample_log, st.sample_log)]
            rec["first_sample_diff"] = same.index(False) if False in same else None
            rec["factor_err"] = max(float(np.abs(res.factors[j] - st.full(j)).max() /
                                          max(np.abs(st.full(j)).max(), 1e-300)) for j in range(3))
            rec["fit"] = [res.final_fit, fits[-1]]
        rec["s"] = round(time.time() - t0, 2)
        print(json.dumps(rec), flush=True)
        out.write(json.dumps(rec) + "\n")
        out.flush()
