"""Factor-Gram timings on the GPU box: the staged tensor-core kernel (default) against the
register-split (RCP_GRAM_SPLIT=1, R <= 96) and FFMA (RCP_GRAM_FFMA=1) kernels of dense.cu.
Prints one JSON line per (n, R).   usage: python tools/lab/gram_time.py [n] [R ...]"""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2210_05105_b200.ops import ops_for  # noqa: E402

dev = torch.device("cuda", 0)
ops = ops_for(dev)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4_800_000
ranks = [int(x) for x in sys.argv[2:]] or [75, 90, 100, 128]


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for R in ranks:
    U = torch.randn(n, R, dtype=torch.float64, device=dev)
    out = {"n": n, "R": R}
    ref = None
    for tag, env in (("staged", {}), ("split", {"RCP_GRAM_SPLIT": "1"}), ("ffma", {"RCP_GRAM_FFMA": "1"})):
        for k in ("RCP_GRAM_SPLIT", "RCP_GRAM_FFMA"):
            os.environ.pop(k, None)
        os.environ.update(env)
        G = ops.gram(U).clone()
        out[tag + "_ms"] = round(timeit(lambda: ops.gram(U)), 3)
        if ref is None:
            ref = G
        else:
            out[tag + "_rel_diff"] = float(((G - ref).abs().max() / ref.abs().max()).item())
    out["staged_tflops"] = round(2.0 * n * R * R / (out["staged_ms"] * 1e-3) / 1e12, 2)
    out["staged_gbps"] = round(8.0 * n * R / (out["staged_ms"] * 1e-3) / 1e9, 1)
    print(json.dumps(out), flush=True)
    del U
