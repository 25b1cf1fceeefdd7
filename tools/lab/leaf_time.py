"""STS tree build timings on the GPU box (leaf 64): staged tensor-core leaf Grams (default)
against the register-split (RCP_LEAF_SPLIT=1, R <= 96) and FFMA (RCP_LEAF_FFMA=1) kernels.
usage: python tools/lab/leaf_time.py [n] [R ...]"""
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


def timeit(fn, reps=3):
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
    out = {"n": n, "R": R, "leaf": 64}
    tree = ops.sts_build(U, 64)
    ref = None
    for tag, env in (("staged", {}), ("split", {"RCP_LEAF_SPLIT": "1"}), ("ffma", {"RCP_LEAF_FFMA": "1"})):
        for k in ("RCP_LEAF_SPLIT", "RCP_LEAF_FFMA"):
            os.environ.pop(k, None)
        os.environ.update(env)
        out[tag + "_build_ms"] = round(timeit(lambda: ops.sts_build(U, 64, tree)), 3)
        if ref is None:
            ref = tree.clone()
        else:
            out[tag + "_identical"] = bool(torch.equal(tree, ref))
    print(json.dumps(out), flush=True)
    del U, tree, ref
