"""R > 64 Gram and STS leaf Grams on a C4-sized factor (4.8M x R): the DMMA split-pair
kernels against the FFMA paths (RCP_GRAM_FFMA=1 / RCP_LEAF_FFMA=1), CUDA events, best of 5
(GPU box)."""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2210_05105_b200 import _lib  # noqa: E402

lib = _lib.load()
P, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
n = int(os.environ.get("N", 4800000))
for R in (75, 90):
    g = torch.Generator(device="cuda").manual_seed(R)
    U = torch.rand((n, R), dtype=torch.float64, device="cuda", generator=g)
    G = torch.empty((R, R), dtype=torch.float64, device="cuda")
    ws = torch.empty(lib.rcp_gram_ws_bytes(i64(n), i32(R)) // 8 + 1, dtype=torch.float64,
                     device="cuda")
    ref = U.T @ U
    rec = {"n": n, "R": R}
    for tag, env in (("dmma", None), ("ffma", "1")):
        if env:
            os.environ["RCP_GRAM_FFMA"] = env
        else:
            os.environ.pop("RCP_GRAM_FFMA", None)
        best = 1e30
        for _ in range(5):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            rc = lib.rcp_gram(P(U.data_ptr()), None, i64(n), i32(R), P(G.data_ptr()), P(ws.data_ptr()), None)
            assert rc == 0, (tag, rc)
            b.record()
            b.synchronize()
            best = min(best, a.elapsed_time(b))
        rec[tag + "_ms"] = round(best, 3)
        rec[tag + "_tflops"] = round(2.0 * n * R * R / (best * 1e-3) / 1e12, 2)
        rec[tag + "_rel_err"] = float(((G - ref).abs().max() / ref.abs().max()).item())
    # STS tree build (leaf Grams + levels), leaf 64
    leaf = 64
    lib.rcp_sts_tree_doubles.restype = ctypes.c_size_t
    tree = torch.empty(lib.rcp_sts_tree_doubles(i64(n), i32(leaf), i32(R)), dtype=torch.float64,
                       device="cuda")
    outs = {}
    for tag, env in (("leaf_dmma", None), ("leaf_ffma", "1")):
        if env:
            os.environ["RCP_LEAF_FFMA"] = env
        else:
            os.environ.pop("RCP_LEAF_FFMA", None)
        best = 1e30
        for _ in range(5):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            tree.fill_(float("nan"))
            rc = lib.rcp_sts_build(P(U.data_ptr()), i64(n), i32(R), i32(leaf), P(tree.data_ptr()), None)
            assert rc == 0, (tag, rc, lib.rcp_last_error())
            b.record()
            b.synchronize()
            best = min(best, a.elapsed_time(b))
        rec[tag + "_ms"] = round(best, 3)
        outs[tag] = tree.clone()
    rec["leaf_rel_diff"] = float(((outs["leaf_dmma"] - outs["leaf_ffma"]).abs().max() /
                                  outs["leaf_ffma"].abs().max()).item())
    rec["leaf_bit_identical"] = bool(torch.equal(outs["leaf_dmma"], outs["leaf_ffma"]))
    rec["tree_finite"] = bool(torch.isfinite(outs["leaf_dmma"]).all())
    print(json.dumps(rec), flush=True)
