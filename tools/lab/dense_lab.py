"""Dense tall-skinny kernels (Gram, leverage, update, STS leaf Grams) on a C4-sized factor
(4.8M x R) for library variants built with different tunables (GPU box).  Build the
variants in the CPU container first (`python tools/lab/dense_lab.py --build`); they go to
tools/lab/sweep/ and travel with the snapshot.  Prints one JSON line per variant: ms per
call (best of 5, CUDA events) and the difference from the first variant's results."""
import ctypes
import json
import os
import sys

LAB = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, LAB)
import sweep_spmm  # noqa: E402

VARIANTS = {   # add {"RCP_...": value} variants to compare tunables
    "base": {},
}


def run(so, n, R):
    import torch
    lib = ctypes.CDLL(so)
    lib.rcp_gram_ws_bytes.restype = ctypes.c_size_t
    lib.rcp_arls_build_ws_bytes.restype = ctypes.c_size_t
    lib.rcp_update_ws_bytes.restype = ctypes.c_size_t
    lib.rcp_sts_tree_doubles.restype = ctypes.c_size_t
    g = torch.Generator(device="cuda").manual_seed(0)
    U = torch.rand((n, R), dtype=torch.float64, device="cuda", generator=g)
    A = torch.randn((R, R), dtype=torch.float64, device="cuda", generator=g)
    Gp = (A @ A.T / R).contiguous()
    P = ctypes.c_void_p
    i64, i32 = ctypes.c_int64, ctypes.c_int
    out = {}

    def timeit(fn):
        best = 1e30
        for _ in range(5):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            b.synchronize()
            best = min(best, a.elapsed_time(b))
        return best

    G = torch.empty((R, R), dtype=torch.float64, device="cuda")
    ws = torch.empty(lib.rcp_gram_ws_bytes(i64(n), i32(R)) // 8 + 1, dtype=torch.float64,
                     device="cuda")
    out["gram_ms"] = timeit(lambda: lib.rcp_gram(P(U.data_ptr()), None, i64(n), i32(R),
                                                 P(G.data_ptr()), P(ws.data_ptr()), None))
    ref = U.T @ U
    out["gram_rel_err"] = float(((G - ref).abs().max() / ref.abs().max()).item())
    dist = torch.empty(n, dtype=torch.float64, device="cuda")
    cdf = torch.empty(n, dtype=torch.float64, device="cuda")
    mass = torch.empty(1, dtype=torch.float64, device="cuda")
    ws = torch.empty(lib.rcp_arls_build_ws_bytes(i64(n), i32(R)) // 8 + 1, dtype=torch.float64,
                     device="cuda")
    out["leverage_build_ms"] = timeit(lambda: lib.rcp_arls_build(
        P(U.data_ptr()), i64(n), i32(R), P(Gp.data_ptr()), P(dist.data_ptr()), P(cdf.data_ptr()),
        P(mass.data_ptr()), P(ws.data_ptr()), None))
    Uo = torch.empty_like(U)
    colsq = torch.empty(R, dtype=torch.float64, device="cuda")
    st = torch.zeros(4, dtype=torch.int32, device="cuda")
    ws = torch.empty(lib.rcp_update_ws_bytes(i64(n), i32(R)) // 8 + 1, dtype=torch.float64,
                     device="cuda")
    out["update_ms"] = timeit(lambda: lib.rcp_update(
        P(U.data_ptr()), i64(n), i32(R), P(Gp.data_ptr()), P(Uo.data_ptr()), P(colsq.data_ptr()),
        P(ws.data_ptr()), P(st.data_ptr()), None))
    leaf = 64
    tree = torch.empty(lib.rcp_sts_tree_doubles(i64(n), i32(leaf), i32(R)), dtype=torch.float64,
                       device="cuda")
    out["sts_build_ms"] = timeit(lambda: lib.rcp_sts_build(P(U.data_ptr()), i64(n), i32(R),
                                                           i32(leaf), P(tree.data_ptr()), None))
    torch.cuda.synchronize()
    flops = 2.0 * n * R * R
    for k in ("gram_ms", "leverage_build_ms", "update_ms"):
        out[k.replace("_ms", "_tflops")] = round(flops / (out[k] * 1e-3) / 1e12, 2)
    return out, (G.clone(), dist.clone(), Uo.clone(), tree.clone())


def main():
    if "--build" in sys.argv:
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(8) as ex:
            list(ex.map(lambda kv: sweep_spmm.build(*kv), VARIANTS.items()))
        return
    n, R = int(os.environ.get("N", 4800000)), int(os.environ.get("R", 50))
    ref = None
    for tag in VARIANTS:
        res, arrs = run(os.path.join(sweep_spmm.OUT, "lib_%s.so" % tag), n, R)
        if ref is None:
            ref = arrs
        res["max_rel_diff"] = max(float(((a - b).abs().max() / b.abs().max()).item())
                                  for a, b in zip(arrs, ref))
        print(json.dumps({"variant": tag, "n": n, "R": R, **res}), flush=True)


if __name__ == "__main__":
    main()
