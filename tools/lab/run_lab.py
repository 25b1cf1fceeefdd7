"""Build and run the lab probes on the GPU box.
    LABMODE=walk|gsync|gather|probe python tools/lab/run_lab.py"""
import ctypes
import glob
import json
import os
import subprocess
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
LAB = os.path.join(ROOT, "tools", "lab")


def build():
    so = os.path.join(LAB, "libspmm_lab.so")
    srcs = [s for s in sorted(glob.glob(os.path.join(ROOT, "paper_2210_05105_b200", "csrc", "*.cu")))
            if not s.endswith(("mttkrp.cu", "sts_walk.cu"))] + \
        [os.path.join(LAB, "spmm_lab.cu"), os.path.join(LAB, "walk_lab.cu")]
    cmd = ["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
           "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", "-shared",
           "-o", so] + srcs
    if not os.path.exists(so) or any(os.path.getmtime(s) > os.path.getmtime(so) for s in srcs):
        subprocess.check_call(cmd)
    return so


def main():
    lab = ctypes.CDLL(build())
    import bench
    from paper_2210_05105_b200 import _lib
    from paper_2210_05105_b200.engine import make_local_cluster
    dev = torch.device("cuda", 0)
    _lib.load()
    cfg = os.environ.get("CFG", "c3")
    sampler = os.environ.get("SAMPLER", "sts")
    if os.environ.get("LABMODE") in ("gather", "gsync"):
        cfg = "c1"
    c, idx, vals = bench.make_tensor(cfg, 0, dev)
    cl = make_local_cluster(c["dims"], idx, vals, c["R"], c["J"], sampler, 0)
    me = cl.ranks[0]
    for rnd in range(1, 4):
        cl.round(rnd)
    res = []

    if os.environ.get("LABMODE") == "gsync":
        sink = torch.zeros(4, dtype=torch.int32, device=dev)
        for iters in (1, 101):
            ms = ctypes.c_float(0)
            rc = lab.lab_gsync_probe(iters, ctypes.c_void_p(sink.data_ptr()), ctypes.byref(ms))
            print(json.dumps({"probe": "grid.sync", "iters": iters, "ms": ms.value, "rc": rc}))
        return
    if os.environ.get("LABMODE") == "gather":
        for rows in (13690, 65536, 1 << 17):
            tab = torch.randn(rows * 64, dtype=torch.float64, device=dev)
            n = 1 << 26
            sink = torch.zeros(8 + n // 2, dtype=torch.float64, device=dev)
            sink[8:].view(torch.int32).copy_(torch.randint(0, rows, (n,), dtype=torch.int32,
                                                           device=dev))
            ms = ctypes.c_float(0)
            lab.lab_gather_probe(ctypes.c_void_p(tab.data_ptr()), ctypes.c_int64(rows),
                                 ctypes.c_int64(n), ctypes.c_void_p(sink.data_ptr()),
                                 ctypes.byref(ms))
            print(json.dumps({"probe": "gather400", "table_MB": rows * 512 / 1e6, "gathers": n,
                              "ms": ms.value, "useful_GBps": n * 400 / ms.value / 1e6,
                              "sector_GBps": n * 416 / ms.value / 1e6}), flush=True)
        return
    if os.environ.get("LABMODE") == "probe":
        out = torch.zeros(28818 * 64 + 64, dtype=torch.float64, device=dev)
        for mode, name in ((0, "red_2x_f64"), (1, "red_1x_f64"), (2, "gather_v2")):
            ms = ctypes.c_float(0)
            nf = 1 << 20
            lab.lab_red_probe(ctypes.c_void_p(out.data_ptr()), ctypes.c_int64(28818), 50,
                              ctypes.c_int64(nf), mode, ctypes.byref(ms))
            print(json.dumps({"probe": name, "rows": nf, "ms": ms.value,
                              "GB/s": nf * 400 / ms.value / 1e6}), flush=True)
        return
    if os.environ.get("LABMODE") == "walk":
        ops = me.ops
        owalk = ops.sts_walk

        def walk_hook(tree, U, leaf, *a, **kw):
            s = torch.cuda.Event(enable_timing=True)
            e = torch.cuda.Event(enable_timing=True)
            s.record()
            owalk(tree, U, leaf, *a, **kw)
            e.record()
            torch.cuda.synchronize()
            J = a[3]
            buf = (ctypes.c_ulonglong * 128)()
            lab.lab_walk_prof(ctypes.c_void_p(ops._ws["sts_walk"].data_ptr()), ctypes.c_int64(J),
                              ctypes.c_int64(U.shape[0]), int(leaf), U.shape[1], buf)
            t = list(buf)
            lv = []
            for l in range(30):
                if t[2 * l] == 0:
                    break
                lv.append((t[2 * l + 1], t[2 * l]))
            end = t[2 * 31]
            fb = 2 * 32
            per = [{"runs": r, "us": round(((lv[i + 1][1] if i + 1 < len(lv) else end) - t0) / 1e3, 1),
                    "first_warp_done_us": round(((~t[fb + 2 * i + 1]) & (2 ** 64 - 1) - t0) / 1e3, 1),
                    "last_warp_done_us": round((t[fb + 2 * i] - t0) / 1e3, 1)}
                   for i, (r, t0) in enumerate(lv)]
            row = {"walk_n": U.shape[0], "leaf": int(leaf), "walk_ms": s.elapsed_time(e),
                   "kernel_us": round((end - lv[0][1]) / 1e3, 1), "levels": per}
            res.append(row)
            print(json.dumps(row), flush=True)
        ops.sts_walk = walk_hook
    else:
        raise SystemExit("LABMODE must be one of walk, gsync, gather, probe")
    cl.round(4)
    torch.cuda.synchronize()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "lab_%s_%s.json" % (cfg, sampler)), "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
