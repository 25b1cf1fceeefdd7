"""Parameter sweep of the segmented SpMM (GPU box): builds the library with
-DRCP_SPMM_CHUNK/-DRCP_SPMM_U/-DRCP_SPMM_BLOCKS_PER_SM variants into tools/lab/sweep/ and
times the sampled-MTTKRP calls of C3 rounds with each (one subprocess per variant)."""
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
OUT = os.path.join(ROOT, "tools", "lab", "sweep")


def build(tag, defs):
    os.makedirs(OUT, exist_ok=True)
    so = os.path.join(OUT, "lib_%s.so" % tag)
    if os.environ.get("SWEEP_PREBUILT") == "1" and os.path.exists(so):
        return so   # built in the CPU container (tools/lab/sweep/ travels with the snapshot)
    srcs = sorted(glob.glob(os.path.join(ROOT, "paper_2210_05105_b200", "csrc", "*.cu")))
    cmd = ["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
           "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", "-shared", "-o", so]
    cmd += ["-D%s=%d" % kv for kv in defs.items()] + srcs
    subprocess.check_call(cmd)
    return so


CHILD = r"""
import sys, json, torch
sys.path.insert(0, %r)
from paper_2210_05105_b200 import _lib
_lib.load(%r)
import bench
from paper_2210_05105_b200.engine import make_local_cluster
dev = torch.device("cuda", 0)
c, idx, vals = bench.make_tensor("c3", 0, dev)
cl = make_local_cluster(c["dims"], idx, vals, c["R"], c["J"], "sts", 0)
me = cl.ranks[0]
orig = me.mttkrp
ev = []
def timed(k):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); out = orig(k); b.record(); ev.append((a, b)); return out
for r in range(1, 4):
    cl.round(r)
me.mttkrp = timed
for r in range(4, 9):
    cl.round(r)
torch.cuda.synchronize()
me.mttkrp = orig
rt = []
for r in range(9, 14):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); cl.round(r, check=False); b.record(); b.synchronize(); rt.append(a.elapsed_time(b))
print(json.dumps({"mttkrp_ms": sum(a.elapsed_time(b) for a, b in ev) / len(ev),
                  "round_ms": sorted(rt)[len(rt) // 2]}))
"""


def main():
    variants = {}
    build_only = "--build-only" in sys.argv
    if build_only:
        sys.argv.remove("--build-only")
    if len(sys.argv) > 1 and sys.argv[1] == "buckets":
        for nb in (128, 256, 512, 1024, 2048):
            variants["b%d" % nb] = {"RCP_BUCKET_MAX": nb}
    elif len(sys.argv) > 1 and sys.argv[1] == "warps":
        for w, mb in ((16, 2), (12, 2), (8, 3), (8, 2)):
            variants["w%d_mb%d" % (w, mb)] = {"RCP_WALK_WARPS": w, "RCP_WALK_MIN_BLOCKS": mb}
    elif len(sys.argv) > 1 and sys.argv[1] == "prof":
        variants["prof0"] = {"RCP_WALK_PROF": 0}
        variants["prof1"] = {"RCP_WALK_PROF": 1}
    elif len(sys.argv) > 1 and sys.argv[1] == "walk":
        for u in (4, 8, 10):
            for mb in (1, 2):
                variants["u%d_mb%d" % (u, mb)] = {"RCP_WALK_UNROLL": u, "RCP_WALK_MIN_BLOCKS": mb}
    elif len(sys.argv) > 1 and sys.argv[1] == "transpose":
        variants["two_pass"] = {"RCP_BUCKET_MIN_ROWS": 4096}
        variants["single_pass"] = {"RCP_BUCKET_MIN_ROWS": 1 << 20}
    else:
        for chunk in (128, 256, 512):
            for u in (2, 4):
                for bps in (4, 8):
                    variants["c%d_u%d_b%d" % (chunk, u, bps)] = {
                        "RCP_SPMM_CHUNK": chunk, "RCP_SPMM_U": u, "RCP_SPMM_BLOCKS_PER_SM": bps}
    res = {}
    if build_only:   # CPU container: build every variant in parallel, run later on the box
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(8) as ex:
            list(ex.map(lambda kv: build(*kv), variants.items()))
        return
    for tag, defs in variants.items():
        so = build(tag, defs)
        out = subprocess.run([sys.executable, "-c", CHILD % (ROOT, so)], capture_output=True,
                             text=True, cwd=ROOT)
        line = [l for l in out.stdout.splitlines() if l.startswith("{")]
        res[tag] = json.loads(line[-1]) if line else out.stderr[-300:]
        print(tag, res[tag], flush=True)
    name = "sweep_%s.json" % (sys.argv[1] if len(sys.argv) > 1 else "spmm")
    with open(os.path.join(ROOT, "gpurun_out", name), "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
