"""Per-level phase trace of the STS walk (GPU box): builds the library with
-DRCP_WALK_TRACE, runs C3 rounds and prints, per tree level, the longest time any warp
spent in each phase of one run (record load, h row, child mass, partition + push)."""
import os
import subprocess
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools", "lab"))
import sweep_spmm  # noqa: E402

so = sweep_spmm.build("trace", {"RCP_WALK_TRACE": 1, "RCP_WALK_PROF": 1})
from paper_2210_05105_b200 import _lib  # noqa: E402
_lib.load(so)
import bench  # noqa: E402
from paper_2210_05105_b200.engine import make_local_cluster  # noqa: E402

dev = torch.device("cuda", 0)
c, idx, vals = bench.make_tensor(os.environ.get("CFG", "c3"), 0, dev)
cl = make_local_cluster(c["dims"], idx, vals, c["R"], c["J"], "sts", 0)
me = cl.ranks[0]
for r in range(1, 4):
    cl.round(r)
ops = me.ops
owalk = ops.sts_walk
lib = _lib.lib()
KMAX = 30


def hook(tree, U, leaf, *a, **kw):
    owalk(tree, U, leaf, *a, **kw)
    torch.cuda.synchronize()
    J = a[3]
    total = lib.rcp_sts_walk_ws_bytes(int(J), U.shape[0], int(leaf), U.shape[1])
    o = total - 256 - 64 * (KMAX + 2)
    ws = kw.get("ws")
    if ws is None:
        ws = ops._ws["sts_walk"]
    t = ws[o:o + 64 * (KMAX + 2)].view(torch.int64).cpu().tolist()
    print("walk n=%d" % U.shape[0])
    for l in range(KMAX):
        if t[2 * l] == 0:
            break
        nxt = t[2 * (l + 1)] if t[2 * (l + 1)] else t[2 * (KMAX + 1)]
        ph = [x / 1e3 for x in t[4 * (KMAX + 2) + 4 * l: 4 * (KMAX + 2) + 4 * l + 4]]
        print("  level %2d runs %6d  %6.1f us  max phase us: record %.1f  h %.1f  mass %.1f  "
              "partition %.1f" % (l, t[2 * l + 1], (nxt - t[2 * l]) / 1e3, *ph))


ops.sts_walk = hook
cl.round(4)
