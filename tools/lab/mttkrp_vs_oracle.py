"""Sampled MTTKRP of real device batches against the oracle, per mode (GPU box): the
engine's first round on a config, every mode's batch through rcp_sampled_mttkrp and the
oracle's gather + downsampled MTTKRP.  One JSON line per mode: max relative error, gathered
nonzeros, and how many output rows differ by more than 1e-12 (diagnostic)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402
from oracle import randcp_oracle as O  # noqa: E402
from paper_2210_05105_b200.engine import make_local_cluster  # noqa: E402

cfg = os.environ.get("CFG", "c2")
dev = torch.device("cuda", 0)
c, idx, vals = bench.make_tensor(cfg, 0, dev)
cl = make_local_cluster(c["dims"], idx, vals, c["R"], c["J"], "sts", 11)
me = cl.ranks[0]
for k in range(me.N):
    cl.sample(k, 1)
    st = me.stores[k]
    out = torch.empty((st.n_rows, me.R), dtype=torch.float64, device=dev)
    stats = torch.zeros(8, dtype=torch.int64, device=dev)
    me.ops.sampled_mttkrp(st, me.X, k, me.H, me.w, out, stats)
    got = out.cpu().numpy()
    ostore = bench.oracle_store_from_device(st)
    csr = O.sampled_csr(ostore, me.X.T.cpu().numpy(), k)
    ref = O.sketched_mttkrp(csr, me.H.cpu().numpy(), me.w.cpu().numpy(), workers=os.cpu_count())
    scale = np.abs(ref).max(axis=1, keepdims=True)
    rel_rows = (np.abs(got - ref) / np.maximum(scale, 1e-300)).max(axis=1)
    print(json.dumps({"mode": k, "n_rows": int(st.n_rows), "rel_err": float(np.abs(got - ref).max() / np.abs(ref).max()),
                      "rows_gt_1e12": int((rel_rows > 1e-12).sum()), "worst_rows": [int(x) for x in np.argsort(-rel_rows)[:5]],
                      "nnz_gpu": int(stats[3]), "nnz_ref": int(csr.nnz)}), flush=True)
