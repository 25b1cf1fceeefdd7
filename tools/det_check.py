"""Determinism probe: two eager C3 clusters in one process, per-round sample hashes and
MTTKRP stats (compare the printed hashes across processes too)."""
import hashlib, sys, torch
sys.path.insert(0, '.')
import bench
from paper_2210_05105_b200.engine import make_local_cluster
dev = torch.device("cuda", 0)
c, idx, vals = bench.make_tensor("c3", 0, dev)
print("tensor", hashlib.sha1(idx.cpu().numpy().tobytes()).hexdigest()[:12],
      hashlib.sha1(vals.cpu().numpy().tobytes()).hexdigest()[:12])
cls = [make_local_cluster(c["dims"], idx, vals, c["R"], c["J"], "sts", 0) for _ in range(2)]
for r in range(1, 7):
    row = []
    for cl in cls:
        s0 = cl.ranks[0].stats.clone()
        cl.round(r)
        torch.cuda.synchronize()
        row.append((hashlib.sha1(cl.ranks[0].X.cpu().numpy().tobytes()).hexdigest()[:10],
                    int((cl.ranks[0].stats - s0)[3])))
    print(r, row)
