import sys, torch
sys.path.insert(0, '.')
import bench
from paper_2210_05105_b200.engine import make_local_cluster
dev = torch.device("cuda", 0)
c, idx, vals = bench.make_tensor("c3", 0, dev)
a = make_local_cluster(c["dims"], idx, vals, c["R"], c["J"], "sts", 0)
b = make_local_cluster(c["dims"], idx, vals, c["R"], c["J"], "sts", 0)
a.round(1); b.round(1)
for r in range(2, 7):
    s0a = a.ranks[0].stats.clone(); s0b = b.ranks[0].stats.clone()
    a.round(r); b.round_graph(r); torch.cuda.synchronize()
    print(r, torch.equal(a.ranks[0].X, b.ranks[0].X), (a.ranks[0].stats - s0a).tolist()[:5], (b.ranks[0].stats - s0b).tolist()[:5],
          float((a.ranks[0].U[0]-b.ranks[0].U[0]).abs().max()))
