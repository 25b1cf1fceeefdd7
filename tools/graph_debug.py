"""Timing probe for graph-replayed rounds: host time of each round_graph call (input
staging for the next round included) against the GPU time of the round."""
import sys, time, torch
sys.path.insert(0, '.')
import bench
from paper_2210_05105_b200.engine import make_local_cluster
dev = torch.device("cuda", 0)
c, idx, vals = bench.make_tensor("c3", 0, dev)
for sampler in ("arls-lev", "sts"):
    cl = make_local_cluster(c["dims"], idx, vals, c["R"], c["J"], sampler, 0)
    cl.round(1)
    for r in range(2, 9):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter(); a.record()
        cl.round_graph(r)
        b.record(); t1 = time.perf_counter(); b.synchronize()
        print("%s round %d: call %.2f ms, gpu %.2f ms" % (sampler, r, (t1 - t0) * 1e3, a.elapsed_time(b)))
