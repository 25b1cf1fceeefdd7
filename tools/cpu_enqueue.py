import sys, time, torch
sys.path.insert(0, '.')
import bench
from paper_2210_05105_b200.engine import make_local_cluster
dev = torch.device("cuda", 0)
c, idx, vals = bench.make_tensor("c3", 0, dev)
for sampler in ("sts", "arls-lev"):
    cl = make_local_cluster(c["dims"], idx, vals, c["R"], c["J"], sampler, 0)
    for r in range(1, 4): cl.round(r)
    torch.cuda.synchronize()
    for r in range(4, 9):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter(); s.record(); cl.round(r, check=False); e.record(); t1 = time.perf_counter()
        e.synchronize(); t2 = time.perf_counter()
        print(sampler, "enqueue %.2f ms, gpu %.2f ms, wall %.2f ms" % ((t1-t0)*1e3, s.elapsed_time(e), (t2-t0)*1e3))
