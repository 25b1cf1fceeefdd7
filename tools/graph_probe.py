"""Timing probe (not a product path): one STS round captured in a CUDA graph and replayed,
against eager launches of the same round.  The replay reuses the captured round's random
streams, so only its time is meaningful."""
import sys, time, torch
sys.path.insert(0, '.')
import bench
from paper_2210_05105_b200.engine import make_local_cluster
dev = torch.device("cuda", 0)
c, idx, vals = bench.make_tensor("c3", 0, dev)
cl = make_local_cluster(c["dims"], idx, vals, c["R"], c["J"], "sts", 0)
for r in range(1, 4): cl.round(r)
torch.cuda.synchronize()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
g = torch.cuda.CUDAGraph()
try:
    with torch.cuda.graph(g, stream=s):
        cl.round(4, check=False)
except Exception as ex:
    print("capture failed:", repr(ex)[:300]); sys.exit(0)
torch.cuda.synchronize()
for rep in range(2):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); cl.round(5 + rep, check=False); b.record(); b.synchronize()
    print("eager %.3f ms" % a.elapsed_time(b))
for rep in range(5):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); g.replay(); b.record(); b.synchronize()
    print("graph %.3f ms" % a.elapsed_time(b))
