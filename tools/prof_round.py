"""One C3 round under cudaProfilerStart/Stop (for ncu --profile-from-start off)."""
import sys, os, torch
sys.path.insert(0, '.')
from paper_2210_05105_b200 import _lib
if os.environ.get("OLDLIB"): _lib.load(os.environ["OLDLIB"])
import bench
from paper_2210_05105_b200.engine import make_local_cluster
dev = torch.device("cuda", 0)
c, idx, vals = bench.make_tensor(os.environ.get("CFG", "c3"), 0, dev)
P = int(os.environ.get("P", "1"))   # virtual ranks (LocalComm): every rank's kernels, one after another
cl = make_local_cluster(c["dims"], idx, vals, c["R"], c["J"], os.environ.get("SAMPLER", "sts"), 0,
                        P=P, balance="nnz" if P > 1 else "rows")
for rnd in range(1, 4): cl.round(rnd)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
cl.round(4)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok")
