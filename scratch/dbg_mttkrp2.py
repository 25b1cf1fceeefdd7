import sys, numpy as np, torch
sys.path.insert(0, '.')
from oracle import randcp_oracle as O
from paper_2210_05105_b200 import synth, _lib
from paper_2210_05105_b200.ops import ops_for
from paper_2210_05105_b200.store import build_store
dims = (40, 35, 30)
idx, vals = synth.small_random(dims, 6000, seed=2)
dev = torch.device("cuda"); ops = ops_for(dev)
R=8; gen = np.random.default_rng(4)
factors = [gen.standard_normal((d, R)) for d in dims]
k = 0
st = build_store(dims, torch.as_tensor(idx, device=dev), torch.as_tensor(vals, device=dev), k)
J = 3000
X = np.stack([gen.integers(0, d, J) for d in dims], 1).astype(np.int64); X[:, k] = -1
H = np.ones((J, R))
for i in range(3):
    if i != k: H *= factors[i][X[:, i]]
w = gen.random(J) + 0.5
out = torch.empty((dims[k], R), dtype=torch.float64, device=dev)
stats = torch.zeros(8, dtype=torch.int64, device=dev)
ops._ws.clear()
ops.sampled_mttkrp(st, torch.as_tensor(np.ascontiguousarray(X.T), device=dev), k,
                   torch.as_tensor(H, device=dev), torch.as_tensor(w, device=dev), out, stats, cap=st.capacity(J))
torch.cuda.synchronize()
ws = ops._ws["mttkrp"].cpu().numpy()
nbytes = ws.size
import ctypes
lay = np.zeros(14, dtype=np.int64)
_lib.call("rcp_mttkrp_layout", J, dims[k], R, nbytes, lay.ctypes.data)
names = ['dkey','dcnt','drep','dlo','dlen','doff','Hs','rcnt','rptr','ed','ev','S','nnz']
L = dict(zip(names, lay[:13].tolist())); cap = int(lay[13]); n_rows = dims[k]
print("cap", cap)
def arr(name, dt, n): return np.frombuffer(ws[L[name]:L[name]+np.dtype(dt).itemsize*n].tobytes(), dtype=dt)
S = int(arr('S', np.int64, 1)[0]); nnz = int(arr('nnz', np.int64, 1)[0])
print("S", S, "nnz", nnz, "stats", stats.cpu().numpy()[:5])
dkey = arr('dkey', np.int64, S); dcnt = arr('dcnt', np.int32, S); drep = arr('drep', np.int32, S)
keys = O.col_keys(X, dims, k)
u, c = np.unique(keys, return_counts=True)
print("distinct ok", np.array_equal(np.sort(dkey), u), "counts ok", np.array_equal(dcnt[np.argsort(dkey)], c))
dlo = arr('dlo', np.int64, S); dlen = arr('dlen', np.int64, S); doff = arr('doff', np.int64, S+1)
ostore = O.Store(dims, idx, vals, k)
a, b = ostore.find(dkey)
print("lookup len ok", np.array_equal(dlen, b-a), "lo ok", np.array_equal(dlo, a))
print("doff ok", np.array_equal(doff, np.concatenate([[0], np.cumsum(dlen)])))
rptr = arr('rptr', np.int64, n_rows+1)
# expected rows counts
ent_rows = np.concatenate([ostore.idx[ostore.col_order[a[i]:b[i]], k] for i in range(S)])
cnt = np.bincount(ent_rows, minlength=n_rows)
print("rptr ok", np.array_equal(rptr, np.concatenate([[0], np.cumsum(cnt)])), rptr[:5], np.concatenate([[0], np.cumsum(cnt)])[:5])
ed = arr('ed', np.int32, nnz); ev = arr('ev', np.float64, nnz)
# check each row's set of (d, v)
bad = 0
for r in range(n_rows):
    got = sorted(zip(ed[rptr[r]:rptr[r+1]].tolist(), ev[rptr[r]:rptr[r+1]].tolist()))
    exp = []
    for i in range(S):
        pos = ostore.col_order[a[i]:b[i]]
        for p in pos:
            if ostore.idx[p, k] == r: exp.append((i, ostore.vals[p]))
    if got != sorted(exp): bad += 1
print("rows with wrong entry sets", bad)
Hs = arr('Hs', np.float64, S*R).reshape(S, R)
sc = dcnt * w[drep]**2
print("Hs ok", np.abs(Hs - sc[:, None] * H[drep]).max())
exp = np.zeros((n_rows, R))
for r in range(n_rows):
    for e in range(rptr[r], rptr[r+1]):
        exp[r] += ev[e] * Hs[ed[e]]
got = out.cpu().numpy()
ref = O.sketched_mttkrp(O.sampled_csr(ostore, X, k), H, w)
print("spmm vs ws-expected", np.abs(got-exp).max(), "exp vs ref", np.abs(exp-ref).max(), "scale", np.abs(ref).max())
print(got[0], exp[0], ref[0])
# run csr_spmm path on same data
import torch as T
rp = T.as_tensor(rptr, device=dev); ci = T.as_tensor(ed.astype(np.int64), device=dev); cv = T.as_tensor(ev, device=dev)
o2 = T.empty((n_rows, R), dtype=T.float64, device=dev)
ops.csr_spmm(rp, ci, cv, T.as_tensor(Hs, device=dev), None, o2)
print("csr_spmm vs exp", np.abs(o2.cpu().numpy()-exp).max())
