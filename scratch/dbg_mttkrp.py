import sys, numpy as np, torch
sys.path.insert(0, '.')
from oracle import randcp_oracle as O
from paper_2210_05105_b200 import synth
from paper_2210_05105_b200.ops import ops_for
from paper_2210_05105_b200.store import build_store
dims = (40, 35, 30)
idx, vals = synth.small_random(dims, 6000, seed=2)
dev = torch.device("cuda"); ops = ops_for(dev)
for R in (8, 37):
  for dup in (False, True):
    gen = np.random.default_rng(4)
    factors = [gen.standard_normal((d, R)) for d in dims]
    k = 0
    st = build_store(dims, torch.as_tensor(idx, device=dev), torch.as_tensor(vals, device=dev), k)
    J = 3000
    X = np.stack([gen.integers(0, d, J) for d in dims], 1).astype(np.int64)
    X[:, k] = -1
    if dup: X[100:400] = X[0]
    H = np.ones((J, R))
    for i in range(3):
        if i != k: H *= factors[i][X[:, i]]
    w = gen.random(J) + 0.5
    if dup: w[100:400] = w[0]
    csr = O.sampled_csr(O.Store(dims, idx, vals, k), X, k)
    ref = O.sketched_mttkrp(csr, H, w)
    out = torch.empty((dims[k], R), dtype=torch.float64, device=dev)
    stats = torch.zeros(8, dtype=torch.int64, device=dev)
    ops.sampled_mttkrp(st, torch.as_tensor(np.ascontiguousarray(X.T), device=dev), k,
                       torch.as_tensor(H, device=dev), torch.as_tensor(w, device=dev), out, stats, cap=st.capacity(J))
    ops.status.check()
    got = out.cpu().numpy()
    err = np.abs(got-ref)
    print("R", R, "dup", dup, "maxerr", err.max(), "scale", np.abs(ref).max(), "rows bad", np.unique(np.nonzero(err > 1e-9*np.abs(ref).max())[0])[:10], "stats", stats.cpu().numpy()[:5], "csr.nnz", csr.nnz)
    bad = np.nonzero(err.max(1) > 1e-9*np.abs(ref).max())[0]
    if bad.size:
        r = bad[0]; print(" row", r, got[r,:4], ref[r,:4], "ratio", (got[r]/ref[r])[:4])
