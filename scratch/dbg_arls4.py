import sys, numpy as np, torch, hashlib
sys.path.insert(0, '.')
from oracle import randcp_oracle as O
import paper_2210_05105_b200 as P
from paper_2210_05105_b200 import synth
sys.path.insert(0,'tests')
from conftest import golden
g0 = golden("als_c1.npz")
idx, vals = synth.planted_c1(seed=0)
t = P.SparseTensorCOO((2000, 1500, 1000), idx, vals)
cfg = P.AlsConfig(rank=8, rounds=9, sampler="arls-lev", samples=4096, schedule="accumulator-stationary", procs=4, seed=3, fit_every=1, record_samples=True, permute=False)
res = P.run_als(cfg, tensor=t)
st = O.AsState((2000,1500,1000), idx, vals, 8, "arls-lev", 4096, seed=3, P=4)
for r in range(8): st.round()
# compare state before round 9
print("grid", res.grid_dims)
X = res.sample_log[24]; 
st.rnd = 9
b = st.draw(0)
d = np.nonzero((X != b.X).any(1))[0]
print("n diff samples", d.size, d[:10])
print(X[d[:5]], b.X[d[:5]])
# inspect cdf boundary distance for mode-1 or 2 draws
k = 0
for i in (1, 2):
    lev = st.lev[i]
    W = lev.C.sum()
    qo = O.lev_split(lev.C, 4096, 3, 9, k, i)
    print("mode", i, "C oracle", lev.C)
    mind = 1.0
    for p, dist in enumerate(lev.dists):
        q = int(qo[p])
        if q == 0: continue
        cdf = dist.cumsum(); cdf /= cdf[-1]
        u = O.stream(3, O.P_LOCAL_DRAW, 9, k, i, p).random(q)
        j = np.searchsorted(cdf, u, side="right")
        lo = np.where(j > 0, cdf[np.maximum(j-1,0)], 0.0)
        hi = cdf[np.minimum(j, len(cdf)-1)]
        dd = np.minimum(np.abs(u - lo), np.abs(hi - u))
        mind = min(mind, dd.min())
        print("  rank", p, "quota", q, "min dist to boundary", dd.min())
    print(" quotas", qo)
# GPU-side C at round 9 start: rerun 8 rounds with the engine directly
from paper_2210_05105_b200.engine import make_local_cluster
from paper_2210_05105_b200.linalg import init_factors
f0,_ = init_factors((2000,1500,1000), 8, 3)
cl = make_local_cluster((2000,1500,1000), torch.as_tensor(idx, device="cuda"), torch.as_tensor(vals, device="cuda"), 8, 4096, "arls-lev", 3, P=4, factors=f0)
for r in range(1, 9): cl.round(r)
for i in (1,2):
    print("gpu C mode", i, cl.ranks[0].C_host[i], "quota", np.random.Generator(np.random.Philox(np.random.SeedSequence(3, spawn_key=(2,9,0,i)))).multinomial(4096, cl.ranks[0].C_host[i]/cl.ranks[0].C_host[i].sum()))
    for p, r in enumerate(cl.ranks):
        d_gpu = r.dist[i].cpu().numpy(); d_or = st.lev[i].dists[p]
        print("  rank", p, "dist maxrel", np.abs(d_gpu-d_or).max()/max(np.abs(d_or).max(),1e-300))
