import sys, numpy as np, torch
sys.path.insert(0, '.')
from oracle import randcp_oracle as O
from paper_2210_05105_b200 import synth
from paper_2210_05105_b200.engine import make_local_cluster
from paper_2210_05105_b200.als import gather_factors
from paper_2210_05105_b200.linalg import init_factors
idx, vals = synth.planted_c1(seed=0)
dims=(2000,1500,1000)
P = int(sys.argv[1]) if len(sys.argv) > 1 else 4
sampler = sys.argv[2] if len(sys.argv) > 2 else "arls-lev"
st = O.AsState(dims, idx, vals, 8, sampler, 4096, seed=3, P=P)
f0,_ = init_factors(dims, 8, 3)
cl = make_local_cluster(dims, torch.as_tensor(idx, device="cuda"), torch.as_tensor(vals, device="cuda"), 8, 4096, sampler, 3, P=P, factors=f0)
for rnd in range(1, 11):
    st.rnd = rnd
    for k in range(3):
        b = st.solve(k)
        Hw = b.H * b.weights[:, None]; Gs = Hw.T @ Hw
        ev = np.linalg.eigvalsh(Gs)
        st.sigma = st.renormalize(k); st.rebuild(k)
        cl.solve(k, rnd); cl.check()
        Xg = cl.ranks[0].X.T.cpu().numpy()
        same = np.array_equal(Xg, b.X)
        got = gather_factors(cl)[k]; ref = st.full(k)
        err = np.abs(got-ref).max()/np.abs(ref).max()
        Cg = cl.ranks[0].C_host[k] if sampler=="arls-lev" and P>1 else None
        Co = st.lev[k].C if sampler=="arls-lev" else None
        print("rnd %d k %d sameX %s factor_relerr %.2e cond(Gs) %.2e lam_min %.2e C_relerr %s" % (rnd, k, same, err, ev.max()/max(ev.min(),1e-300), ev.min(), None if Cg is None else "%.2e" % (np.abs(Cg-Co).max()/np.abs(Co).max())), flush=True)
