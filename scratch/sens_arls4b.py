import sys, numpy as np
sys.path.insert(0, '.')
from oracle import randcp_oracle as O
from paper_2210_05105_b200 import synth
idx, vals = synth.planted_c1(seed=0)
sts = []
for eps in (0.0, 2**-52):
    st = O.AsState((2000,1500,1000), idx, vals*(1+eps), 8, "arls-lev", 4096, seed=3, P=4)
    for r in range(7): st.round()
    sts.append(st)
st0, st1 = sts
k = 0; rnd = 8
for i in (1, 2):
    C0, C1 = st0.lev[i].C, st1.lev[i].C
    q0 = O.lev_split(C0, 4096, 3, rnd, k, i); q1 = O.lev_split(C1, 4096, 3, rnd, k, i)
    print("mode", i, "C diff", np.abs(C0-C1).max(), "quotas", q0, q1)
    for p in range(4):
        d0 = st0.lev[i].dists[p]; d1 = st1.lev[i].dists[p]
        if q0[p] == 0: continue
        cdf0 = d0.cumsum(); cdf0 /= cdf0[-1]; cdf1 = d1.cumsum(); cdf1 /= cdf1[-1]
        u = O.stream(3, O.P_LOCAL_DRAW, rnd, k, i, p).random(q0[p])
        j0 = np.searchsorted(cdf0, u, 'right'); j1 = np.searchsorted(cdf1, u, 'right')
        dd = np.nonzero(j0 != j1)[0]
        print("  rank", p, "n flips", dd.size, [(float(u[t]), float(cdf0[j0[t]-1]) if j0[t]>0 else 0.0, float(cdf0[min(j0[t], len(cdf0)-1)])) for t in dd[:3]])
        # zero-mass check
        print("   dist zeros", int((d0 == 0).sum()), "of", d0.size, "cdf plateau at u?", int((np.abs(cdf0 - u[:,None]).min(1) == 0).sum()) if q0[p] < 5000 else -1)
