import sys, numpy as np, hashlib
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from oracle import randcp_oracle as O
from paper_2210_05105_b200 import synth
from conftest import golden
g0 = golden("als_c1.npz")
idx, vals = synth.planted_c1(seed=0)
for P in (2, 4):
  for eps in (0.0, 2**-52, -2**-52, 2**-50):
    v = vals * (1 + eps)
    st, fits = O.run_as((2000,1500,1000), idx, v, 8, "arls-lev", 4096, 10, seed=3, P=P, fit=False)
    hs = [hashlib.sha256(np.ascontiguousarray(X).tobytes()).hexdigest() for X in st.sample_log]
    ref = [str(h) for h in g0["arlslev_p%d_hash" % P]]
    mism = [i for i,(a,b) in enumerate(zip(hs, ref)) if a != b]
    print("P", P, "eps", eps, "first mismatch", mism[:1])
