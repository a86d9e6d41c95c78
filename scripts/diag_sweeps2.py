import sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2405_16076_b200 as oid
from synth import ChannelFlow
gen = ChannelFlow(48, 33, 48, seed=1003)
m = gen.m
p = oid.make_params(m=m, k=200, ell=512, b_max=32, n_cap=1000, lam=-1.0, seed=0, profile=True)
eng = oid.Engine(p)
for e in range(14):
    X = torch.from_numpy(np.asfortranarray(gen.block(32*e, 32*e+32))).cuda()
    eng.ingest_block(X)
    est = eng.error_estimate()
    c = eng.get(9)
    if e in (0, 1, 6, 13):
        print(e, "G ", c[0][:30].tolist())
        print(e, "SJ", c[1][:16].tolist())
        print(e, "core", c[2][:20].tolist())
        mu = np.sort(eng.get(6))[::-1]
        print(e, "mu", mu[[0, 10, 100, 200, 300, 400, 511]], "lam", eng.scalars()["lam"], flush=True)
