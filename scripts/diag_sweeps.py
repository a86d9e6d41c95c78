import sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2405_16076_b200 as oid
from synth import ChannelFlow
gen = ChannelFlow(48, 33, 48, seed=1003)
m = gen.m
p = oid.make_params(m=m, k=200, ell=512, b_max=32, n_cap=1000, lam=-1.0, seed=0, profile=True)
eng = oid.Engine(p)
for e in range(12):
    X = torch.from_numpy(np.asfortranarray(gen.block(32*e, 32*e+32))).cuda()
    torch.cuda.synchronize(); t0 = time.time()
    eng.ingest_block(X); torch.cuda.synchronize(); t1 = time.time()
    est = eng.error_estimate(); t2 = time.time()
    c = eng.get(9)
    ns = [(c[u] > 0).sum() + 1 for u in range(3)]
    print(e, f"ingest {1e3*(t1-t0):.1f} ms  est {1e3*(t2-t1):.1f} ms  sweeps G/SJ/core {ns}  est_rel {est['est_rel']:.4f}", flush=True)
print(eng.stats())
