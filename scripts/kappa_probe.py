"""kappa(S_J) per estimate along the C1, C3r and C3 streams (K1F), to size a kappa gate for A9Q."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from __graft_entry__ import build
build()
import paper_2405_16076_b200 as oid
from synth import c1_matrix, ChannelFlow, C3, C3R
dev = torch.device("cuda", 0)
A = c1_matrix(); s = np.linalg.svd(A, compute_uv=False); lam = float(np.sum(s[20:] ** 2) / 20)
p = oid.make_params(m=4096, k=20, ell=48, b_max=16, n_cap=512, lam=lam, split=(16, 16, 16), seed=0, k1_mode=4)
eng = oid.Engine(p); Ad = torch.from_numpy(np.asfortranarray(A)).to(dev)
ks = []
for j in range(0, 512, 16):
    eng.ingest_block(Ad[:, j:j + 16]); ks.append(eng.error_estimate()["kappa"])
print("C1 kappa", " ".join(f"{k:.1e}" for k in ks)); eng.close()
for name, gen, n in (("C3r", ChannelFlow(48, 33, 48, seed=C3R.data_seed), 1000), ("C3", ChannelFlow(192, 129, 192, seed=C3.data_seed), 640)):
    p = oid.make_params(m=gen.m, k=200, ell=512, b_max=32, n_cap=1024, lam=-1.0, seed=0, k1_mode=4)
    eng = oid.Engine(p); ks = []
    for j in range(0, n, 32):
        X = gen.block_torch(j, min(n, j + 32), dev).T
        eng.ingest_block(X); ks.append(eng.error_estimate()["kappa"]); del X
    print(name, "kappa", " ".join(f"{k:.1e}" for k in ks)); eng.close()
