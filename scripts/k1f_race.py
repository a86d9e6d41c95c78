import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from __graft_entry__ import build
build()
import paper_2405_16076_b200 as oid
dev = torch.device("cuda", 0)
m, b, ell, calls = int(sys.argv[1]), 32, 512, int(sys.argv[2])
g = torch.Generator(device="cpu").manual_seed(0)
Xh = torch.randn(b, m, generator=g, dtype=torch.float64) * torch.logspace(-3, 3, b, dtype=torch.float64)[:, None]
X = Xh.to(dev).T
p = oid.make_params(m=m, k=8, ell=ell, b_max=64, n_cap=4096, lam=-1.0, seed=5, dtype="f64", k1_mode=oid.K1_TC_INT8)
eng = oid.Engine(p); eng.ingest_sketch(X); torch.cuda.synchronize()
ex = eng.partials(0)[: (ell + 1) * b].clone(); eng.close()
p = oid.make_params(m=m, k=8, ell=ell, b_max=64, n_cap=4096, lam=-1.0, seed=5, dtype="f64", k1_mode=oid.K1_TC_FAST)
eng = oid.Engine(p)
outs = []
for c in range(calls):
    eng.ingest_sketch(X)
    outs.append(eng.partials(0)[: (ell + 1) * b].clone())
torch.cuda.synchronize()
Y = ex[:ell * b].view(b, ell).T
colmax = X.abs().amax(0)
nbad = 0
for c, f in enumerate(outs):
    d = ((Y - f[:ell * b].view(b, ell).T).abs() / (m ** 0.5 * colmax[None, :])).cpu().numpy()
    if d.max() > 1e-6:
        nbad += 1
        bad = np.argwhere(d > 1e-6)
        print(f"call {c}: max {d.max():.2e} cols {sorted(set(bad[:, 1].tolist()))} nrows {len(set(bad[:, 0].tolist()))}")
print(f"{nbad} bad of {calls}; counters {eng.get(15)[-8:].tolist()}")
