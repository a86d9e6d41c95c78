import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from __graft_entry__ import build
build()
import paper_2405_16076_b200 as oid
dev = torch.device("cuda", 0)
m, b, ell = int(sys.argv[1]) if len(sys.argv) > 1 else 300000, 32, 512
g = torch.Generator(device="cpu").manual_seed(0)
Xh = torch.randn(b, m, generator=g, dtype=torch.float64) * torch.logspace(-3, 3, b, dtype=torch.float64)[:, None]
X = Xh.to(dev).T
def run(mode, calls):
    p = oid.make_params(m=m, k=8, ell=ell, b_max=64, n_cap=4096, lam=-1.0, seed=5, dtype="f64", k1_mode=mode)
    eng = oid.Engine(p)
    outs = []
    for _ in range(calls):
        eng.ingest_sketch(X); torch.cuda.synchronize()
        outs.append(eng.partials(0)[: (ell + 1) * b].clone().cpu().numpy())
        if mode == oid.K1_TC_FAST:
            gE = eng.get(15)
            print("   counters", gE[-8:].tolist(), "col1 guesses (units 0..7)", gE[:-8].reshape(256, 32)[:8, 1].tolist(),
                  "min/max over units col1", gE[:-8].reshape(256, 32)[:148, 1].min(), gE[:-8].reshape(256, 32)[:148, 1].max())
    eng.close()
    return outs
ex = run(oid.K1_TC_INT8, 1)[0]
Y = ex[:ell*b].reshape(b, ell).T
colmax = X.abs().amax(0).cpu().numpy()
for ci, f in enumerate(run(oid.K1_TC_FAST, 5)):
    Yf = f[:ell*b].reshape(b, ell).T
    d = np.abs(Y - Yf) / (np.sqrt(m) * colmax[None, :])
    bad = np.argwhere(d > 1e-6)
    cols = sorted(set(bad[:, 1].tolist()))
    rows = sorted(set(bad[:, 0].tolist()))
    print(f"call {ci}: max {d.max():.2e} bad entries {len(bad)} cols {cols[:10]} rows {rows[:8]}..{rows[-3:] if rows else ''} n {np.abs(ex[ell*b:]-f[ell*b:]).max()/np.abs(ex[ell*b:]).max():.1e}")
