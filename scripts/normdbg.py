import numpy as np, torch, sys
sys.path.insert(0, '.')
from __graft_entry__ import build; build()
import paper_2405_16076_b200 as oid
for (m, nc, ell, dt) in [(5000, 7, 24, np.float64), (4096, 16, 48, np.float64), (70001, 32, 512, np.float64), (100000, 64, 512, np.float64), (5120, 64, 256, np.float32)]:
    rng = np.random.default_rng(m + nc)
    X = rng.standard_normal((m, nc)).astype(dt) * rng.uniform(0.1, 10, nc).astype(dt)
    X[rng.integers(0, m, 5), 0] *= 1e5
    p = oid.make_params(m=m, k=min(8, ell), ell=ell, b_max=64, n_cap=256, lam=0.0, seed=12345, dtype="f64" if dt == np.float64 else "f32")
    e = oid.Engine(p)
    e.ingest_sketch(torch.from_numpy(np.asfortranarray(X)).cuda())
    part = e.partials(0).cpu().numpy()
    ng = part[ell * nc: ell * nc + nc]
    nrm = np.sum(X.astype(np.float64) ** 2, axis=0)
    print(m, nc, ell, dt.__name__, "max rel norm err %.3e" % np.max(np.abs(ng - nrm) / nrm), np.abs(ng - nrm) / nrm)
