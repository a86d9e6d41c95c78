"""A9Q vs the fp64 A9 on the same K1F stream: G after each estimate (relative to sqrt(G_ii G_jj)),
and the mean A9 launch time (profile events) on C3r or the full C3 grid."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from __graft_entry__ import build
build()
import paper_2405_16076_b200 as oid
from synth import ChannelFlow, C3, C3R
full = "--full" in sys.argv
dev = torch.device("cuda", 0)
gen = ChannelFlow(192, 129, 192, seed=C3.data_seed) if full else ChannelFlow(48, 33, 48, seed=C3R.data_seed)
b, nblk = 32, (6 if full else 10)
def run(a9q):
    p = oid.make_params(m=gen.m, k=200, ell=512, b_max=b, n_cap=nblk * b, lam=-1.0, seed=0, k1_mode=oid.K1_TC_FAST, profile=True,
                        a9q=a9q)
    eng = oid.Engine(p)
    Gs, ts = [], []
    for blk in range(nblk):
        X = gen.block_torch(blk * b, (blk + 1) * b, dev).T
        eng.ingest_block(X)
        st0 = eng.stats()
        eng.error_estimate()
        st = eng.stats()
        Gs.append(eng.get(11).copy())
        ts.append((st["a9_ms"] - st0["a9_ms"]) / max(1, st["a9_launches"] - st0["a9_launches"]))
        del X
    J = eng.J()
    eng.close()
    return Gs, ts, J
Gq, tq, Jq = run(True)
Ge, te, Je = run(False)
assert np.array_equal(Jq, Je), "J differs"
for e, (a, b_) in enumerate(zip(Gq, Ge)):
    d = np.sqrt(np.outer(np.diag(b_), np.diag(b_))) + 1e-300
    print(f"estimate {e}: max |dG|/sqrt(GiiGjj) {np.max(np.abs(a - b_) / d):.2e}  A9Q {tq[e]:.3f} ms  fp64 A9 {te[e]:.3f} ms")
