"""Diagnostics: Jacobi rotation counts per sweep (oid_get field 9) for the Gram eigen path on a
C2 prefix (pseudo-inverse regime), per epoch."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from __graft_entry__ import build
build()
import paper_2405_16076_b200 as oid
from synth import ImageStream, C2
img = ImageStream(seed=C2.data_seed)
p = oid.make_params(m=C2.m, k=C2.k, ell=C2.ell, b_max=C2.b, n_cap=2048, lam=-1.0, seed=0, dtype="f32", profile=True)
eng = oid.Engine(p)
for e in range(12):
    X = torch.from_numpy(np.asfortranarray(img.block(e * 64, (e + 1) * 64))).cuda()
    eng.ingest_block(X)
    torch.cuda.synchronize()
    c = eng.get(9)
    sc = eng.scalars()
    nz = [int(v) for v in c[0] if v > 0]
    print(e, "lam", sc["lam"], "sweeps", len(nz), "rotations", nz[:12], "post_ms", round(eng.stats()["post_ms"], 3))
    eng.stats_reset()
