"""Small C1 run through the public API (ingest every block, estimate, finalize) for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck): `compute-sanitizer --tool X
python scripts/sanitize_c1.py [--argmin]`.  Checks the result against the oracle at the end so a
sanitizer-perturbed run that goes wrong also fails."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from __graft_entry__ import build  # noqa: E402

build()
import paper_2405_16076_b200 as oid  # noqa: E402
from oracle import OracleOID, OracleParams  # noqa: E402
from synth import c1_matrix  # noqa: E402

coeff = "argmin" if "--argmin" in sys.argv else "alg4"
m, n, b, k, ell = 2048, 96, 16, 10, 36
split = (6, 12, 18)
A = c1_matrix(seed=1001, m=m, n=n, rank=10, noise=1e-6)
eng = oid.Engine(oid.make_params(m=m, k=k, ell=ell, b_max=b, n_cap=n, lam=0.0, split=split, seed=2, coeff=coeff))
o = OracleOID(OracleParams(m=m, k=k, ell=ell, ell1=6, ell2=12, ell3=18, lam=0.0, seed=2, coeff=coeff))
Ad = torch.from_numpy(np.asfortranarray(A)).cuda()
for j in range(0, n, b):
    eng.ingest_block(Ad[:, j:j + b])
    o.ingest_block(A[:, j:j + b])
    est = eng.error_estimate()
fin = eng.finalize(basis=True)
assert np.array_equal(fin["J"], o.J)
P = fin["P"].cpu().numpy()
rel = np.linalg.norm(P - o.P) / np.linalg.norm(o.P)
assert rel < 1e-6, rel
print(f"sanitize_c1 ok ({coeff}): relP {rel:.2e}, est_rel {est['est_rel']:.3e}, stats {eng.stats()['launches']} launches")
