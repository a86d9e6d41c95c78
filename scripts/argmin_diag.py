import sys, numpy as np
sys.path.insert(0, '.')
import __graft_entry__ as ge; ge.build()
import torch, paper_2405_16076_b200 as oid
from oracle import OracleParams, OracleOID
from synth import c1_matrix
m, n, b, k, ell = 2000, 160, 16, 12, 36
A = c1_matrix(seed=51, m=m, n=n, rank=14, noise=1e-3)
split = (6, 12, 18)
eng = oid.Engine(oid.make_params(m=m, k=k, ell=ell, b_max=b, n_cap=n, lam=0.0, split=split, seed=8, coeff="argmin"))
o = OracleOID(OracleParams(m=m, k=k, ell=ell, ell1=6, ell2=12, ell3=18, lam=0.0, seed=8, coeff="argmin"))
Ad = torch.from_numpy(np.asfortranarray(A)).cuda()
for e, j in enumerate(range(0, n, b)):
    eng.ingest_block(Ad[:, j:j + b]); lg = o.ingest_block(A[:, j:j + b])
    row = eng.get(14)[e]
    print(e, int(row[1]), lg.qstar, np.round(row[2:6] / o.frob2, 7), np.round(np.array(lg.e2q) / o.frob2, 7))
