"""A9Q vs fp64 A9 on C1 (K1F): relative G error and the NA-Hutch++ components after each estimate."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from __graft_entry__ import build
build()
import paper_2405_16076_b200 as oid
from synth import c1_matrix
dev = torch.device("cuda", 0)
A = c1_matrix(); s = np.linalg.svd(A, compute_uv=False); lam = float(np.sum(s[20:] ** 2) / 20)
Ad = torch.from_numpy(np.asfortranarray(A)).to(dev)
def run(a9q):
    p = oid.make_params(m=4096, k=20, ell=48, b_max=16, n_cap=512, lam=lam, split=(16, 16, 16), seed=0, k1_mode=4, a9q=a9q)
    eng = oid.Engine(p); out = []
    for j in range(0, 512, 16):
        eng.ingest_block(Ad[:, j:j + 16]); est = eng.error_estimate(); out.append((eng.get(11).copy(), est))
    basis = eng.finalize(basis=True)["basis"].cpu().numpy(); J = eng.J(); eng.close(); return out, basis, J
q, bq, Jq = run(True); e, be, Je = run(False)
print("J equal", np.array_equal(Jq, Je))
for i in (0, 3, 7, 15, 31):
    Gq, Ge = q[i][0], e[i][0]
    d = np.sqrt(np.outer(np.diag(Ge), np.diag(Ge))) + 1e-300
    print(i, f"max|dG|/sqrt(GiiGjj) {np.max(np.abs(Gq - Ge) / d):.2e}", "T", q[i][1]["T"], e[i][1]["T"], "gpp", q[i][1]["gpp"], e[i][1]["gpp"], "frob2", e[i][1]["frob2"])
G = be.T @ be
print("final fp64 A9 G vs basis dot: ", np.max(np.abs(e[-1][0] - G) / (np.sqrt(np.outer(np.diag(G), np.diag(G))) + 1e-300)))
print("final A9Q G vs basis dot: ", np.max(np.abs(q[-1][0] - G) / (np.sqrt(np.outer(np.diag(G), np.diag(G))) + 1e-300)))
print("max |basis| per column", np.max(np.abs(be), axis=0)[:5], "min nonzero col max", np.min(np.max(np.abs(be), axis=0)))
