"""Diagnostics: per-step phase timing of the cluster tridiagonalisation (A4) on C3 (OID_K1_DEBUG=1)."""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["OID_K1_DEBUG"] = "1"
import __graft_entry__ as ge
ge.build()
import paper_2405_16076_b200 as oid
from synth import ChannelFlow, C3

gen = ChannelFlow(192, 129, 192, seed=C3.data_seed)
dev = torch.device("cuda", 0)
p = oid.make_params(m=gen.m, k=C3.k, ell=C3.ell, b_max=C3.b, n_cap=256, lam=-1.0, seed=0)
e = oid.Engine(p)
for blk in range(3):
    X = gen.block_torch(blk * C3.b, (blk + 1) * C3.b, dev).T
    e.ingest_block(X)
    torch.cuda.synchronize()
    T = e.get(12)[: C3.ell - 2].astype(np.float64)
    ph1 = T[:, 1] - T[:, 0]      # column scatter (incl. phase-3 update of the previous step)
    b1 = T[:, 2] - T[:, 1]       # cluster barrier 1
    ph2 = T[:, 3] - T[:, 2]      # reflector + matvec + p scatter + barrier 2
    step = np.diff(T[:, 0])
    print(f"block {blk}: cycles/step median {np.median(step):.0f} mean {np.mean(step):.0f}; "
          f"phase1 {np.median(ph1):.0f}  barrier1 {np.median(b1):.0f}  phase2+barrier2 {np.median(ph2):.0f}  "
          f"phase3 {np.median(step - ph1[:-1] - b1[:-1] - ph2[:-1]):.0f}; total {(T[-1,3]-T[0,0])/1.965e6:.3f} ms")
