"""Diagnostics: one C3 block ingested, then estimates (basis Gram with nd = admissions of the block)."""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__ as ge
ge.build()
import paper_2405_16076_b200 as oid
from synth import ChannelFlow, C3

gen = ChannelFlow(192, 129, 192, seed=1003)
dev = torch.device("cuda", 0)
p = oid.make_params(m=gen.m, k=C3.k, ell=C3.ell, b_max=C3.b, n_cap=1000, lam=-1.0, seed=0, profile=True)
eng = oid.Engine(p)
X = gen.block_torch(0, C3.b, dev).T
eng.ingest_block(X)
eng.error_estimate()
torch.cuda.synchronize()
eng.stats_reset()
eng.ingest_block(gen.block_torch(C3.b, 2 * C3.b, dev).T)
e = eng.error_estimate()
st = eng.stats()
print("est_ms", st["est_ms"], e)
