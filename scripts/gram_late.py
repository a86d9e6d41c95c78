"""Diagnostics: A9 (basis Gram) time late in the C3 stream (small nd), one stream, CUDA events
around oid_estimate_begin (dirty list + A9 + partial sums; the A10 factors run on side stream 2)."""
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
p = oid.make_params(m=gen.m, k=C3.k, ell=C3.ell, b_max=C3.b, n_cap=1000, lam=-1.0, seed=0)
eng = oid.Engine(p)
out = torch.empty(8, dtype=torch.float64, device=dev)
prevJ = None
for blk in range(28):
    X = gen.block_torch(blk * C3.b, (blk + 1) * C3.b, dev).T
    eng.ingest_block(X)
    torch.cuda.synchronize()
    J = eng.J()
    nd = None if prevJ is None else int(((J != prevJ) & (J >= 0)).sum())
    prevJ = J
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    eng.estimate_begin()
    b.record()
    eng.estimate_end(out)
    torch.cuda.synchronize()
    if blk >= 20:
        ms = a.elapsed_time(b)
        print(f"block {blk}: changed slots {nd}, A9 {ms:.3f} ms, {22.83 / ms:.2f} TB/s of basis read")
