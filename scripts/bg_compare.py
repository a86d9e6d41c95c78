"""Diagnostics: A9 basis Gram of the TMA+DMMA kernel vs the cp.async kernel (OID_BG_SIMT=1) on
the C3 stream, same process; prints per-block max |dG| / scale and the estimates."""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__ as ge
ge.build()
import paper_2405_16076_b200 as oid
from synth import ChannelFlow, C3

nblk = int(sys.argv[1]) if len(sys.argv) > 1 else 6
gen = ChannelFlow(192, 129, 192, seed=C3.data_seed)
dev = torch.device("cuda", 0)
p = oid.make_params(m=gen.m, k=C3.k, ell=C3.ell, b_max=C3.b, n_cap=64 * 32, lam=-1.0, seed=0, profile=True)
os.environ["OID_BG_SIMT"] = "0"
e1 = oid.Engine(p)
os.environ["OID_BG_SIMT"] = "1"
e2 = oid.Engine(p)
for blk in range(nblk):
    X = gen.block_torch(blk * C3.b, (blk + 1) * C3.b, dev).T
    out = []
    for e in (e1, e2):
        e.ingest_block(X)
        out.append(e.error_estimate())
    G1, G2 = e1.get(11), e2.get(11)
    d = np.sqrt(np.abs(np.diag(G2)))
    sc = np.outer(d, d) + 1e-300
    print(blk, "J equal", np.array_equal(e1.J(), e2.J()), "max|dG|/scale %.3e" % np.max(np.abs(G1 - G2) / sc),
          "est tc %.6e simt %.6e" % (out[0]["est_rel"], out[1]["est_rel"]), "e2 %.6e %.6e" % (out[0]["e2"], out[1]["e2"]))
for e, name in ((e1, "tc"), (e2, "simt")):
    st = e.stats()
    print(name, {k: st[k] for k in ("k1_ms", "post_ms", "est_ms")})
