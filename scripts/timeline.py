"""Diagnostics: per-step stream timeline of the bench loop (OID_TIMELINE=1), two streams
(ingest high priority, estimate low) unless --one-stream.  Prints each tagged mark in ms.
--workload C3 (default) or C5r; --start S skips S blocks first."""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["OID_TIMELINE"] = "1"
import __graft_entry__ as ge
ge.build()
import paper_2405_16076_b200 as oid
from synth import ChannelFlow, LowRankStream, C3, C5R

one = "--one-stream" in sys.argv
steps = 6
start = int(sys.argv[sys.argv.index("--start") + 1]) if "--start" in sys.argv else 0
wl = sys.argv[sys.argv.index("--workload") + 1] if "--workload" in sys.argv else "C3"
if wl == "C5r":
    cfg, gen = C5R, LowRankStream(m=C5R.m, seed=1005)
    dt = "f32"
else:
    cfg, gen = C3, ChannelFlow(192, 129, 192, seed=1003)
    dt = "f64"
dev = torch.device("cuda", 0)
p = oid.make_params(m=gen.m, k=cfg.k, ell=cfg.ell, b_max=cfg.b, n_cap=cfg.n, lam=-1.0, seed=0, dtype=dt,
                    k1_mode=int(sys.argv[sys.argv.index("--k1") + 1]) if "--k1" in sys.argv else 4,
                    a9q="--a9fp64" not in sys.argv)
I = torch.cuda.Stream(dev, priority=-1)
E = I if one else torch.cuda.Stream(dev, priority=0)
eng = oid.Engine(p, stream=I, estimate_stream=E)
blocks = [gen.block_torch(s * cfg.b, (s + 1) * cfg.b, dev).T for s in range(start + steps)]
torch.cuda.synchronize()
out = torch.empty(8, dtype=torch.float64, device=dev)
for s in range(start):
    eng.ingest_block(blocks[s])
    eng.estimate_begin()
    eng.estimate_end(out)
torch.cuda.synchronize()
eng.get(13)   # drop the warm-up marks
blocks = blocks[start:]
pipe = "--pipeline" in sys.argv
for s in range(steps):
    eng.ingest_block(blocks[s])
    if pipe:
        if s > 0:
            eng.estimate_end(out)
        eng.estimate_begin()
    else:
        eng.estimate_begin()
        eng.estimate_end(out)
if pipe:
    eng.estimate_end(out)
torch.cuda.synchronize()
tl = eng.get(13)
sc = eng.scalars()
print("lambda", sc["lam"], "shift", sc["shift"], "dmax", sc["dmax"], "kappa", sc["kappa"])
names = {1: "K1 start", 2: "K1 end", 3: "commit start", 4: "post chain end", 5: "copy start", 6: "copy end",
         11: "S_J chain start (side)", 12: "S_J chain end (side)", 7: "est begin (E)", 13: "est_pre start (side)",
         14: "est_pre end (side)", 15: "  tridiag end", 16: "  tri_scores end", 8: "Gram start (E)", 9: "Gram end (E)", 10: "est end (E)"}
rows = [(int(t), ms) for t, ms in tl if t >= 0]
for t, ms in rows:
    print(f"{ms:9.3f}  {names.get(t, t)}")
k1s = [ms for t, ms in rows if t == 1]
print("K1 start deltas:", np.round(np.diff(k1s), 3))
