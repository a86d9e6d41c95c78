"""NA-Hutch++ estimate (Alg 8) against the true relative error of the ID,
||A_obs - A_J P||_F / ||A_obs||_F (plain definition, numpy fp64 on the host), along the C3r
stream (BJ configs[2] on the 48x33x48 grid, lambda = paper surrogate, seed 0), through the CUDA
engine; also the A12 run report's per-estimate log.  Writes JSON to stdout."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from __graft_entry__ import build  # noqa: E402

build()
import paper_2405_16076_b200 as oid  # noqa: E402
from synth import ChannelFlow, C3R  # noqa: E402

cfg = C3R
gen = ChannelFlow(48, 33, 48, seed=cfg.data_seed)
A = gen.block(0, cfg.n)
split = oid.hutch_split(cfg.ell)
p = oid.make_params(m=cfg.m, k=cfg.k, ell=cfg.ell, b_max=cfg.b, n_cap=cfg.n, lam=-1.0, split=split, seed=0)
eng = oid.Engine(p)
Ad = torch.from_numpy(np.asfortranarray(A)).cuda()
rows = []
for e, j in enumerate(range(0, cfg.n, cfg.b)):
    eng.ingest_block(Ad[:, j:j + cfg.b])
    n_obs = min(cfg.n, j + cfg.b)
    if (e + 1) % 4 == 0 or n_obs in (800, cfg.n):
        est = eng.error_estimate()
        fin = eng.finalize(basis=True)
        B = fin["basis"].cpu().numpy()
        P = fin["P"].cpu().numpy()
        Ao = A[:, :n_obs]
        true_rel = float(np.linalg.norm(Ao - B @ P) / np.linalg.norm(Ao))
        rows.append(dict(n_obs=n_obs, est_rel=float(est["est_rel"]), e2=float(est["e2"]), true_rel=true_rel,
                         ratio=float(est["est_rel"] / true_rel) if true_rel > 0 else None, flags=int(est["flags"])))
        print(rows[-1], file=sys.stderr, flush=True)
rep = eng.report()
print(json.dumps({"workload": "C3r (m=228096, n=1000, b=32, k=200, l=512, lambda=-1, seed 0)",
                  "checkpoints": rows, "report_totals": {k: v for k, v in rep.items() if not k.endswith("_log")}},
                 indent=1))
