"""K1 determinism under concurrent load: one engine sketches the same blocks again and again
(oid_ingest_sketch, output = the (ell + 1) x b partials) on its own stream while other work runs
on the default stream; every repetition must give bitwise the reference sketch taken alone.

  python scripts/k1_determinism.py [--k1 2] [--reps 20] [--load engine|matmul|none]"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from synth import ChannelFlow, C3R   # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--k1", type=int, default=2)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--load", default="engine")
    args = ap.parse_args()
    from __graft_entry__ import build
    build()
    import paper_2405_16076_b200 as oid
    cfg = C3R
    nblk = 8
    A = ChannelFlow(48, 33, 48, seed=cfg.data_seed).block(0, nblk * cfg.b)
    Ad = torch.from_numpy(np.asfortranarray(A)).to("cuda:0")
    X = [Ad[:, j:j + cfg.b] for j in range(0, nblk * cfg.b, cfg.b)]
    a, b = cfg.ell // 6, cfg.ell // 3

    def params(k1):
        return oid.make_params(m=cfg.m, k=cfg.k, ell=cfg.ell, b_max=cfg.b, n_cap=nblk * cfg.b, lam=-1.0,
                               split=(a, b, cfg.ell - a - b), seed=0, k1_mode=k1)

    hi = torch.cuda.Stream(priority=-1)
    eng = oid.Engine(params(args.k1), stream=hi)
    ref = []
    for e in range(nblk):
        with torch.cuda.stream(hi):
            eng.ingest_sketch(X[e])
            ref.append(eng.partials(0).clone())
    torch.cuda.synchronize()
    ref = [r.cpu().numpy() for r in ref]
    nbad = 0
    for rep in range(args.reps):
        load = oid.Engine(params(args.k1)) if args.load == "engine" else None
        M = torch.randn(4096, 4096, device="cuda:0", dtype=torch.float64) if args.load == "matmul" else None
        outs = []
        torch.cuda.synchronize()
        for e in range(nblk):
            if load is not None:
                load.ingest_block(X[e])
                load.estimate_begin()
                load.estimate_end()
            elif M is not None:
                M = M @ M * 1e-2
            with torch.cuda.stream(hi):
                eng.ingest_sketch(X[e])
                outs.append(eng.partials(0).clone())
        torch.cuda.synchronize()
        for e in range(nblk):
            o = outs[e].cpu().numpy()
            d = np.flatnonzero(o != ref[e])
            if d.size:
                nbad += 1
                Y, R = o[:cfg.ell * cfg.b].reshape(cfg.b, cfg.ell), ref[e][:cfg.ell * cfg.b].reshape(cfg.b, cfg.ell)
                cols = np.flatnonzero((Y != R).any(axis=1))
                rows = np.flatnonzero((Y != R).any(axis=0))
                print(f"rep {rep} block {e}: {d.size} entries differ, cols {cols.tolist()[:12]} rows "
                      f"[{rows.min() if rows.size else -1}..{rows.max() if rows.size else -1}] ({rows.size}), "
                      f"max rel {np.abs(Y - R).max() / np.abs(R).max():.2e}", flush=True)
        del load
    print(f"K1 mode {args.k1} load {args.load}: {nbad} differing block sketches of {args.reps * nblk}", flush=True)


if __name__ == "__main__":
    main()
