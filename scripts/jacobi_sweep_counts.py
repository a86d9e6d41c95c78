"""Diagnostics: rotations per sweep of the warm-started two-sided block Jacobi (A4/A5 eigenvector
path, use 0) per epoch on the C2 and C5r streams, and the per-ingest wall time."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2405_16076_b200 as oid
from synth import CONFIGS, ImageStream, LowRankStream

def run(name, nblk):
    c = CONFIGS[name]
    p = oid.make_params(m=c.m, k=c.k, ell=c.ell, b_max=c.b, n_cap=c.b * nblk, lam=c.lam, split=c.split, seed=0,
                        dtype=c.dtype)
    eng = oid.Engine(p)
    gen = ImageStream(seed=c.data_seed) if name == "C2" else LowRankStream(m=c.m, seed=c.data_seed)
    for e in range(nblk):
        A = gen.block(e * c.b, (e + 1) * c.b)
        X = torch.from_numpy(np.asfortranarray(A.astype(np.float32 if c.dtype == "f32" else np.float64))).cuda()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eng.ingest_block(X)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) * 1e3
        cnt = eng.get(9)
        cnt = np.asarray(cnt).reshape(-1, 48)[0]
        nz = [int(v) for v in cnt if v]
        print(f"{name} epoch {e:3d} ingest {dt:8.2f} ms  sweeps {len(nz):2d} rotations/sweep {nz}", flush=True)

run("C2", 12)
run("C5r", 8)
