"""K1-only driver for ncu captures and quick timing: C3-sized block(s), ingest_sketch only."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from __graft_entry__ import build
build()
import paper_2405_16076_b200 as oid
from synth import ChannelFlow, LowRankStream

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--grid", default="192,129,192")
ap.add_argument("--b", type=int, default=32)
ap.add_argument("--ell", type=int, default=512)
ap.add_argument("--mode", type=int, default=0)
ap.add_argument("--omega-cache", type=int, default=0)
ap.add_argument("--lowrank-m", type=int, default=0, help="C5-shaped slab: m rows of the fp32 low-rank stream")
a = ap.parse_args()
grid = tuple(int(x) for x in a.grid.split(","))
dev = torch.device("cuda", 0)
if a.lowrank_m:
    gen = LowRankStream(m=a.lowrank_m, seed=1005)
    X = gen.block_torch(0, a.b, dev).T
else:
    gen = ChannelFlow(*grid, seed=1003)
    X = gen.block_torch(0, a.b, dev).T
p = oid.make_params(m=gen.m, k=200, ell=a.ell, b_max=a.b, n_cap=64 * a.b, lam=-1.0, seed=0, profile=True,
                    dtype="f32" if X.dtype == torch.float32 else "f64", k1_mode=a.mode,
                    omega_cache=bool(a.omega_cache))
eng = oid.Engine(p)
for r in range(a.reps):
    eng.ingest_sketch(X)          # repeated sketches without commit are allowed (pending block replaced)
torch.cuda.synchronize()
st = eng.stats()
print(f"K1 {st['k1_ms'] / st['k1_launches']:.3f} ms/launch over {st['k1_launches']} launches, mode {st['k1_mode_used']}, "
      f"{gen.m * a.b * X.element_size() / (st['k1_ms'] / st['k1_launches'] * 1e-3) / 1e9:.1f} GB/s")
