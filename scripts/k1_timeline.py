"""K1 per-role timeline of CTA 0 (OID_K1_DEBUG=1): where does each tile's time go?"""
import os, sys
os.environ["OID_K1_DEBUG"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from __graft_entry__ import build
build()
import paper_2405_16076_b200 as oid
from synth import ChannelFlow
gen = ChannelFlow(192, 129, 192, seed=1003)
X = gen.block_torch(0, 32, torch.device("cuda", 0)).T
p = oid.make_params(m=gen.m, k=200, ell=512, b_max=32, n_cap=64 * 32, lam=-1.0, seed=0, profile=True)
eng = oid.Engine(p)
for _ in range(3):
    eng.ingest_sketch(X)
torch.cuda.synchronize()
d = eng.get(10).astype(np.float64)
n = int(np.sum(d[3] > 0))
A, B, M0, M1, T = (d[i][:n] for i in range(5))
base = T[0]
print(f"tiles {n}; total {M1[-1] - base:.0f} cycles ({(M1[-1] - base) / n:.0f}/tile)")
dt = lambda x: np.diff(x)
print("per-tile cadence (median cycles): A ready %.0f  B ready %.0f  MMA start %.0f  MMA issued %.0f  TMA %.0f" %
      tuple(np.median(dt(x)) for x in (A, B, M0, M1, T)))
print("MMA start - A ready (median): %.0f ; MMA start - B ready: %.0f ; MMA issue duration: %.0f" %
      (np.median(M0 - A), np.median(M0 - B), np.median(M1 - M0)))
print("A ready - MMA issued(t-2) [gen latency after slot free]: %.0f" % np.median(A[2:] - M1[:-2]))
print("B ready - TMA issue (same tile): %.0f" % np.median(B - T))
S0, S1, S2, S3, S4 = (d[i][:n] for i in range(5, 10))
print("slicer (median cycles): prefetch load %.0f | wait b_empty + convert %.0f | fence+bar %.0f | decide+bar_or %.0f | epi/next %.0f" %
      (np.median(S1 - S0), np.median(S2 - S1), np.median(S3 - S2), np.median(S4 - S3), np.median(S0[1:] - S4[:-1])))
for t in [0, 1, 2, 3, 10, 100, 1000, n - 1]:
    print(t, "A %.0f B %.0f M0 %.0f M1 %.0f T %.0f" % (A[t] - base, B[t] - base, M0[t] - base, M1[t] - base, T[t] - base))
# slicer rows (group of tile t): 5 before x_full wait, 6 after load + b_empty wait, 7 after convert +
# bar_or, 8 after the token wait, 9 after the bookkeeping
print("slicer phases (median cycles): x wait+load+b_empty %.0f | convert+bar_or %.0f | token wait %.0f | bookkeeping %.0f | to next own tile %.0f" %
      (np.median(S1 - S0), np.median(S2 - S1), np.median(S3 - S2), np.median(S4 - S3), np.median(S0[2:] - S4[:-2])))
