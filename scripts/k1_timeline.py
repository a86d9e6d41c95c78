"""K1 per-role timeline of CTA 0 (OID_K1_DEBUG=1): where does each tile's time go?

Rows (k1_tc.cuh): 0 A ready (generator arrive), 1 B ready (slicer arrive), 2 MMA start (both
stages ready), 3 MMA issued, 4 TMA issue, 5 slicer tile start, 6 slicer after x_full wait,
7 slicer after b_empty wait, 8 slicer after convert + bar_or, 9 raise flag of the tile."""
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
p = oid.make_params(m=gen.m, k=200, ell=512, b_max=32, n_cap=64 * 32, lam=-1.0, seed=0, profile=True,
                    k1_mode=int(os.environ.get("K1_MODE", "3")))
eng = oid.Engine(p)
for _ in range(3):
    eng.ingest_sketch(X)
torch.cuda.synchronize()
d = eng.get(10).astype(np.float64)
n = int(np.sum(d[3] > 0))
A, B, M0, M1, T, S0, S1, S2, S3, F, SL = (d[i][:n] for i in range(11))
base = T[0]
print(f"tiles {n}; total {M1[-1] - base:.0f} cycles ({(M1[-1] - base) / n:.0f}/tile)")
G0 = d[11].reshape(16, 256)
print('raises per slicer warp (CTA 0, columns x tiles):', d[10][4000:4008].astype(int).tolist())
I0, I1 = d[9][:min(n, 2048)], d[9][2048:2048 + min(n, 2048)]
print("issuer: loop top -> a_full done %.0f ; a_full -> b_full done + fence %.0f ; prev issued -> loop top %.0f" %
      (np.median(I1[100:n-1] - I0[100:n-1]), np.median(M0[100:n-1] - I1[100:n-1]), np.median(I0[101:n] - M1[100:n-1])))
print("slicer warps (CTA 0: 0-7, CTA 1: 8-15) publish vs MMA start, tiles 100..250 (median cycles before):",
      [int(np.median(M0[100:250] - G0[w, 100:250])) for w in range(16)])

dt = lambda x: np.diff(x)
print("per-tile cadence (median cycles): A ready %.0f  B ready %.0f  MMA start %.0f  MMA issued %.0f  TMA %.0f" %
      tuple(np.median(dt(x)) for x in (A, B, M0, M1, T)))
print("MMA start - A ready (median): %.0f ; MMA start - B ready: %.0f ; MMA issue duration: %.0f" %
      (np.median(M0 - A), np.median(M0 - B), np.median(M1 - M0)))
print("B ready - TMA issue (same tile): %.0f" % np.median(B - T))
print("slicer: after x_full -> loads+norms done %.0f ; -> b_empty done %.0f" % (np.median(SL - S1), np.median(S2 - SL)))
print("slicer (median cycles): x_full wait %.0f | load+norms+b_empty wait %.0f | convert+bar_or %.0f | publish %.0f | to next %.0f" %
      (np.median(S1 - S0), np.median(S2 - S1), np.median(S3 - S2), np.median(B - S3), np.median(S0[1:] - B[:-1])))
for t in [0, 1, 2, 3, 10, 100, 1000, n - 1]:
    print(t, "A %.0f B %.0f M0 %.0f M1 %.0f T %.0f S0 %.0f" % (A[t] - base, B[t] - base, M0[t] - base, M1[t] - base, T[t] - base, S0[t] - base))
dM = np.diff(M0)
print("MMA-start gaps: mean %.0f median %.0f; total above 2x median: %.0f cycles" % (dM.mean(), np.median(dM), dM[dM > 2 * np.median(dM)].sum()))
big = np.argsort(-dM)[:12]
print("largest gaps (tile: cycles):", [(int(i) + 1, int(dM[i])) for i in sorted(big)])
