"""Reading R2 ablation: the Gauss-16 sketch law against the paper's Gaussian Omega, CPU oracle.

For each of N sketch seeds and each law, run the oracle over a stream and record
  * the true relative reconstruction error ||A - A_J P||_F / ||A||_F after the last block (Alg 4),
  * the NA-Hutch++ estimate r_hat and its cross-trace error (T_hat - T)/||A||^2 (Alg 8),
then compare the laws by mean, standard error and the difference of means.
Streams: C1 (BASELINE config 0, fixed lambda, split 16/16/16) and a C2 prefix (first 1024 frames
of BASELINE config 1, paper surrogate lambda).  Writes profiles/r2_omega_law_study.json.

    python scripts/r2_study.py [--seeds 60]
"""
import argparse
import json
import math
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import OracleParams, OracleOID                      # noqa: E402
from synth import c1_matrix, ImageStream, C2                     # noqa: E402


def run(A, b, k, ell, split, lam, seed, law):
    o = OracleOID(OracleParams(m=A.shape[0], k=k, ell=ell, ell1=split[0], ell2=split[1], ell3=split[2], lam=lam,
                               seed=seed, omega_law=law))
    for j in range(0, A.shape[1], b):
        o.ingest_block(A[:, j:j + b])
    fro = float(np.sum(A * A))
    rec = o.C @ o.P
    err = math.sqrt(float(np.sum((A - rec) ** 2)) / fro)
    est = o.error_estimate()
    T = float(np.sum(A * rec))
    return dict(err=err, est_rel=est["est_rel"], dT=(est["T"] - T) / fro, e2_neg=bool(est["negative"]))


def summarize(vals):
    v = np.asarray(vals, dtype=np.float64)
    return dict(mean=float(v.mean()), se=float(v.std(ddof=1) / math.sqrt(v.size)), std=float(v.std(ddof=1)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", type=int, default=60)
    a = ap.parse_args()
    A1 = c1_matrix()
    s1 = np.linalg.svd(A1, compute_uv=False)
    lam1 = float(np.sum(s1[20:] ** 2) / 20)
    A2 = ImageStream(C2.data_seed).block(0, 1024).astype(np.float64)
    cases = {"C1": (A1, 16, 20, 48, (16, 16, 16), lam1), "C2_prefix1024": (A2, 64, 100, 256, C2.split, -1.0)}
    out = {"seeds": a.seeds, "cases": {}}
    t0 = time.time()
    for name, (A, b, k, ell, split, lam) in cases.items():
        res = {}
        for law in ("gauss16", "gaussian"):
            rows = [run(A, b, k, ell, split, lam, s, law) for s in range(a.seeds)]
            res[law] = {key: summarize([r[key] for r in rows]) for key in ("err", "est_rel", "dT")}
            res[law]["e2_negative_fraction"] = float(np.mean([r["e2_neg"] for r in rows]))
        diff = {}
        for key in ("err", "est_rel", "dT"):
            d = res["gauss16"][key]["mean"] - res["gaussian"][key]["mean"]
            se = math.hypot(res["gauss16"][key]["se"], res["gaussian"][key]["se"])
            diff[key] = dict(diff=d, se=se, z=d / se if se > 0 else 0.0)
        res["gauss16_minus_gaussian"] = diff
        out["cases"][name] = res
        print(name, json.dumps(diff), flush=True)
    out["seconds"] = time.time() - t0
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "r2_omega_law_study.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
