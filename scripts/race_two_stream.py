"""Repro for the two-stream estimate race (tests/test_gpu_parity.py::test_two_stream_estimates_match_one_stream).

A reference run (one engine alone, caller's default stream) is taken first; then two engines A and B
run interleaved block by block, each with its own stream set-up ("default": the caller's default
stream; "hi": ingest and estimate on one side stream; "hilo": ingest on a high-priority stream,
estimate on a low-priority one, delayed by a device spin), and each engine's estimates and J are
compared with the reference.  RACE_MODES selects variants by name."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from synth import ChannelFlow, C3R   # noqa: E402

NBLK = 8
SPLIT = os.environ.get("RACE_SPLIT", "0") == "1"   # B: sketch, copy of the sketch partials, commit
YREF = []


def params(oid):
    cfg = C3R
    a, b = cfg.ell // 6, cfg.ell // 3
    split = (a, b, cfg.ell - a - b)
    return oid.make_params(m=cfg.m, k=cfg.k, ell=cfg.ell, b_max=cfg.b, n_cap=NBLK * cfg.b, lam=-1.0, split=split, seed=0,
                           k1_mode=int(os.environ.get("RACE_K1", "0")))


class Runner:
    def __init__(self, oid, setup, env, delay):
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        self.setup, self.delay = setup, delay
        self.hi = self.lo = None
        if setup == "default":
            self.eng = oid.Engine(params(oid))
        elif setup == "hi":
            self.hi = torch.cuda.Stream(priority=-1)
            self.eng = oid.Engine(params(oid), stream=self.hi, estimate_stream=self.hi)
        else:
            self.hi = torch.cuda.Stream(priority=-1)
            self.lo = torch.cuda.Stream(priority=0)
            self.eng = oid.Engine(params(oid), stream=self.hi, estimate_stream=self.lo)
        for k, v in old.items():
            if v is None:
                os.environ.pop(k)
            else:
                os.environ[k] = v
        self.out = torch.empty((NBLK, 8), dtype=torch.float64, device="cuda:0")
        self.ycopy = []

    def step(self, e, X):
        if self.hi is not None:
            with torch.cuda.stream(self.hi):
                if SPLIT:
                    self.eng.ingest_sketch(X)
                    self.ycopy.append(self.eng.partials(0).clone())
                    self.eng.ingest_commit(X)
                else:
                    self.eng.ingest_block(X)
        else:
            self.eng.ingest_block(X)
        if self.delay and self.lo is not None:
            with torch.cuda.stream(self.lo):
                torch.cuda._sleep(self.delay)
        self.eng.estimate_begin()
        self.eng.estimate_end(self.out[e])


def blocks():
    cfg = C3R
    gen = ChannelFlow(48, 33, 48, seed=cfg.data_seed)
    A = gen.block(0, NBLK * cfg.b)
    Ad = torch.from_numpy(np.asfortranarray(A)).to("cuda:0")
    return [Ad[:, j:j + cfg.b] for j in range(0, NBLK * cfg.b, cfg.b)]


REF = {}


def snapshot(eng):
    return dict(J=eng.J(), S=eng.get(2), G=eng.get(3), sc=eng.get(4), rep=eng.report())


def compare(name, ref_out, ref_J, r):
    o = r.out.cpu().numpy()
    bad = np.flatnonzero((o != ref_out).any(axis=1))
    J = r.eng.J()
    msg = f"{name}: bad rows {bad.tolist()} J {'ok' if np.array_equal(J, ref_J) else 'DIFF'}"
    if bad.size and REF:
        d = snapshot(r.eng)
        S, R = d["S"], REF["S"]
        print("S shape", S.shape, flush=True)
        dm = S != R
        cols = np.flatnonzero(dm.any(axis=0))
        rows = np.flatnonzero(dm.any(axis=1))
        rel = np.abs(S - R).max() / np.abs(R).max()
        msg += (f" | S entries differing {int(dm.sum())} of {dm.size}, max rel {rel:.3e}, rows {rows[:8].tolist()}..({rows.size})"
                f" cols {cols[:8].tolist()}..({cols.size}) G {'ok' if np.array_equal(d['G'], REF['G']) else 'DIFF'}")
        # per-column max relative difference for the first differing columns
        for c in cols[:4]:
            msg += f" [col {c}: {int(dm[:, c].sum())} entries, max rel {np.abs(S[:, c] - R[:, c]).max() / np.abs(R[:, c]).max():.2e}]"
        msg += f" sc diff idx {np.flatnonzero(d['sc'] != REF['sc']).tolist()}"
        for key in ("epoch_log",):
            if key in d["rep"]:
                a, b = d["rep"][key], REF["rep"][key]
                first = next((i for i, (x, y) in enumerate(zip(a, b)) if x != y), None)
                msg += f" | first differing {key} row {first}: {a[first] if first is not None else ''} vs {b[first] if first is not None else ''}"
                break
        else:
            msg += f" | report keys {list(d['rep'].keys())}"
    return bad.size, msg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=4)
    args = ap.parse_args()
    from __graft_entry__ import build
    build()
    import paper_2405_16076_b200 as oid
    X = blocks()
    ref = Runner(oid, "default", {}, 0)
    for e in range(NBLK):
        ref.step(e, X[e])
    torch.cuda.synchronize()
    ref_out, ref_J = ref.out.cpu().numpy(), ref.eng.J()
    REF.update(snapshot(ref.eng))
    if SPLIT:   # solo sketches of every block
        hs = torch.cuda.Stream(priority=-1)
        ys = Runner(oid, "hi", {}, 0)
        for e in range(NBLK):
            with torch.cuda.stream(ys.hi):
                ys.eng.ingest_sketch(X[e])
                YREF.append(ys.eng.partials(0).clone())
        torch.cuda.synchronize()
        YREF[:] = [y.cpu().numpy() for y in YREF]
        del ys
    del ref
    D = 4_000_000
    variants = {
        # name: ((setupA, envA, delayA), (setupB, envB, delayB) or None)
        "solo-hilo": (("hilo", {}, D), None),
        "def+hilo": (("default", {}, 0), ("hilo", {}, D)),
        "def+hi": (("default", {}, 0), ("hi", {}, 0)),
        "hi+hi": (("hi", {}, 0), ("hi", {}, 0)),
        "hi+hilo": (("hi", {}, 0), ("hilo", {}, D)),
        "def+def": (("default", {}, 0), ("default", {}, 0)),
        "noside2": (("default", {"OID_NO_SIDE": "1"}, 0), ("hilo", {"OID_NO_SIDE": "1"}, D)),
        "noside-hi": (("hi", {"OID_NO_SIDE": "1"}, 0), ("hi", {"OID_NO_SIDE": "1"}, 0)),
    }
    sel = os.environ.get("RACE_MODES", "all")
    for name, (a, b) in variants.items():
        if sel != "all" and name not in sel.split(","):
            continue
        fa = fb = 0
        for rep in range(args.reps):
            ra = Runner(oid, *a)
            rb = Runner(oid, *b) if b else None
            torch.cuda.synchronize()
            for e in range(NBLK):
                ra.step(e, X[e])
                if rb:
                    rb.step(e, X[e])
            torch.cuda.synchronize()
            na, da = compare("A", ref_out, ref_J, ra)
            nb, db = compare("B", ref_out, ref_J, rb) if rb else (0, "")
            fa += na > 0
            fb += nb > 0
            if na or nb:
                print(f"{name} rep{rep}: {da}; {db}", flush=True)
            if rb is not None and rb.ycopy:
                for e, yc in enumerate(rb.ycopy):
                    y = yc.cpu().numpy()
                    if not YREF:
                        break
                    if not np.array_equal(y, YREF[e]):
                        print(f"   B sketch of block {e} differs from the solo sketch right after K1: "
                              f"{int((y != YREF[e]).sum())} entries", flush=True)
            del ra, rb
        print(f"VARIANT {name}: A failed {fa}/{args.reps}, B failed {fb}/{args.reps}", flush=True)


if __name__ == "__main__":
    main()
