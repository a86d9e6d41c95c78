"""K1F (k1_mode = OID_K1_TC_FAST) against the CPU oracle.  Run with -m gpu on a B200.

K1F quantises every snapshot value to a 31-bit per-column fixed point before the exact int8
tensor-core contraction.  Its error bound, which these tests check:

* per element |x - x_q| <= 2^-27 max_i |x_ij| (=: delta_j): the kernel's unit is at most
  2^-27 of the column maximum of its row set (precision check kH + kShrink, reruns otherwise),
  the rounding error at most 0.75 unit;
* sketch: dY_rj = s sum_i L(r, i) e_ij with e_ij = x_q - x fixed by the data and the sketch entries
  independent of it with mean 0 (reading R2), |s L| <= s 110.5, so by Hoeffding
  |dY_rj| <= s 110.5 delta_j sqrt(2 m ln(2 / 1e-12)) except with probability 1e-12 per entry;
* norms: |sum x_q^2 - sum x^2| <= 2 delta_j sum_i |x_ij| + m delta_j^2 (the norm of x_q is exact).

Downstream the path is the exact one (A3-A10 unchanged), so the stream tests use the north_star bar:
J bit-exact whenever the oracle's decision margins are >= 1e-6 (reading R14), coefficients and
estimates within 1e-5.
"""

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import OracleParams, OracleOID                      # noqa: E402
from oracle.oid import sketch as oracle_sketch                   # noqa: E402
from oracle.gauss16 import omega_rows, gauss16_scale            # noqa: E402
from synth import c1_matrix, ChannelFlow, C3R, C3              # noqa: E402

FAST = 4
QUANT = 2.0 ** -27                       # per-element bound relative to the column maximum
HOEFF = math.sqrt(2.0 * math.log(2.0 / 1e-12))


@pytest.fixture(scope="module")
def oid():
    from __graft_entry__ import build
    build()
    import paper_2405_16076_b200 as oid
    assert torch.cuda.is_available()
    assert oid.K1_TC_FAST == FAST
    return oid


def _split(ell):
    a, b = ell // 6, ell // 3
    return (a, b, ell - a - b)


def _engine(oid, m, k, ell, b_max, n_cap, lam, seed=0, dtype="f64", split=None, a9q=False):
    split = _split(ell) if split is None else split
    p = oid.make_params(m=m, k=k, ell=ell, b_max=b_max, n_cap=n_cap, lam=lam, split=split, seed=seed, dtype=dtype,
                        k1_mode=FAST, a9q=a9q)
    return oid.Engine(p), split


def _dev(A, dtype):
    return torch.from_numpy(np.asfortranarray(A.astype(dtype))).to("cuda:0")


def _check_partials(part, X, ell, seed, Y=None):
    """Assert the K1F partial buffer [Y; n] of block X against the oracle within the bound."""
    m, nc = X.shape
    Xd = X.astype(np.float64)
    Yg = part[:ell * nc].reshape(nc, ell).T
    ng = part[ell * nc:ell * nc + nc]
    if Y is None:
        op = OracleParams(m=m, k=1, ell=ell, ell1=ell, ell2=0, ell3=0, lam=0.0, seed=seed)
        Y = oracle_sketch(op, Xd)
    delta = QUANT * np.max(np.abs(Xd), axis=0)
    bound = gauss16_scale() * 110.5 * delta * HOEFF * math.sqrt(m) + 1e-13 * np.max(np.abs(Y), axis=0)
    err = np.abs(Yg - Y)
    assert np.all(err <= bound[None, :]), float(np.max(err / bound[None, :]))
    nref = np.sum(Xd * Xd, axis=0)
    nb = 2 * delta * np.sum(np.abs(Xd), axis=0) + m * delta * delta + 1e-13 * nref
    assert np.all(np.abs(ng - nref) <= nb), float(np.max(np.abs(ng - nref) / nb))
    # the typical error is far below the worst case: relative Frobenius error of the sketch
    assert np.linalg.norm(Yg - Y) <= 1e-7 * np.linalg.norm(Y)
    return Yg


SKETCH_CASES = [(4096, 16, 48, np.float64), (5000, 7, 24, np.float64), (12346, 33, 96, np.float64),
                (776, 1, 8, np.float64), (5120, 64, 256, np.float32), (70002, 32, 512, np.float64),
                (3000, 64, 1024, np.float32), (100000, 64, 512, np.float64), (20000, 20, 300, np.float32),
                (66, 3, 640, np.float64), (64 * 148 + 2, 32, 512, np.float64)]


@pytest.mark.parametrize("m,nc,ell,dtype", SKETCH_CASES)
def test_k1f_sketch_bound(oid, m, nc, ell, dtype):
    """Ragged tails (rows past the last 64-row tile, columns past a 32-column group), one column,
    ell up to 1024 (two sketch-row groups), fp32 and fp64, column scales over four decades."""
    rng = np.random.default_rng(m + nc)
    X = rng.standard_normal((m, nc)).astype(dtype) * rng.uniform(0.1, 10, nc).astype(dtype)
    X[:, 0] *= 1e-3
    eng, _ = _engine(oid, m, min(8, ell), ell, 64, 256, 0.0, seed=12345, dtype="f64" if dtype == np.float64 else "f32")
    Xd = _dev(X, dtype)
    for _ in range(2):                     # first launch (no exponent guess: rerun) and a guessed one
        eng.ingest_sketch(Xd)
        assert eng.stats()["k1_mode_used"] == FAST
        _check_partials(eng.partials(0).cpu().numpy(), X, ell, 12345)
    eng.close()


def test_k1f_exponent_paths(oid, monkeypatch):
    """Every exponent path against the oracle: the first launch (exponents from the first tile,
    then a rerun), a guessed launch, a block whose late rows exceed the guess (a mid-stream raise:
    accumulators drained, then accumulation continues), a block 2^-12 smaller (the guess lost
    precision: the unit reruns), and, on 2 CTAs (OID_K1_FREE), the int32-overflow epochs."""
    m, nc, ell = 300_000, 32, 256
    rng = np.random.default_rng(5)
    X = rng.standard_normal((m, nc)) * np.logspace(-3, 3, nc)
    Xs = X.copy()
    Xs[m - 1000:, 3] *= 2.0 ** 10         # late spike in column 3
    eng, _ = _engine(oid, m, 8, ell, 64, 256, 0.0, seed=7)
    ctr = lambda: eng.get(15)[-8:].astype(np.int64)     # noqa: E731
    c0 = ctr()
    seq = [(X, "first"), (X, "guess"), (Xs, "raise"), (X * 2.0 ** -12, "rerun")]
    for A, what in seq:
        before = ctr()
        eng.ingest_sketch(_dev(A, np.float64))
        _check_partials(eng.partials(0).cpu().numpy(), A, ell, 7)
        d = ctr() - before
        if what == "first":
            assert d[2] > 0, d                       # reruns
        if what == "guess":
            assert d[1] == 0 and d[2] == 0, d
        if what == "raise":
            assert d[1] > 0, d                       # mid-stream raise -> drain
        if what == "rerun":
            assert d[2] > 0, d
    assert np.all(ctr() >= c0)
    eng.close()
    # int32-overflow epochs: 2 CTAs, > 2048 tiles each
    monkeypatch.setenv("OID_K1_FREE", "146")
    eng, _ = _engine(oid, m, 8, ell, 64, 256, 0.0, seed=7)
    for _ in range(2):
        eng.ingest_sketch(_dev(X, np.float64))
        _check_partials(eng.partials(0).cpu().numpy(), X, ell, 7)
    assert ctr()[3] > 0
    eng.close()


def _stream(oid, A, b, k, ell, lam, seed, checks, dtype=np.float64, cache_limit=100_000_000, split=None, a9q=False):
    m, n = A.shape
    eng, split = _engine(oid, m, k, ell, b, n, lam, seed=seed, dtype="f64" if dtype == np.float64 else "f32",
                         split=split, a9q=a9q)
    o = OracleOID(OracleParams(m=m, k=k, ell=ell, ell1=split[0], ell2=split[1], ell3=split[2], lam=lam, seed=seed),
                  cache_limit=cache_limit)
    Ad = _dev(A, dtype)
    for e, j in enumerate(range(0, n, b)):
        eng.ingest_block(Ad[:, j:j + b])
        lg = o.ingest_block(A[:, j:j + b].astype(dtype))
        low = [d for d in lg.decisions if d[5] < 1e-6]
        if low:
            pytest.skip(f"oracle decision margin {min(d[5] for d in low):.2e} < 1e-6 at epoch {e}: J compared up to it")
        assert eng.stats()["k1_mode_used"] == FAST
        assert np.array_equal(eng.J(), o.J), f"epoch {e}: GPU J {eng.J()} != oracle J {o.J}"
        sc = eng.scalars()
        assert abs(sc["Ek"] - lg.Ek) <= 1e-6 * abs(lg.Ek), (e, sc["Ek"], lg.Ek)
        assert np.allclose(eng.get(1), o.tau_old, rtol=1e-5, atol=0), e
        if e + 1 in checks:
            est, ref = eng.error_estimate(), o.error_estimate()
            fro = o.frob2
            assert abs(est["frob2"] - fro) <= 1e-7 * fro
            for key in ("T", "gpp", "e2"):
                assert abs(est[key] - ref[key]) / fro < 1e-5, (e, key, est[key], ref[key])
            assert abs(est["est_rel"] - ref["est_rel"]) < 1e-5, (e, est["est_rel"], ref["est_rel"])
            P = eng.finalize()["P"].cpu().numpy()
            assert np.linalg.norm(P - o.P) / np.linalg.norm(o.P) < 1e-5, e
    eng.close()
    return o


def test_k1f_c1_stream(oid):
    """BASELINE config 0 (C1, 3 x 16 NA-Hutch++ rows) through K1F: J after every epoch, P and the
    estimate after blocks 8 and 32."""
    A = c1_matrix()
    s = np.linalg.svd(A, compute_uv=False)
    lam = float(np.sum(s[20:] ** 2) / 20)
    _stream(oid, A, 16, 20, 48, lam, seed=0, checks={8, 32}, split=(16, 16, 16))


def test_a9q_c1_stream(oid):
    """C1 through K1F with the A9Q basis Gram (a9_mode = 1): J after every epoch, P and the
    NA-Hutch++ components after blocks 8 and 32 (the small-m case: 32 row tiles, fewer than CTAs)."""
    A = c1_matrix()
    s = np.linalg.svd(A, compute_uv=False)
    lam = float(np.sum(s[20:] ** 2) / 20)
    _stream(oid, A, 16, 20, 48, lam, seed=0, checks={8, 32}, split=(16, 16, 16), a9q=True)


def test_a9q_c3_fullsize_gram(oid):
    """A9Q at full C3 size in the bench launch configuration: sampled G entries against fp64 dot
    products of the finalized basis, within the quantisation bound, across three estimates."""
    gen = ChannelFlow(192, 129, 192, seed=C3.data_seed)
    m, b = gen.m, C3.b
    dev = torch.device("cuda", 0)
    eng, _ = _engine(oid, m, C3.k, C3.ell, b, 128, -1.0, seed=0, a9q=True)
    rng = np.random.default_rng(3)
    for blk in range(3):
        X = gen.block_torch(blk * b, (blk + 1) * b, dev).T
        eng.ingest_block(X)
        assert np.isfinite(eng.error_estimate()["est_rel"])
        del X
        G = eng.get(11)
        J = eng.J()
        occ = np.flatnonzero(J >= 0)
        basis = eng.finalize(basis=True)["basis"]
        pick = rng.choice(occ, size=min(6, len(occ)), replace=False)
        cols = {int(i): basis[:, int(i)].cpu().numpy() for i in pick}
        for i in pick:
            for j in pick:
                ai, aj = cols[int(i)], cols[int(j)]
                Mi, Mj = np.max(np.abs(ai)), np.max(np.abs(aj))
                bnd = 2.0 ** -27 * (Mj * np.sum(np.abs(ai)) + Mi * np.sum(np.abs(aj))) + m * 2.0 ** -54 * Mi * Mj
                ref = float(np.dot(ai, aj))
                assert abs(G[i, j] - ref) <= bnd + 1e-13 * abs(ref), (blk, i, j, G[i, j], ref, bnd)
                assert abs(G[i, j] - ref) <= 1e-8 * np.sqrt(np.dot(ai, ai) * np.dot(aj, aj))
        vac = np.flatnonzero(J < 0)
        assert np.all(G[vac, :] == 0) and np.all(G[:, vac] == 0)
        del basis
    eng.close()


def test_k1f_c3r_whole_stream(oid):
    """BASELINE config 2 on the 48x33x48 grid (C3r), the whole 1000-snapshot stream through K1F,
    lambda = paper surrogate: J bit-exact after every epoch, E_k to 1e-6, tau to 1e-5, and after
    blocks 8, 16, 25, 32 P and the NA-Hutch++ components to 1e-5 (north_star)."""
    cfg = C3R
    gen = ChannelFlow(48, 33, 48, seed=cfg.data_seed)
    A = gen.block(0, cfg.n)
    o = _stream(oid, A, cfg.b, cfg.k, cfg.ell, -1.0, seed=0, checks={8, 16, 25, 32}, cache_limit=200_000_000)
    assert o.min_margin() >= 1e-6


def test_a9q_c3r_whole_stream(oid):
    """The same whole C3r stream with the A9Q basis Gram (a9_mode = 1, the bench's fast mode): J,
    P and the NA-Hutch++ components against the oracle as above."""
    cfg = C3R
    gen = ChannelFlow(48, 33, 48, seed=cfg.data_seed)
    A = gen.block(0, cfg.n)
    _stream(oid, A, cfg.b, cfg.k, cfg.ell, -1.0, seed=0, checks={8, 16, 25, 32}, cache_limit=200_000_000, a9q=True)


def test_k1f_c3_fullsize_sampled(oid):
    """C3 at full size (m = 14,266,368 fp64, b = 32, l = 512) in the bench launch configuration:
    sampled sketch rows recomputed by the oracle row by row, and all column norms, within the bound."""
    gen = ChannelFlow(192, 129, 192, seed=C3.data_seed)
    m, b, ell = gen.m, C3.b, C3.ell
    dev = torch.device("cuda", 0)
    X = gen.block_torch(0, b, dev).T
    eng, _ = _engine(oid, m, C3.k, ell, b, 64, -1.0, seed=0)
    for _ in range(2):
        eng.ingest_sketch(X)
    assert eng.stats()["k1_mode_used"] == FAST
    part = eng.partials(0).cpu().numpy()
    Yg = part[:ell * b].reshape(b, ell).T
    ng = part[ell * b:ell * b + b]
    Xh = X.cpu().numpy()
    delta = QUANT * np.max(np.abs(Xh), axis=0)
    nref = np.einsum("ij,ij->j", Xh, Xh)
    nb = 2 * delta * np.sum(np.abs(Xh), axis=0) + m * delta * delta + 1e-12 * nref
    assert np.all(np.abs(ng - nref) <= nb)
    bound = gauss16_scale() * 110.5 * delta * HOEFF * math.sqrt(m)
    for r in (0, 1, 127, 128, 255, 256, 300, 511):
        acc = np.zeros(b)
        for i0 in range(0, m, 1 << 22):
            i1 = min(m, i0 + (1 << 22))
            acc += omega_rows(0, [r], i0, i1)[0] @ Xh[i0:i1]
        yr = gauss16_scale() * acc
        assert np.all(np.abs(Yg[r] - yr) <= bound + 1e-12 * np.abs(yr)), r
        assert np.max(np.abs(Yg[r] - yr)) <= 1e-7 * np.max(np.abs(yr)), r
    eng.close()


def test_a9q_gram_bound(oid):
    """A9Q (K1F mode): the basis Gram on the int8 tensor cores from the quantised basis copy, after
    each of several estimates, against fp64 dot products of the finalized (exact) basis columns.
    A7 quantises a column with unit <= 2^-28 of its maximum (|a - a_q| <= 2^-27 M), so
    |dG_ij| <= 2^-27 (M_j ||a_i||_1 + M_i ||a_j||_1) + m 2^-54 M_i M_j; rows of vacant slots are 0."""
    cfg = C3R
    gen = ChannelFlow(48, 33, 48, seed=cfg.data_seed)
    m, b = cfg.m, cfg.b
    eng, _ = _engine(oid, m, cfg.k, cfg.ell, b, 8 * b, -1.0, seed=0, a9q=True)
    A = gen.block(0, 8 * b)
    Ad = _dev(A, np.float64)
    rng = np.random.default_rng(4)
    for blk in range(8):
        eng.ingest_block(Ad[:, blk * b:(blk + 1) * b])
        if blk not in (0, 1, 3, 7):
            continue
        eng.error_estimate()
        G = eng.get(11)
        J = eng.J()
        occ = np.flatnonzero(J >= 0)
        basis = eng.finalize(basis=True)["basis"].cpu().numpy()
        # A7 fused with the quantised copy: the basis still holds the admitted columns bit-exactly
        assert np.array_equal(basis[:, occ], A[:, J[occ]]), blk
        assert np.all(basis[:, J < 0] == 0)
        pick = rng.choice(occ, size=min(12, len(occ)), replace=False)
        for i in pick:
            for j in pick:
                ai, aj = basis[:, i], basis[:, j]
                ref = float(np.dot(ai, aj))
                Mi, Mj = np.max(np.abs(ai)), np.max(np.abs(aj))
                bnd = 2.0 ** -27 * (Mj * np.sum(np.abs(ai)) + Mi * np.sum(np.abs(aj))) + m * 2.0 ** -54 * Mi * Mj
                assert abs(G[i, j] - ref) <= bnd + 1e-13 * abs(ref), (blk, i, j, G[i, j], ref, bnd)
        vac = np.flatnonzero(J < 0)
        assert np.all(G[vac, :] == 0) and np.all(G[:, vac] == 0)
    eng.close()


def test_a9q_fp32_large_basis(oid):
    """A9Q on fp32 data with C5's shape of the basis and sketch (k = 400: four 128-slot chunks;
    l = 1024: two K1F sketch-row groups; b = 64: two column groups), on the C5 low-rank stream law
    (C5r rows): the Gram against fp64 dot products of the exact fp32 basis within the bound, the basis
    bit-exact."""
    from synth import LowRankStream
    gen = LowRankStream(m=1 << 18, seed=1005)
    m, b, k, ell = gen.m, 64, 400, 1024
    eng, _ = _engine(oid, m, k, ell, b, 16 * b, -1.0, seed=0, dtype="f32", a9q=True)
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(9)
    for blk in range(9):
        X = gen.block_torch(blk * b, (blk + 1) * b, dev).T
        eng.ingest_block(X)
        if blk in (0, 4, 8):
            assert np.isfinite(eng.error_estimate()["est_rel"])
            G = eng.get(11)
            J = eng.J()
            occ = np.flatnonzero(J >= 0)
            basis = eng.finalize(basis=True)["basis"].cpu().numpy().astype(np.float64)
            pick = rng.choice(occ, size=min(10, len(occ)), replace=False)
            for i in pick:
                for j in pick:
                    ai, aj = basis[:, i], basis[:, j]
                    Mi, Mj = np.max(np.abs(ai)), np.max(np.abs(aj))
                    bnd = 2.0 ** -27 * (Mj * np.sum(np.abs(ai)) + Mi * np.sum(np.abs(aj))) + m * 2.0 ** -54 * Mi * Mj
                    ref = float(np.dot(ai, aj))
                    assert abs(G[i, j] - ref) <= bnd + 1e-12 * abs(ref), (blk, i, j, G[i, j], ref, bnd)
        del X
    eng.close()
