"""Pins of the CPU oracle against what the paper and mathematics fix (not against itself).

Each test names the passage it follows.  P:n = PAPER.md line n, S:n = SPEC.md line n.
"""

import itertools
import math
import os

import numpy as np
import pytest

from oracle import philox4x32_10, uniform24, gauss16_magnitudes, gauss16_levels, gauss16_scale, omega_rows
from oracle.gauss16 import omega_nibbles
from oracle.oid import (OracleParams, OracleOID, ridge_scores, ridge_lambda, eig_gram, select,
                        alg4_coefficients, hutchpp_estimate, sketch, alg5_coefficients, alg6_coefficients,
                        alg7_coefficients, extend_prev, sketch_pinv)
from synth import c1_matrix, low_rank_matrix


def _params(m, k, ell, lam, seed=0, split=None, **kw):
    if split is None:
        a, b = ell // 6, ell // 3
        split = (a, b, ell - a - b)
    return OracleParams(m=m, k=k, ell=ell, ell1=split[0], ell2=split[1], ell3=split[2], lam=lam, seed=seed, **kw)


# ------------------------------------------------------------------ Philox (reading R1)

def test_philox_known_answer_vectors(golden_dir):
    rows = [l.split() for l in open(os.path.join(golden_dir, "philox4x32_10_kat.txt")) if l.strip() and not l.startswith("#")]
    assert len(rows) == 6
    for r in rows:
        c0, c1, c2, c3, k0, k1 = (int(x, 16) for x in r[:6])
        want = [int(x, 16) for x in r[6:]]
        got = [int(x) for x in philox4x32_10(c0, c1, c2, c3, k0, k1)]
        assert got == want


def test_uniform24_grid_and_range():
    u = uniform24(12345, np.arange(5000), 3, 7)
    assert np.all(u >= 0) and np.all(u < 1)
    assert np.all(u * 2 ** 24 == np.floor(u * 2 ** 24))
    assert abs(u.mean() - 0.5) < 4 * math.sqrt(1 / 12 / u.size)


def test_uniform24_known_answers_from_curand(golden_dir):
    """Selection draws u(e, i, x) (reading R6: Philox counter (e, i, x, 1), first output word, top 24
    bits) against cuRAND's Philox4x32-10 (tests/golden/uniform24_kat.txt, scripts/golden/uniform24_kat.cu):
    pins the counter layout, the tag and the choice of output word."""
    rows = [l.split() for l in open(os.path.join(golden_dir, "uniform24_kat.txt")) if l.strip() and not l.startswith("#")]
    assert len(rows) >= 8
    for r in rows:
        seed, e, i, x = int(r[0], 16), int(r[1]), int(r[2]), int(r[3], 16)
        w0 = int(r[4], 16)
        u = float(r[8])
        assert u == (w0 >> 8) * 2.0 ** -24
        assert float(uniform24(seed, e, i, x)) == u, (r, float(uniform24(seed, e, i, x)))


# ------------------------------------------------------------------ Gauss-16 (reading R2)

def _inv_norm_bisect(p):
    """Independent inverse normal CDF: bisection on 0.5*erfc(-x/sqrt 2) (stdlib libm)."""
    lo, hi = -10.0, 10.0
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if 0.5 * math.erfc(-mid / math.sqrt(2.0)) < p:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


def _phi(x):
    return math.exp(-0.5 * x * x) / math.sqrt(2.0 * math.pi) if math.isfinite(x) else 0.0


def test_gauss16_table_independent_construction():
    """Bin centroids of the 16 equiprobable N(0,1) bins, rebuilt with stdlib erfc/exp only."""
    want = []
    for k in range(8):
        a = _inv_norm_bisect((k + 8) / 16.0) if k > 0 else 0.0
        b = _inv_norm_bisect((k + 9) / 16.0) if k < 7 else math.inf
        c = 16.0 * (_phi(a) - _phi(b))
        want.append(round(56.0 * c - 0.5))
    assert list(gauss16_magnitudes()) == want == [4, 13, 22, 32, 43, 56, 74, 110]
    L = gauss16_levels()
    assert np.all(L[8:] == -L[:8])                 # odd in the sign bit -> mean exactly 0
    assert np.all(np.diff(L[:8]) > 0) and L[0] > 0
    q = L - 0.5                                     # the integers the tensor cores see
    assert np.all(q == np.round(q)) and q.min() >= -128 and q.max() <= 127


def test_gauss16_unit_variance_and_shape():
    L = gauss16_levels()
    s = gauss16_scale()
    assert abs(s * s * np.mean(L * L) - 1.0) < 4e-16
    z = np.sort(s * L)
    # equiprobable 16-point law: KS distance to N(0,1) ~ 1/32 + centroid offset
    from scipy.stats import norm
    cdf = norm.cdf(z)
    ks = max(np.max(np.abs(np.arange(1, 17) / 16 - cdf)), np.max(np.abs(np.arange(0, 16) / 16 - cdf)))
    assert ks < 0.045
    kurt = np.mean(z ** 4)
    assert 2.5 < kurt < 2.7                          # sub-Gaussian, below the Gaussian 3


def test_omega_nibble_layout_from_kat():
    """Nibble n(r, i) = nibble (i & 7) of word (i & 31) >> 3 of the Philox block (i >> 5, r, 0, 0).

    Checked against the KAT row (c0=1, c1=1, key (2, 1)) of tests/golden: seed 0x100000002,
    sketch row 1, data rows 32..63."""
    nib = omega_nibbles(0x100000002, [1], 32, 64)[0]
    words = [0x4f560ce1, 0xabeeceff, 0x650ea1f9, 0xc098974e]
    want = [(words[i >> 3] >> (4 * (i & 7))) & 15 for i in range(32)]
    assert list(nib) == want


def test_omega_entries_uniform_and_moments():
    Z = omega_rows(7, np.arange(64), 0, 1 << 14) * gauss16_scale()
    n = Z.size
    assert abs(Z.mean()) < 4 / math.sqrt(n)
    assert abs(Z.var() - 1.0) < 4 * math.sqrt(2.0 / n)
    nib = omega_nibbles(7, np.arange(64), 0, 1 << 14)
    counts = np.bincount(nib.ravel(), minlength=16)
    assert np.all(np.abs(counts - n / 16) < 5 * math.sqrt(n / 16))
    # rows independent: empirical correlation of two sketch rows ~ 0
    c = np.corrcoef(Z[0], Z[1])[0, 1]
    assert abs(c) < 4 / math.sqrt(Z.shape[1])


def test_omega_rows_offsets_consistent():
    full = omega_rows(3, np.arange(5), 0, 200)
    part = omega_rows(3, np.arange(5), 37, 133)
    assert np.array_equal(full[:, 37:133], part)


# ------------------------------------------------------------------ sketch

def test_sketch_slab_additivity():
    """Philox is keyed on GLOBAL rows, so shard sketches sum to the full sketch."""
    X = np.random.default_rng(0).standard_normal((1000, 7))
    p = _params(1000, 4, 12, 0.0, seed=9)
    Y = sketch(p, X)
    cut = 377
    p1 = _params(1000, 4, 12, 0.0, seed=9, row_begin=0, row_end=cut)
    p2 = _params(1000, 4, 12, 0.0, seed=9, row_begin=cut, row_end=1000)
    Ys = sketch(p1, X[:cut]) + sketch(p2, X[cut:])
    assert np.allclose(Y, Ys, rtol=1e-13, atol=1e-13)


def test_sketch_identity_mode():
    """Identity sketch (Omega = I, l = m) makes S = A exactly."""
    X = np.random.default_rng(1).standard_normal((40, 5))
    p = _params(40, 4, 40, 0.0)
    Y = sketch(p, X, Qcache=np.eye(40) / gauss16_scale())
    assert np.allclose(Y, X, rtol=1e-15, atol=1e-15)


def test_sketch_jl_norm_statistic():
    """E ||Omega a||^2 = l ||a||^2 for unit-variance i.i.d. entries."""
    rng = np.random.default_rng(2)
    X = rng.standard_normal((2000, 200))
    X /= np.linalg.norm(X, axis=0)
    p = _params(2000, 4, 32, 0.0, seed=5)
    Y = sketch(p, X)
    r = np.sum(Y * Y, axis=0) / 32
    assert abs(r.mean() - 1.0) < 4 * math.sqrt(2 / 32 / 200) + 0.01


def test_gram_and_frob_invariants():
    """SS^T accumulated column block by block equals S S^T; ||A_obs||^2 equals direct sum."""
    A = np.random.default_rng(3).standard_normal((500, 48))
    o = OracleOID(_params(500, 6, 24, 0.0, seed=1))
    for b in range(6):
        o.ingest_block(A[:, 8 * b:8 * b + 8])
    assert np.allclose(o.gram, o.S @ o.S.T, rtol=1e-12, atol=1e-10)
    assert math.isclose(o.frob2, float(np.sum(A * A)), rel_tol=1e-13)
    assert o.n_obs == 48 and o.S.shape == (24, 48)


# ------------------------------------------------------------------ ridge lambda / scores

def test_topk_energy_worked_example():
    """Gram = diag(4, 1), k = 1 -> E_k = 4."""
    mu, W = eig_gram(np.diag([4.0, 1.0]))
    p = _params(2, 1, 2, -2.0, split=(0, 1, 1))
    lam, Ek = ridge_lambda(p, mu, 0.0, 5.0)
    assert Ek == 4.0
    assert lam == pytest.approx((5.0 - 4.0) / (2 * 1))


def test_ridge_surrogate_worked_example():
    """Streaming ridge surrogate lambda_s = (||A_obs||^2 - ||S_k||^2)/k (eq:sketch_ridge_leverage_score,
    P:341) with S = Y/sqrt(l) (reading R3: ||S_k||^2 = E_k/l, E_k the sum of the k largest
    eigenvalues of YY^T), clamped at 0 (R8), and the sketch-tail variant (tr - E_k)/(l k).
    Hand-computed: l = 4, k = 2, eigenvalues (8, 4, 2, 1) -> E_k = 12, E_k/l = 3."""
    mu = np.array([8.0, 4.0, 2.0, 1.0])
    p = _params(100, 2, 4, -1.0, split=(1, 1, 2))
    lam, Ek = ridge_lambda(p, mu, 5.0, 15.0)
    assert Ek == 12.0 and lam == 1.0                     # (5 - 3) / 2
    lam, _ = ridge_lambda(p, mu, 2.0, 15.0)
    assert lam == 0.0                                    # (2 - 3) / 2 < 0, clamped
    p2 = _params(100, 2, 4, -2.0, split=(1, 1, 2))
    lam, _ = ridge_lambda(p2, mu, 5.0, 15.0)
    assert lam == 0.375                                  # (15 - 12) / (4 * 2)
    p0 = _params(100, 2, 4, 0.25, split=(1, 1, 2))
    assert ridge_lambda(p0, mu, 5.0, 15.0)[0] == 0.25    # fixed lambda
    # k >= rank: E_k = trace, so lambda_s = (||A||^2 - tr/l)/k
    p3 = _params(100, 4, 4, -1.0, split=(1, 1, 2))
    assert ridge_lambda(p3, mu, 5.0, 15.0)[0] == (5.0 - 15.0 / 4.0) / 4.0


def test_scores_lambda0_equal_exact_leverage():
    """At lam = 0 and l >= rank(A): sketched scores equal exact leverage ||V(j,:)||^2 and sum to rank."""
    A = low_rank_matrix(11, 300, 80, 7)
    p = _params(300, 4, 20, 0.0, seed=4)
    Y = sketch(p, A)
    mu, W = eig_gram(Y @ Y.T)
    tau = ridge_scores(mu, W, 0.0, Y)
    U, s, Vt = np.linalg.svd(A, full_matrices=False)
    lev = np.sum(Vt[:7] ** 2, axis=0)
    assert np.max(np.abs(tau - lev)) < 1e-9
    assert abs(tau.sum() - 7.0) < 1e-9


def test_scores_closed_form_identity_sketch():
    """Identity sketch: tau_j = sum_q sigma_q^2/(sigma_q^2 + lam) V_jq^2 (eq:ridge-leverage-score)."""
    A = np.random.default_rng(5).standard_normal((30, 12))
    lam = 0.7
    mu, W = eig_gram(A @ A.T)
    tau = ridge_scores(mu, W, lam, A)
    U, s, Vt = np.linalg.svd(A, full_matrices=False)
    want = np.sum((s ** 2 / (s ** 2 + lam))[:, None] * Vt ** 2, axis=0)
    assert np.allclose(tau, want, rtol=1e-11, atol=1e-13)


def test_scores_hand_case(golden_dir):
    """A = I_2, k = 1 -> lam = ||A - A_1||^2/1 = 1, tau = 0.5 each."""
    A = np.eye(2)
    mu, W = eig_gram(A @ A.T)
    tau = ridge_scores(mu, W, 1.0, A)
    assert np.allclose(tau, [0.5, 0.5], atol=1e-15)


def test_scaled_unscaled_equivalence():
    """Reading R3: (Y/sqrt l)^T (YY^T/l + lam I)^-1 (Y/sqrt l) == y^T (YY^T + l lam I)^+ y."""
    rng = np.random.default_rng(6)
    Y = rng.standard_normal((16, 40))
    l, lam = 16, 0.3
    S = Y / math.sqrt(l)
    want = np.sum(S * np.linalg.solve(S @ S.T + lam * np.eye(l), S), axis=0)
    mu, W = eig_gram(Y @ Y.T)
    got = ridge_scores(mu, W, l * lam, Y)
    assert np.allclose(got, want, rtol=1e-11)


def test_lemma1_scores_decrease_when_columns_added():
    """Lemma 1, reading R13: with lam fixed, tau_j([A b]) <= tau_j(A)."""
    rng = np.random.default_rng(7)
    worst = -np.inf
    for _ in range(100):
        m, n = rng.integers(3, 12), rng.integers(1, 10)
        A = rng.standard_normal((m, n))
        b = rng.standard_normal((m, 1)) * rng.uniform(0.1, 3)
        lam = rng.uniform(0.01, 2)
        mu, W = eig_gram(A @ A.T)
        t0 = ridge_scores(mu, W, lam, A)
        Ab = np.hstack([A, b])
        mu, W = eig_gram(Ab @ Ab.T)
        t1 = ridge_scores(mu, W, lam, A)
        worst = max(worst, float(np.max(t1 - t0)))
    assert worst <= 1e-12


# ------------------------------------------------------------------ selection

def test_c1_first_block_forced_admissions():
    """On C1 block 1 every admission probability clamps to 1 (tau f >= 1), so J = 0..15 regardless of u."""
    A = c1_matrix()
    k = 20
    s = np.linalg.svd(A, compute_uv=False)
    lam = float(np.sum(s[k:] ** 2) / k)
    o = OracleOID(_params(4096, 20, 48, lam, split=(16, 16, 16), seed=0))
    lg = o.ingest_block(A[:, :16])
    assert list(lg.J[:16]) == list(range(16)) and np.all(lg.J[16:] == -1)
    assert np.all(lg.tau_cand * o.p.admission_factor() >= 1.0)
    assert np.array_equal(o.C[:, :16], A[:, :16])      # bit-exact copies


def test_no_eviction_when_scores_unchanged():
    """tau_i == tau_old_i gives eviction probability 0."""
    J = np.arange(5)
    tau_old = np.full(5, 0.4)
    for e in range(200):
        J2, t2, adm, _ = select(1, e, J, tau_old, tau_old.copy(), np.array([0.9]), np.array([False]), 2.0, 100)
        assert np.array_equal(J2, J) and not adm


def test_eviction_frequency_matches_probability():
    """Alg 3 step 20: an occupied slot whose score drops from tau_old to tau is evicted with
    probability 1 - tau/tau_old.  Monte Carlo over 4000 epochs (independent draws u(e, i, EVICT)),
    for two score ratios: frequencies within 4 binomial standard errors."""
    for tau_old, tau_new in ((0.8, 0.2), (0.5, 0.45)):
        ev = 0
        trials = 4000
        for e in range(trials):
            J, _, _, _ = select(7, e, np.array([5]), np.array([tau_old]), np.array([tau_new]), np.zeros(0),
                                np.zeros(0, dtype=bool), 1.0, 100)
            ev += J[0] < 0
        p = 1.0 - tau_new / tau_old
        assert abs(ev / trials - p) <= 4 * math.sqrt(p * (1 - p) / trials), (tau_old, tau_new, ev / trials, p)


def test_admission_frequency_matches_probability():
    """a single vacant slot admits with probability min(1, tau f)."""
    trials = 4000
    tau, f = 0.3, 1.0
    hits = 0
    for e in range(trials):
        J2, _, adm, _ = select(77, e, np.array([-1]), np.ones(1), np.zeros(1), np.array([tau]), np.array([False]), f, 0)
        hits += len(adm)
    freq = hits / trials
    assert abs(freq - tau) < 4 * math.sqrt(tau * (1 - tau) / trials)


def test_first_success_and_consumption():
    """Reading R4: first success wins, admitted candidates are consumed, zero columns skipped."""
    J2, t2, adm, _ = select(5, 0, np.full(3, -1), np.ones(3), np.zeros(3),
                            np.array([0.0, 1.0, 1.0, 1.0]), np.array([True, False, False, False]), 10.0, 50)
    assert list(J2) == [51, 52, 53] and adm == [(0, 1), (1, 2), (2, 3)]
    assert list(t2) == [1.0, 1.0, 1.0]


# ------------------------------------------------------------------ Alg 4

def _stream(A, params, b):
    o = OracleOID(params)
    for j in range(0, A.shape[1], b):
        o.ingest_block(A[:, j:j + b])
    return o


def test_alg4_exact_recovery_rank_deficient():
    """Exactly rank-r data, k >= r, l >= r => ||A - A_J P|| / ||A|| <= 1e-12 once rank(A_J) = r."""
    A = low_rank_matrix(21, 200, 60, 5)
    o = _stream(A, _params(200, 8, 24, 0.0, seed=3), 10)
    err = np.linalg.norm(A - o.C @ o.P) / np.linalg.norm(A)
    assert np.linalg.matrix_rank(o.C) == 5
    assert err < 1e-12


def test_alg4_self_representation():
    """With S_J of full column rank, P(:, J_i) = e_i."""
    A = np.random.default_rng(8).standard_normal((150, 40))
    o = _stream(A, _params(150, 6, 20, 0.0, seed=2), 8)
    occ = np.nonzero(o.J >= 0)[0]
    sub = o.P[np.ix_(occ, o.J[occ])]
    assert np.allclose(sub, np.eye(occ.size), atol=1e-12)


def test_alg4_identity_sketch_is_least_squares():
    """Identity sketch: Alg 4 equals the exact LS coefficients argmin ||A_J X - A|| (eq:coeff_ID1)."""
    rng = np.random.default_rng(9)
    A = rng.standard_normal((25, 30))
    J = np.array([3, -1, 7, 12])
    P, _ = alg4_coefficients(A, J)
    X, *_ = np.linalg.lstsq(A[:, [3, 7, 12]], A, rcond=None)
    assert np.allclose(P[[0, 2, 3]], X, atol=1e-12)
    assert np.all(P[1] == 0.0)


# ------------------------------------------------------------------ NA-Hutch++ 

def test_hutchpp_p_zero_gives_frob():
    """P = 0 => estimate^2 == ||A_obs||^2 exactly."""
    rng = np.random.default_rng(10)
    S = rng.standard_normal((24, 30))
    out = hutchpp_estimate(S, rng.standard_normal((24, 5)), np.zeros((5, 30)), np.eye(5), 3.5, 4, 8, 12)
    assert out["e2"] == 3.5 and out["T"] == 0.0


def test_hutchpp_exact_when_reconstruction_exact():
    """A = A_J P exactly => the NA-Hutch++ cross trace equals tr(A (A_J P)^T) (B~ exact when rank <= c1 l)."""
    A = low_rank_matrix(12, 120, 40, 4)
    p = _params(120, 6, 24, 0.0, seed=11, split=(6, 8, 10))
    o = _stream(A, p, 8)
    out = o.error_estimate()
    T_true = float(np.trace(A.T @ (o.C @ o.P)))
    assert abs(out["T"] - T_true) / np.sum(A * A) < 1e-10
    assert abs(out["e2"]) / np.sum(A * A) < 1e-10


def test_hutchpp_unbiased_over_sketch_seeds():
    """NA-Hutch++ is unbiased for tr(A (A_J P)^T) given P: mean over seeds within 3 s.e."""
    rng = np.random.default_rng(13)
    m, n, t, ell = 150, 40, 5, 30
    A = rng.standard_normal((m, n)) @ np.diag(np.linspace(2, 0.2, n))
    J = np.arange(t)
    P = rng.standard_normal((t, n)) * 0.3
    G = A[:, J].T @ A[:, J]
    T_true = float(np.trace(A @ (A[:, J] @ P).T))
    diffs = []
    for seed in range(300):
        p = _params(m, t, ell, 0.0, seed=seed, split=(5, 10, 15))
        S = sketch(p, A)
        out = hutchpp_estimate(S, S[:, J], P, G, float(np.sum(A * A)), 5, 10, 15)
        diffs.append((out["T"] - T_true) / np.sum(A * A))
    d = np.array(diffs)
    assert abs(d.mean()) < 3 * d.std(ddof=1) / math.sqrt(d.size)


def test_hutchpp_unbiased_with_deflation_rank_below_t():
    """NA-Hutch++ with l1 = 2 < t = 16 (split (2, 4, 24)): B = A (A_J P)^T has rank 16 > l1, so the
    low-rank part B~ captures little and the Omega_3 correction (1/l3)[tr(O3 A (O3 A_J P)^T)
    - tr(...)] carries most of tr(B); with P = A_J^+ A (flat spectrum, A_J P the
    projection of A) tr(B) = ||A_J P||_F^2 > 0.  The estimate is unbiased: mean over 400
    sketch seeds within 3 standard errors of the exact trace."""
    rng = np.random.default_rng(23)
    m, n, t, ell = 200, 48, 16, 30
    A = rng.standard_normal((m, n))
    J = np.arange(t)
    P = np.linalg.pinv(A[:, J]) @ A
    G = A[:, J].T @ A[:, J]
    fro = float(np.sum(A * A))
    T_true = float(np.trace(A @ (A[:, J] @ P).T))
    diffs = []
    for seed in range(400):
        p = _params(m, t, ell, 0.0, seed=1000 + seed, split=(2, 4, 24))
        S = sketch(p, A)
        out = hutchpp_estimate(S, S[:, J], P, G, fro, 2, 4, 24)
        diffs.append((out["T"] - T_true) / fro)
    d = np.array(diffs)
    assert abs(d.mean()) < 3 * d.std(ddof=1) / math.sqrt(d.size)


def test_hutchpp_estimate_quality_moderate_error():
    """Error estimates are informative when ||E||^2/||A||^2 >= 1e-2 (S:439 style): |e^ - e|/e <= 0.5 in >= 80% of seeds."""
    rng = np.random.default_rng(14)
    A = low_rank_matrix(15, 300, 60, 6) + 0.3 * rng.standard_normal((300, 60))
    ok = 0
    runs = 20
    for seed in range(runs):
        o = _stream(A, _params(300, 6, 36, -1.0, seed=seed), 12)
        e = np.linalg.norm(A - o.C @ o.P)
        est = o.error_estimate()["est_abs"]
        ok += abs(est - e) / e <= 0.5
    assert ok >= 0.8 * runs


# ------------------------------------------------------------------ whole-run bounds

def test_brute_force_subset_lower_bound():
    """min over all k-subsets of ||A - A_J A_J^+ A|| <= oracle error; truncated SVD error <= that."""
    rng = np.random.default_rng(16)
    A = low_rank_matrix(17, 40, 14, 4) + 0.05 * rng.standard_normal((40, 14))
    o = _stream(A, _params(40, 3, 12, -1.0, seed=1), 7)
    err = np.linalg.norm(A - o.C @ o.P)
    best = min(np.linalg.norm(A - A[:, list(S)] @ np.linalg.pinv(A[:, list(S)]) @ A)
               for S in itertools.combinations(range(14), 3))
    s = np.linalg.svd(A, compute_uv=False)
    assert math.sqrt(np.sum(s[3:] ** 2)) <= best + 1e-12
    assert best <= err + 1e-12


def test_exact_rank_stream_selects_full_rank_basis():
    """rank-5 stream, t = 8 => selected basis has numerical rank 5 in >= 18/20 seeds."""
    good = 0
    for seed in range(20):
        A = low_rank_matrix(100 + seed, 120, 48, 5)
        o = _stream(A, _params(120, 8, 24, -1.0, seed=seed), 8)
        good += np.linalg.matrix_rank(o.C, tol=1e-8 * np.linalg.norm(A)) == 5
    assert good >= 18


# ------------------------------------------------------------------ Algs 5-7 and the argmin (NEXT-1)

def test_alg5_identity_sketch_is_exact_least_squares():
    """Alg 5 with the identity sketch (the JL-scaled Omega = I, i.e. the unit-variance Z = sqrt(l) I
    of reading R3 with l = m, so Y = A_J^T A_obs exactly) is the exact least-squares solution
    A_J^+ A_obs (eq:coeff_ID1), including a vacant slot (R10)."""
    rng = np.random.default_rng(31)
    A = rng.standard_normal((40, 25))
    J = np.array([2, -1, 11, 17, 20])
    occ = J >= 0
    G = np.zeros((5, 5))
    G[np.ix_(occ, occ)] = A[:, J[occ]].T @ A[:, J[occ]]
    P = alg5_coefficients(math.sqrt(40) * A, J, G)
    X, *_ = np.linalg.lstsq(A[:, J[occ]], A, rcond=None)
    assert np.allclose(P[occ], X, atol=1e-11)
    assert np.all(P[~occ] == 0.0)


def test_alg5_differs_from_alg4_under_a_real_sketch():
    """With a genuine (l < m) sketch, Alg 5's exact Gram makes it a different estimator from Alg 4
    (it 'uses both original and sketched column bases'), but it still reproduces the
    basis columns' own coefficients up to the sketch's distortion of A_J^T A_J."""
    p = _params(300, 6, 24, 0.0, seed=4)
    A = np.random.default_rng(32).standard_normal((300, 30))
    S = sketch(p, A)
    J = np.array([1, 4, 9, 15, 22, 28])
    G = A[:, J].T @ A[:, J]
    P4, _ = alg4_coefficients(S, J)
    P5 = alg5_coefficients(S, J, G)
    assert np.linalg.norm(P5 - P4) > 1e-3 * np.linalg.norm(P4)
    # the normal equations of P:468 with the unit-variance sketch: G P5 = S_J^T S / l
    Y = S[:, J].T @ S / 24
    assert np.allclose(G @ P5, Y, rtol=1e-10, atol=1e-9 * np.abs(Y).max())
    # and Y is an unbiased estimate of A_J^T A (E[Z^T Z] = l I): the mean over 200 sketch seeds
    acc = np.zeros((6, 30))
    for s_ in range(100):
        Ss = sketch(_params(300, 6, 24, 0.0, seed=s_), A)
        acc += Ss[:, J].T @ Ss
    Ym = acc / (100 * 24)
    assert np.linalg.norm(Ym - A[:, J].T @ A) < 0.15 * np.linalg.norm(A[:, J].T @ A)


def test_alg6_box_reading_equals_alg4_for_full_rank_sketch():
    """Alg 6 as its box writes it (dP = argmin ||Omega A_J X - r_A|| over the whole Omega A_J):
    P_prev + S_J^+ (S - S_J P_prev) = S_J^+ S when S_J has full column rank, whatever P_prev
    (a sign error in the residual or the zero-out applied to the wrong rows fails)."""
    rng = np.random.default_rng(33)
    S = rng.standard_normal((20, 30))
    J = np.array([0, 5, 9, -1, 14])
    J_prev = np.array([0, 6, 9, 3, -1])
    Pp = rng.standard_normal((5, 30))
    P6 = alg6_coefficients(S, J, J_prev, Pp)
    P4, _ = alg4_coefficients(S, J)
    assert np.allclose(P6, P4, atol=1e-11)


def test_alg6_rank_deficient_keeps_unchanged_prev_rows():
    """Rank-deficient S_J (a duplicated basis column): the min-norm dP leaves the null-space part of
    P_prev, so Alg 6 = Alg 4 + (I - S_J^+ S_J) P_prev(zeroed rows) - the case where it differs."""
    rng = np.random.default_rng(34)
    S = rng.standard_normal((12, 20))
    S[:, 7] = S[:, 3]
    J = np.array([3, 7, 10])
    J_prev = np.array([3, 7, 11])
    Pp = rng.standard_normal((3, 20))
    P6 = alg6_coefficients(S, J, J_prev, Pp)
    P4, _ = alg4_coefficients(S, J)
    Z = sketch_pinv(S[:, J], J)
    Pz = Pp.copy()
    Pz[2] = 0.0                                        # slot 2 changed: its row is zeroed
    assert np.allclose(P6, P4 + (np.eye(3) - Z @ S[:, J]) @ Pz, atol=1e-11)
    assert np.linalg.norm(P6 - P4) > 1e-3


def test_alg7_transform_exact_when_old_basis_in_new_span():
    """Alg 7: A_Jprev = A_J B exactly => T = R^+ Q^T A_Jprev = B, so A_J P7 = A_Jprev P_prev;
    unchanged basis => T = I and P7 = P_prev."""
    rng = np.random.default_rng(35)
    C = rng.standard_normal((50, 4))
    B = rng.standard_normal((4, 4))
    Pp = rng.standard_normal((4, 9))
    J = np.array([1, 2, 3, 4])
    P7 = alg7_coefficients(C, C @ B, J, Pp)
    assert np.allclose(P7, B @ Pp, atol=1e-11)
    assert np.allclose(alg7_coefficients(C, C, J, Pp), Pp, atol=1e-12)


def test_extend_prev_uses_previous_basis_sketch_pinv():
    """Reading R15: the new block's columns of P_prev are (Omega A_Jprev)^+ (Omega A_new)."""
    rng = np.random.default_rng(36)
    S = rng.standard_normal((16, 12))
    Jp = np.array([0, 2, -1, 5])
    Zp = sketch_pinv(S[:, np.maximum(Jp, 0)] * (Jp >= 0), Jp)
    Pprev = rng.standard_normal((4, 8))
    Pe = extend_prev(Pprev, Zp, S[:, 8:])
    assert np.array_equal(Pe[:, :8], Pprev)
    X, *_ = np.linalg.lstsq(S[:, [0, 2, 5]], S[:, 8:], rcond=None)
    assert np.allclose(Pe[[0, 1, 3], 8:], X, atol=1e-11) and np.all(Pe[2, 8:] == 0.0)


def test_argmin_mode_picks_the_smallest_estimate_and_exact_rank_recovers():
    """Alg 3 steps 28-32: every epoch the chosen P is the candidate with the smallest
    unclamped NA-Hutch++ estimate (ties to the lowest algorithm number); on exactly rank-5 data
    with k = 8 the chosen P reconstructs A_obs exactly once the basis has rank 5."""
    A = low_rank_matrix(41, 160, 48, 5)
    p = _params(160, 8, 24, 0.0, seed=5, coeff="argmin")
    o = OracleOID(p)
    for j in range(0, 48, 8):
        lg = o.ingest_block(A[:, j:j + 8])
        assert len(lg.e2q) == 4
        assert lg.qstar == 4 + int(np.argmin(lg.e2q))
    n = o.n_obs
    assert np.linalg.matrix_rank(o.C) == 5
    assert np.linalg.norm(A[:, :n] - o.C @ o.P) / np.linalg.norm(A[:, :n]) < 1e-10


def test_argmin_mode_not_worse_than_alg4_on_c1():
    """On C1-like data (rank 10 + noise) the argmin's chosen P is, at the last epoch, no worse by the
    true error than 1.05x Alg 4's (the estimate is what it minimises; a wrong choice rule - argmax,
    or a stale P_prev - typically fails by far)."""
    A = c1_matrix(seed=43, m=512, n=96, rank=10, noise=1e-3)
    p4 = _params(512, 12, 36, 0.0, seed=6)
    pa = _params(512, 12, 36, 0.0, seed=6, coeff="argmin")
    o4, oa = OracleOID(p4), OracleOID(pa)
    for j in range(0, 96, 12):
        o4.ingest_block(A[:, j:j + 12])
        oa.ingest_block(A[:, j:j + 12])
    assert np.array_equal(o4.J, oa.J)                   # selection does not depend on P
    e4 = np.linalg.norm(A - o4.C @ o4.P)
    ea = np.linalg.norm(A - oa.C @ oa.P)
    assert ea <= 1.05 * e4, (ea, e4, [lg.qstar for lg in oa.log])


# ------------------------------------------------------------------ paper-literal t-column epochs (NEXT-2)

def test_t_epochs_equal_block_epochs_when_b_equals_t():
    """With blocks of exactly t columns the buffer fills once per block: the t-column epochs are the
    block epochs (same J, tau_old, P after every block)."""
    A = c1_matrix(seed=61, m=300, n=48, rank=8, noise=1e-3)
    ob = OracleOID(_params(300, 8, 24, 0.0, seed=3))
    ot = OracleOID(_params(300, 8, 24, 0.0, seed=3, epochs="t"))
    for j in range(0, 48, 8):
        ob.ingest_block(A[:, j:j + 8])
        ot.ingest_block(A[:, j:j + 8])
        # (the Gram is accumulated per column in "t" mode: equal up to rounding)
        assert np.array_equal(ob.J, ot.J) and np.allclose(ob.tau_old, ot.tau_old, rtol=1e-12)
        assert np.allclose(ob.P, ot.P, atol=1e-11)


def test_t_epochs_cross_block_boundaries():
    """t = 8, blocks of 5: an epoch after every 8th column (columns 8, 16, ..., 40 of 42), its
    candidates exactly the 8 buffered columns (global indices [8e, 8e + 8)), even when they span two
    blocks; the 2 leftover columns stay buffered (sketched and counted, no epoch yet)."""
    A = c1_matrix(seed=62, m=300, n=42, rank=8, noise=1e-3)
    o = OracleOID(_params(300, 8, 24, 0.0, seed=4, epochs="t"))
    for j in range(0, 42, 5):
        o.ingest_block(A[:, j:j + 5])
    assert o.epoch == 5 and len(o._D) == 2 and o.n_obs == 42
    assert abs(o.frob2 - np.sum(A * A)) <= 1e-12 * np.sum(A * A)
    for lg in o.log:
        for (_, _, r, *_rest) in [d for d in lg.decisions if d[0] == "admit"]:
            assert 0 <= r < 8
        Jnew = set(lg.J[lg.J >= 0].tolist())
        assert all(0 <= ji < 8 * (lg.epoch + 1) for ji in Jnew)
    # the estimate covers all 42 observed columns (current basis' LS for the 2 buffered ones)
    assert o.current_P().shape == (8, 42)


def test_t_epochs_first_epoch_forced_admissions():
    """the first t columns only fill D; at the first epoch every slot is vacant and the
    first t columns are the candidates (C1 first-block argument with D = the first t columns)."""
    A = c1_matrix(seed=63, m=400, n=20, rank=10, noise=1e-6)
    o = OracleOID(_params(400, 10, 30, 0.0, seed=5, epochs="t"))
    o.ingest_block(A[:, :7])
    assert o.epoch == 0 and np.all(o.J == -1)
    o.ingest_block(A[:, 7:14])
    assert o.epoch == 1
    assert np.all((o.J == -1) | (o.J < 10))
