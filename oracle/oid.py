"""Plain fp64 oracle of the hot path of Algorithm 3 (single-pass randomized ID).

Follows the paper step by step in its notation:
  * sketch s_j = Omega a_j and SS^T += s_j s_j^T          (Alg 3 steps 10-11)
  * ||A_obs||_F^2 += ||a_j||^2                             (Alg 3 step 13)
  * ridge scores tau = (Omega a)^T (SS^T + lam I)^+ (Omega a)
    with lam = (||A_obs||^2 - ||S_k||^2)/k                 (eq:sketch_ridge_leverage_score)
  * tau_i = min(tau_old_i, tau_i) for the basis C          (Alg 3 step 16)
  * eviction with probability 1 - tau_i/tau_old_i          (Alg 3 step 20)
  * admission with probability tau_r^D c (k log k + k log(1/delta)/eps)/t  (Alg 3 step 24)
  * coefficients P = (Omega A_J)^+ (Omega A_obs)           (Alg 4, eq:coeff_rID_fullsketch)
  * optionally (coeff="argmin") Algs 5-7 beside Alg 4 and the per-epoch choice of the candidate
    with the smallest NA-Hutch++ estimate                  (Alg 3 steps 28-32)
  * NA-Hutch++ estimate of ||A_obs - A_J P||_F             (Alg 8, eq:NAhutchPP_expansion P:589,
                                                            eq:NAhutchPP_2nd_term P:595-597)
with the readings R1-R14 of DESIGN.md section 3 (one ingest block = one epoch,
first-success admission, Omega scaling, etc.).  Dense linear algebra uses numpy
/ LAPACK routines (eigh, svd, pinv) as single steps; nothing is blocked, fused
or reordered beyond the formulas.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""

from dataclasses import dataclass, field
import math

import numpy as np

from .philox import uniform24, EVICT
from .gauss16 import gauss16_scale, omega_rows

PINV_RCOND = 1e-12   # reading R9: pseudo-inverse cutoff 1e-12 * max (P:341, P:431 only write "+")


@dataclass
class OracleParams:
    m: int                 # global rows (spatial dimension)
    k: int                 # target rank = basis size t (k = t)
    ell: int               # sketch rows l = k + p
    ell1: int              # NA-Hutch++ row split c1*l, c2*l, c3*l
    ell2: int
    ell3: int
    lam: float             # >= 0: fixed ridge; -1: streaming surrogate; -2: sketch tail (R8)
    eps: float = 0.5
    delta: float = 0.05
    c: float = 1.0         # admission constant c (unset in the paper; R5)
    seed: int = 0
    row_begin: int = 0     # this shard's global row range
    row_end: int = -1
    omega_law: str = "gauss16"   # "gauss16" (reading R2, the build's law) or "gaussian" (the paper's
                                 # randn; numpy draws, for the R2 ablation only - not the GPU's)
    coeff: str = "alg4"          # "alg4": Alg 4 every epoch (the hot path); "argmin": Algs 4-7 and the
                                 # NA-Hutch++ argmin every epoch (NEXT-1)
    epochs: str = "block"        # "block": one ingest block = one epoch (reading R4, the hot path);
                                 # "t": the paper's buffer - an epoch whenever t columns have been
                                 # buffered in D, across block boundaries (NEXT-2)

    @property
    def t(self):
        return self.k

    @property
    def m_loc(self):
        re = self.m if self.row_end < 0 else self.row_end
        return re - self.row_begin

    def admission_factor(self):
        """c (k log k + k log(1/delta)/eps) / t, natural log (reading R5)."""
        k = self.k
        return self.c * (k * math.log(k) + k * math.log(1.0 / self.delta) / self.eps) / self.t


# --------------------------------------------------------------------------- steps

def sketch(params, X, Qcache=None):
    """Y = Omega X for this shard's rows (Alg 3 step 10), unit-variance Omega.

    X: m_loc x ncols, promoted exactly to fp64 (reading R12).  Row chunks are
    accumulated in fp64.  Returns Y (ell x ncols).
    """
    X = np.asarray(X, dtype=np.float64)
    rb = params.row_begin
    m_loc = X.shape[0]
    if params.omega_law == "gaussian":
        return gaussian_omega(params)[:, rb:rb + m_loc] @ X
    acc = np.zeros((params.ell, X.shape[1]))
    chunk = 1 << 16
    for i0 in range(0, m_loc, chunk):
        i1 = min(m_loc, i0 + chunk)
        if Qcache is not None:
            Q = Qcache[:, i0:i1]
        else:
            Q = omega_rows(params.seed, np.arange(params.ell), rb + i0, rb + i1)
        acc += Q @ X[i0:i1]
    return gauss16_scale() * acc


def gaussian_omega(params):
    """Omega = randn(l, m) with unit variance (reading R3), from numpy's PCG64 keyed on the
    seed: the paper's Gaussian sketch for the R2 ablation."""
    key = (params.seed, params.ell, params.m)
    if _GAUSS_CACHE.get("key") != key:
        _GAUSS_CACHE["key"] = key
        _GAUSS_CACHE["Z"] = np.random.default_rng([params.seed, 0x5EED]).standard_normal((params.ell, params.m))
    return _GAUSS_CACHE["Z"]


_GAUSS_CACHE = {}


def column_norms2(X):
    """||a_j||_2^2 (Alg 3 step 13)."""
    X = np.asarray(X, dtype=np.float64)
    return np.einsum("ij,ij->j", X, X)


def eig_gram(gram):
    """Eigen-decomposition of the symmetric l x l Gram SS^T (numpy.linalg.eigh).

    Returns eigenvalues in descending order and matching eigenvectors (columns).
    """
    mu, W = np.linalg.eigh(gram)
    order = np.argsort(-mu, kind="stable")
    return mu[order], W[:, order]


def ridge_lambda(params, mu_desc, frob2, trace_gram):
    """Effective ridge lambda (reading R8).

    lam >= 0: fixed, lam = ||A - A_k||^2/k computed by the caller.
    lam = -1: paper's streaming surrogate (||A_obs||^2 - ||S_k||^2)/k,
              with S = Y/sqrt(l) so ||S_k||^2 = E_k / l (reading R3), clamped >= 0.
    lam = -2: sketch-tail surrogate ||S - S_k||^2 / k = (tr - E_k)/(l k).
    E_k = sum of the k largest eigenvalues of the unscaled Gram YY^T.
    """
    ell, k = params.ell, params.k
    Ek = float(np.sum(mu_desc[:k]))
    if params.lam >= 0:
        return float(params.lam), Ek
    if params.lam == -1:
        return max(0.0, (frob2 - Ek / ell) / k), Ek
    if params.lam == -2:
        return max(0.0, (trace_gram - Ek) / (ell * k)), Ek
    raise ValueError("lam must be >= 0, -1 or -2")


def ridge_scores(mu, W, shift, Ycols):
    """tau(y) = y^T (YY^T + shift I)^+ y via the eigen-decomposition.

    shift = l * lam (reading R3: the paper's S = Y/sqrt(l) with ridge lam equals
    the unscaled Gram with ridge l*lam).  Terms whose denominator mu_i + shift
    is not above 1e-12 * max are dropped (pseudo-inverse, reading R9).
    """
    d = mu + shift
    dmax = float(np.max(d)) if d.size else 0.0
    if dmax <= 0.0:
        return np.zeros(Ycols.shape[1])
    keep = d > PINV_RCOND * dmax
    T = W[:, keep].T @ Ycols
    return np.sum(T * T / d[keep][:, None], axis=0)


def select(seed, epoch, J, tau_old, tau_slot_new, tau_cand, cand_zero, factor, base_index):
    """Alg 3 steps 15-27 with readings R4-R7.

    For slot i = 0..t-1 in order: if occupied, tau_i = min(tau_old_i, tau_i)
    (step 16) and it is evicted when u(e,i,EVICT) < 1 - tau_i/tau_old_i
    (step 20), else tau_old_i = tau_i (step 21).  If (then) vacant, candidates
    r = 0..ncols-1 are scanned in arrival order; the first with
    u(e,i,r) < min(1, tau_r * factor) is admitted (first success, consumed;
    zero columns never admitted).  Returns J, tau_old, admissions [(slot, r)],
    and every evaluated decision with its margin (reading R14).
    """
    J = np.array(J, dtype=np.int64, copy=True)
    tau_old = np.array(tau_old, dtype=np.float64, copy=True)
    ncols = len(tau_cand)
    consumed = np.zeros(ncols, dtype=bool)
    admits, decisions = [], []
    for i in range(J.size):
        if J[i] >= 0:
            tau_i = min(tau_old[i], tau_slot_new[i])
            rho = tau_i / tau_old[i] if tau_old[i] > 0 else 1.0
            p_ev = 1.0 - rho
            u = float(uniform24(seed, epoch, i, EVICT))
            decisions.append(("evict", i, -1, u, p_ev, abs(u - p_ev) / max(rho, 2.0 ** -24)))
            if u < p_ev:
                J[i] = -1
                tau_old[i] = 1.0
            else:
                tau_old[i] = tau_i
        if J[i] < 0:
            for r in range(ncols):
                if consumed[r] or cand_zero[r]:
                    continue
                p_raw = tau_cand[r] * factor
                p = min(1.0, p_raw)
                u = float(uniform24(seed, epoch, i, r))
                decisions.append(("admit", i, r, u, p_raw, abs(u - p_raw) / max(p_raw, 2.0 ** -24)))
                if u < p:
                    J[i] = base_index + r
                    tau_old[i] = tau_cand[r]
                    consumed[r] = True
                    admits.append((i, r))
                    break
    return J, tau_old, admits, decisions


def alg4_coefficients(S_obs, J):
    """Alg 4: P = argmin_X ||Omega A_J X - Omega A_obs||_F = (Omega A_J)^+ (Omega A_obs).

    Min-norm solution through the SVD of S_J with cutoff 1e-12 sigma_max
    (reading R9); rows of vacant slots are zero (reading R10).  Returns
    (P, kappa(S_J) over the kept singular values).
    """
    t = J.size
    n_obs = S_obs.shape[1]
    P = np.zeros((t, n_obs))
    occ = np.nonzero(J >= 0)[0]
    if occ.size == 0:
        return P, 1.0
    SJ = S_obs[:, J[occ]]
    U, sig, Vt = np.linalg.svd(SJ, full_matrices=False)
    if sig[0] <= 0:
        return P, math.inf
    keep = sig > PINV_RCOND * sig[0]
    pinv = (Vt[keep].T / sig[keep]) @ U[:, keep].T
    P[occ] = pinv @ S_obs
    return P, float(sig[0] / sig[keep][-1])


def pinv_psd(G):
    """G^+ of a symmetric positive semi-definite matrix by its eigen-decomposition, eigenvalues
    below 1e-12 * max dropped (reading R9).  Used for the paper's G^-1 (Alg 5)."""
    if G.size == 0:
        return np.zeros_like(G)
    mu, W = np.linalg.eigh(G)
    mmax = float(np.max(mu))
    if mmax <= 0.0:
        return np.zeros_like(G)
    keep = mu > PINV_RCOND * mmax
    return (W[:, keep] / mu[keep]) @ W[:, keep].T


def alg5_coefficients(S_obs, J, G):
    """Alg 5: P = G^-1 Y, G = A_J^T A_J (exact, t x t), Y = (Omega A_J)^T (Omega A_obs)
    "approximates A_J^T A_obs using sketched data".  The paper's Omega there is the JL-scaled
    one (E[Omega^T Omega] = I); S stores the unit-variance Z A (reading R3, E[Z^T Z] = l I), so
    Y = S_J^T S / l.  G^-1 read as the pseudo-inverse of the occupied block (R9); rows of vacant
    slots zero (R10)."""
    t, n_obs = J.size, S_obs.shape[1]
    ell = S_obs.shape[0]
    P = np.zeros((t, n_obs))
    occ = np.nonzero(J >= 0)[0]
    if occ.size == 0:
        return P
    SJ = S_obs[:, J[occ]]
    P[occ] = pinv_psd(G[np.ix_(occ, occ)]) @ ((SJ.T @ S_obs) / ell)
    return P


def sketch_pinv(SJ_full, J):
    """(Omega A_J)^+ (t x l) with R9's cutoff on the singular values, vacant rows zero."""
    t, ell = J.size, SJ_full.shape[0]
    Z = np.zeros((t, ell))
    occ = np.nonzero(J >= 0)[0]
    if occ.size:
        Z[occ] = np.linalg.pinv(SJ_full[:, occ], rcond=PINV_RCOND)
    return Z


def extend_prev(P_prev, Z_prev, S_new):
    """Reading R15: P_prev (t x n_prev, the previous epoch's chosen coefficients) has no columns for
    the epoch's new block; Algs 6 and 7 take them as the new columns' coefficients in the PREVIOUS
    basis, (Omega A_Jprev)^+ (Omega A_new) (Alg 4 with J_prev), so that every candidate covers A_obs."""
    return np.concatenate([P_prev, Z_prev @ S_new], axis=1)


def alg6_coefficients(S_obs, J, J_prev, P_prev_ext):
    """Alg 6: zero the rows of P_prev whose basis column changed
    (eq:coeff_update_residual_zeroout), r_A = Omega A_obs - Omega A_J P_prev,
    dP = argmin_X ||Omega A_J X - r_A|| (the box: the whole Omega A_J, min-norm, R9),
    P = P_prev + dP."""
    t, ell = J.size, S_obs.shape[0]
    Pp = P_prev_ext.copy()
    Pp[J != J_prev] = 0.0
    SJ = np.zeros((ell, t))
    occ = J >= 0
    SJ[:, occ] = S_obs[:, J[occ]]
    r = S_obs - SJ @ Pp
    return Pp + sketch_pinv(SJ, J) @ r


def alg7_coefficients(C, C_prev, J, P_prev_ext):
    """Alg 7: A_J = QR (occupied columns), T = R^+ Q^T A_Jprev (R9 cutoff), P = T P_prev.
    C, C_prev: the basis before / after this epoch's replacements (vacant columns zero)."""
    t = J.size
    T = np.zeros((t, t))
    occ = np.nonzero(J >= 0)[0]
    if occ.size:
        Q, R = np.linalg.qr(C[:, occ])
        T[occ] = np.linalg.pinv(R, rcond=PINV_RCOND) @ (Q.T @ C_prev)
    return T @ P_prev_ext


def hutchpp_estimate(S_obs, SJ, P, G, frob2, ell1, ell2, ell3):
    """Alg 8: NA-Hutch++ estimate of ||A_obs - A_J P||_F^2.

    S_obs: l x n unit-variance sketch Omega A_obs; SJ = Omega A_J (l x t);
    P: t x n; G = A_J^T A_J (t x t, exact); frob2 = ||A_obs||_F^2.
    Row blocks I1, I2, I3 are contiguous (reading R11).  The cross trace
    tr(A (A_J P)^T) follows eq:NAhutchPP_2nd_term literally; the
    expansion eq:NAhutchPP_expansion gives the estimate.
    Returns dict(e2, T, gpp, est_abs, est_rel, negative).
    """
    I1 = slice(0, ell1)
    I2 = slice(ell1, ell1 + ell2)
    I3 = slice(ell1 + ell2, ell1 + ell2 + ell3)
    O1A, O2A, O3A = S_obs[I1], S_obs[I2], S_obs[I3]
    AJP = SJ @ P
    O2AJP, O3AJP = AJP[I2], AJP[I3]
    M = np.linalg.pinv(O1A @ O2AJP.T, rcond=PINV_RCOND)          # (Omega1 A (Omega2 A_J P)^T)^+
    term1 = np.trace(M @ (O1A @ P.T) @ G @ (O2A @ P.T).T)
    if ell3 > 0:
        t3a = np.trace(O3A @ O3AJP.T)
        t3b = np.trace(O3AJP @ O2A.T @ M @ O1A @ O3AJP.T)
        T = term1 + (t3a - t3b) / ell3
    else:
        T = term1
    gpp = np.trace(G @ P @ P.T)                                     # ||A_J P||_F^2
    e2 = frob2 - 2.0 * T + gpp
    est = math.sqrt(max(e2, 0.0))
    return dict(e2=float(e2), T=float(T), gpp=float(gpp), est_abs=est,
                est_rel=est / math.sqrt(frob2) if frob2 > 0 else 0.0, negative=bool(e2 < 0))


# --------------------------------------------------------------------------- driver

@dataclass
class EpochLog:
    epoch: int
    lam_eff: float
    Ek: float
    tau_slot: np.ndarray
    tau_cand: np.ndarray
    J: np.ndarray
    tau_old: np.ndarray
    admits: list
    decisions: list = field(repr=False)
    kappa: float = 1.0
    qstar: int = 4                 # coeff="argmin": the chosen algorithm
    e2q: tuple = ()                # its candidates' unclamped NA-Hutch++ estimates, Algs 4..7


class OracleOID:
    """Step-by-step oracle of Algorithm 3's hot path; one ingest block = one epoch (R4)."""

    def __init__(self, params, cache_omega=True, cache_limit=100_000_000):
        self.p = params
        t, ell = params.t, params.ell
        assert params.ell1 + params.ell2 + params.ell3 == ell
        self.S = np.zeros((ell, 0))
        self.gram = np.zeros((ell, ell))
        self.frob2 = 0.0
        self.n_obs = 0
        self.epoch = 0
        self.J = np.full(t, -1, dtype=np.int64)
        self.tau_old = np.ones(t)
        self.C = np.zeros((params.m_loc, t))                         # basis
        self.P = np.zeros((t, 0))
        self._D = []                                                 # buffered (index, a, s, ||a||^2), epochs="t"
        self.Z = np.zeros((t, ell))                                  # (Omega A_J)^+ of the last epoch
        self.kappa = 1.0
        self.qstar = 4
        self.log = []
        self._Q = None
        if cache_omega and params.omega_law == "gauss16" and ell * params.m_loc <= cache_limit:
            rb = params.row_begin
            self._Q = omega_rows(params.seed, np.arange(ell), rb, rb + params.m_loc)

    def ingest_block(self, X, partial_sketch=None, partial_norms=None):
        """One block.  epochs="block": one epoch over the block's columns (R4); epochs="t": the
        columns are buffered in D and an epoch runs each time D holds t of them.
        Returns the last epoch's log (None if no epoch ran).  partial_sketch/norms: already
        all-reduced [Y; n] (multi-shard runs)."""
        p = self.p
        X = np.asarray(X, dtype=np.float64)
        ncols = X.shape[1]
        Y = sketch(p, X, self._Q) if partial_sketch is None else np.asarray(partial_sketch, np.float64)
        nrm = column_norms2(X) if partial_norms is None else np.asarray(partial_norms, np.float64)
        if p.epochs == "block":
            self._observe(Y, nrm)
            return self._epoch(X, Y, nrm, self.n_obs - ncols)
        last = None
        for c in range(ncols):
            self._observe(Y[:, c:c + 1], nrm[c:c + 1])                # every column sketched and counted
            self._D.append((self.n_obs - 1, X[:, c], Y[:, c], nrm[c]))   # d_count = a_j
            if len(self._D) == p.t:                                    # count = t: epoch
                base = self._D[0][0]
                Xd = np.stack([d[1] for d in self._D], axis=1)
                Yd = np.stack([d[2] for d in self._D], axis=1)
                nd = np.array([d[3] for d in self._D])
                self._D = []
                last = self._epoch(Xd, Yd, nd, base)
        return last

    def _observe(self, Y, nrm):
        self.S = np.concatenate([self.S, Y], axis=1)                  # S <- [S, s_j]
        self.gram = self.gram + Y @ Y.T                               # SS^T += s s^T
        self.frob2 += float(np.sum(nrm))                              # ||A_obs||^2
        self.n_obs += Y.shape[1]

    def _epoch(self, X, Y, nrm, base):
        """Alg 3 steps 15-32 over the candidate columns X (sketches Y, squared norms nrm), whose
        global indices are base, base + 1, ...."""
        p = self.p
        mu, W = eig_gram(self.gram)
        lam_eff, Ek = ridge_lambda(p, mu, self.frob2, float(np.trace(self.gram)))
        shift = p.ell * lam_eff
        occ = self.J >= 0
        tau_slot = np.zeros(p.t)
        if occ.any():
            tau_slot[occ] = ridge_scores(mu, W, shift, self.S[:, self.J[occ]])
        tau_cand = ridge_scores(mu, W, shift, Y)
        cand_zero = nrm == 0.0
        J, tau_old, admits, decisions = select(p.seed, self.epoch, self.J, self.tau_old, tau_slot,
                                               tau_cand, cand_zero, p.admission_factor(), base)
        C_prev, J_prev, P_prev, Z_prev = self.C.copy(), self.J.copy(), self.P, self.Z
        for (i, r) in admits:                                          # c_i = d_r
            self.C[:, i] = X[:, r]
        for i in range(p.t):                                           # evicted and not refilled
            if J[i] < 0:
                self.C[:, i] = 0.0
        self.J, self.tau_old = J, tau_old
        P4, self.kappa = alg4_coefficients(self.S, self.J)            # Alg 4
        SJ = np.zeros((p.ell, p.t))
        SJ[:, J >= 0] = self.S[:, J[J >= 0]]
        self.Z = sketch_pinv(SJ, J)
        qstar, e2q = 4, ()
        if p.coeff == "argmin":
            # Alg 3 steps 28-32: all four candidates, NA-Hutch++ on each, argmin
            G = self.basis_gram()
            Pext = extend_prev(P_prev, Z_prev, self.S[:, P_prev.shape[1]:])
            cands = [P4, alg5_coefficients(self.S, J, G), alg6_coefficients(self.S, J, J_prev, Pext),
                     alg7_coefficients(self.C, C_prev, J, Pext)]
            e2q = tuple(hutchpp_estimate(self.S, SJ, Pq, G, self.frob2, p.ell1, p.ell2, p.ell3)["e2"] for Pq in cands)
            qi = int(np.argmin(e2q))                                   # first minimum: lowest algorithm number
            qstar, self.P = 4 + qi, cands[qi]
        else:
            self.P = P4
        self.qstar = qstar
        self.log.append(EpochLog(self.epoch, lam_eff, Ek, tau_slot, tau_cand, J.copy(), tau_old.copy(),
                                 admits, decisions, self.kappa, qstar, e2q))
        self.epoch += 1
        return self.log[-1]

    def basis_gram(self):
        """G = A_J^T A_J from the stored basis; vacant columns are zero."""
        return self.C.T @ self.C

    def current_P(self):
        """Coefficients of every observed column: the last epoch's P, extended to columns observed
        since by the current basis' sketched LS (Alg 4 with the current J; = S_J^+ S in Alg 4 mode)."""
        return extend_prev(self.P, self.Z, self.S[:, self.P.shape[1]:])

    def error_estimate(self, G=None):
        p = self.p
        SJ = np.zeros((p.ell, p.t))
        occ = self.J >= 0
        SJ[:, occ] = self.S[:, self.J[occ]]
        G = self.basis_gram() if G is None else G
        return hutchpp_estimate(self.S, SJ, self.current_P(), G, self.frob2, p.ell1, p.ell2, p.ell3)

    def min_margin(self):
        return min((d[5] for lg in self.log for d in lg.decisions), default=math.inf)

    def first_low_margin_epoch(self, thresh=1e-6):
        for lg in self.log:
            if any(d[5] < thresh for d in lg.decisions):
                return lg.epoch
        return None
