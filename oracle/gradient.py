"""Plain fp64 oracle of the gradient-enhanced variant (paper section "Enhancing the
randomized ID with estimated gradient information"), with reading Q17:

  * simplex-gradient operators G^p from the 1-ring axis neighbours of each grid node, per field:
    K_q = [x(v_r) - x(v_q)]_r, G^p(q, N_q(k)) = K_q^+(p, k), G^p(q, q) = -sum_k K_q^+(p, k)
    (eq:gradient_estimation_mat);
  * augmented candidate sketch [Omega a; Omega G^1 a; ...; Omega G^d a] for the ridge leverage
    scores (the gradient estimate is concatenated with a_j), energy
    ||a||^2 + sum_p ||G^p a||^2;
  * coefficients P(mu) = argmin ||Omega(A_J X - A)||^2 + mu sum_p ||Omega(G^p A_J X - G^p A)||^2
    (eq:opt_grad_fullsketch), i.e. the stacked least-squares problem;
  * sketched GCV(mu) (eq:GCV_COmega, verbatim including the (Omega G^p Omega^T)^T
    factor) and golden-section search in log10(mu) on [-3, 3] at the end.

Grid and data layout (reading Q17): a snapshot stacks nf fields; field f occupies rows
[f nx ny, (f+1) nx ny) in row-major order (node (i, j) at f nx ny + i ny + j, coordinates
x = i hx, y = j hy); axis neighbours only (2-D: up to 4 per node), spacing h = 1/(N-1) on the
unit square unless given; the gradient weight (the paper's lambda in eq:opt_grad) is called mu.

Dense/sparse linear algebra (pinv, lstsq-free SVD pinv, scipy.sparse products) are single
steps.  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""

import math

import numpy as np
import scipy.sparse as sp

from .oid import (OracleOID, OracleParams, PINV_RCOND, alg4_coefficients, column_norms2, eig_gram, ridge_lambda,
                  ridge_scores, select, sketch, EpochLog)
from .gauss16 import gauss16_scale, omega_rows


def grid_gradient_operators(nf, nx, ny, hx=None, hy=None):
    """[G^1, G^2] (scipy CSR, m x m, m = nf nx ny) of eq:gradient_estimation_mat.

    For node q the 1-ring neighbourhood N_q is its axis neighbours inside the grid; K_q stacks
    x(v_r) - x(v_q) (n_q x 2) and K_q^+ is its Moore-Penrose pseudo-inverse.
    """
    hx = 1.0 / (nx - 1) if hx is None else hx
    hy = 1.0 / (ny - 1) if hy is None else hy
    m = nf * nx * ny
    rows = ([], [])
    cols = ([], [])
    vals = ([], [])
    for f in range(nf):
        base = f * nx * ny
        for i in range(nx):
            for j in range(ny):
                q = base + i * ny + j
                nbr, dx = [], []
                for (di, dj) in ((1, 0), (-1, 0), (0, 1), (0, -1)):
                    ii, jj = i + di, j + dj
                    if 0 <= ii < nx and 0 <= jj < ny:
                        nbr.append(base + ii * ny + jj)
                        dx.append((di * hx, dj * hy))
                K = np.array(dx, dtype=np.float64)             # n_q x 2
                Kp = np.linalg.pinv(K)                          # 2 x n_q
                for p in range(2):
                    for kk, r in enumerate(nbr):
                        rows[p].append(q)
                        cols[p].append(r)
                        vals[p].append(Kp[p, kk])
                    rows[p].append(q)
                    cols[p].append(q)
                    vals[p].append(-float(np.sum(Kp[p])))
    return [sp.csr_matrix((vals[p], (rows[p], cols[p])), shape=(m, m)) for p in range(2)]


def grid_gradient_operators_3d(nf, nx, ny, nz, hx=None, hy=None, hz=None):
    """[G^1, G^2, G^3] (scipy CSR, m x m, m = nf nx ny nz) of eq:gradient_estimation_mat
    on a 3-D grid (NEXT-4: the channel-flow analogue): node (i, j, l) of field f at row
    f nx ny nz + (i ny + j) nz + l, coordinates (i hx, j hy, l hz), 1-ring = the axis neighbours
    (up to 6); K_q stacks x(v_r) - x(v_q) (n_q x 3), K_q^+ its pseudo-inverse."""
    hx = 1.0 / (nx - 1) if hx is None else hx
    hy = 1.0 / (ny - 1) if hy is None else hy
    hz = 1.0 / (nz - 1) if hz is None else hz
    m = nf * nx * ny * nz
    rows, cols, vals = ([], [], []), ([], [], []), ([], [], [])
    steps = ((1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1))
    for f in range(nf):
        base = f * nx * ny * nz
        for i in range(nx):
            for j in range(ny):
                for l in range(nz):
                    q = base + (i * ny + j) * nz + l
                    nbr, dx = [], []
                    for (di, dj, dl) in steps:
                        ii, jj, ll = i + di, j + dj, l + dl
                        if 0 <= ii < nx and 0 <= jj < ny and 0 <= ll < nz:
                            nbr.append(base + (ii * ny + jj) * nz + ll)
                            dx.append((di * hx, dj * hy, dl * hz))
                    Kp = np.linalg.pinv(np.array(dx, dtype=np.float64))     # 3 x n_q
                    for p in range(3):
                        for kk, r in enumerate(nbr):
                            rows[p].append(q)
                            cols[p].append(r)
                            vals[p].append(Kp[p, kk])
                        rows[p].append(q)
                        cols[p].append(q)
                        vals[p].append(-float(np.sum(Kp[p])))
    return [sp.csr_matrix((vals[p], (rows[p], cols[p])), shape=(m, m)) for p in range(3)]


def stacked_coefficients(S, Sg, J, mu):
    """P(mu) of eq:opt_grad_fullsketch: the minimiser of
    ||S_J X - S||^2 + mu sum_p ||S^p_J X - S^p||^2 with S = Omega A_obs, S^p = Omega G^p A_obs,
    i.e. X = [S_J; sqrt(mu) S^1_J; ...]^+ [S; sqrt(mu) S^1; ...] (min-norm, R9 cutoff).
    Rows of vacant slots are zero (R10)."""
    t = J.size
    P = np.zeros((t, S.shape[1]))
    occ = np.nonzero(J >= 0)[0]
    if occ.size == 0:
        return P
    r = math.sqrt(mu)
    lhs = np.vstack([S[:, J[occ]]] + [r * Sp[:, J[occ]] for Sp in Sg])
    rhs = np.vstack([S] + [r * Sp for Sp in Sg])
    P[occ] = np.linalg.pinv(lhs, rcond=PINV_RCOND) @ rhs
    return P


def gcv(S, Sg, SJ, SgJ, OGO, mu):
    """Sketched GCV(mu) of eq:GCV_COmega, verbatim:
    C(mu) = Omega A_J ((Omega A_J)^T Omega A_J + mu sum_p (Omega G^p A_J)^T Omega G^p A_J)^{-1}
            (Omega A_J + mu sum_p (Omega G^p Omega^T)^T Omega G^p A_J)^T,
    GCV = ||(I - C) Omega A||_F^2 / tr(I - C)^2.  SJ, SgJ: occupied columns only; OGO[p] =
    Omega G^p Omega^T (l x l).  The inverse is the R9 pseudo-inverse."""
    H = SJ.T @ SJ + mu * sum(SpJ.T @ SpJ for SpJ in SgJ)
    R = SJ + mu * sum(OGO[p].T @ SgJ[p] for p in range(len(SgJ)))
    C = SJ @ np.linalg.pinv(H, rcond=PINV_RCOND) @ R.T
    ell = S.shape[0]
    E = (np.eye(ell) - C) @ S
    return float(np.sum(E * E) / np.trace(np.eye(ell) - C) ** 2)


def golden_section(f, a, b, tol=1e-3):
    """Golden-section search for a minimum of a unimodal f on [a, b] (Kiefer 1953);
    stops when the bracket is shorter than tol; returns the midpoint of the final bracket."""
    invphi = (math.sqrt(5.0) - 1.0) / 2.0
    c = b - invphi * (b - a)
    d = a + invphi * (b - a)
    fc, fd = f(c), f(d)
    while b - a > tol:
        if fc < fd:
            b, d, fd = d, c, fc
            c = b - invphi * (b - a)
            fc = f(c)
        else:
            a, c, fc = c, d, fd
            d = a + invphi * (b - a)
            fd = f(d)
    return 0.5 * (a + b)


class OracleGradOID(OracleOID):
    """Algorithm 3 with the gradient-augmented scores (A11); one ingest block = one epoch (R4).
    Gops: [G^1, ..., G^d] for this shard's rows (full-rank-space operators on the local rows)."""

    def __init__(self, params, Gops, cache_omega=True):
        super().__init__(params, cache_omega)
        self.G = Gops
        d = len(Gops)
        self.Sg = [np.zeros((params.ell, 0)) for _ in range(d)]
        self.gram = np.zeros(((d + 1) * params.ell, (d + 1) * params.ell))
        self.frob2_aug = 0.0       # ||A_obs||^2 + sum_p ||G^p A_obs||^2 (augmented energy, A11(2))

    def ingest_block(self, X, partial_sketch=None, partial_norms=None):
        p = self.p
        X = np.asarray(X, dtype=np.float64)
        ncols = X.shape[1]
        GX = [Gp @ X for Gp in self.G]                                  # G^p a_j
        Y = sketch(p, X, self._Q)
        Yg = [sketch(p, g, self._Q) for g in GX]
        Yaug = np.vstack([Y] + Yg)                                      # [Omega a; Omega G^p a]
        nrm = column_norms2(X)
        nrm_aug = nrm + sum(column_norms2(g) for g in GX)               # augmented energy
        base = self.n_obs
        self.S = np.concatenate([self.S, Y], axis=1)
        self.Sg = [np.concatenate([Sp, Yp], axis=1) for Sp, Yp in zip(self.Sg, Yg)]
        self.gram = self.gram + Yaug @ Yaug.T
        self.frob2 += float(np.sum(nrm))                                 # plain energy (estimates)
        self.frob2_aug += float(np.sum(nrm_aug))
        self.n_obs += ncols
        mu, W = eig_gram(self.gram)
        lam_eff, Ek = ridge_lambda(p, mu, self.frob2_aug, float(np.trace(self.gram)))
        shift = p.ell * lam_eff
        Saug = np.vstack([self.S] + self.Sg)
        occ = self.J >= 0
        tau_slot = np.zeros(p.t)
        if occ.any():
            tau_slot[occ] = ridge_scores(mu, W, shift, Saug[:, self.J[occ]])
        tau_cand = ridge_scores(mu, W, shift, Yaug)
        cand_zero = nrm == 0.0
        J, tau_old, admits, decisions = select(p.seed, self.epoch, self.J, self.tau_old, tau_slot,
                                               tau_cand, cand_zero, p.admission_factor(), base)
        for (i, r) in admits:
            self.C[:, i] = X[:, r]
        for i in range(p.t):
            if J[i] < 0:
                self.C[:, i] = 0.0
        self.J, self.tau_old = J, tau_old
        self.P, self.kappa = alg4_coefficients(self.S, self.J)        # plain Alg 4 (estimates)
        self.log.append(EpochLog(self.epoch, lam_eff, Ek, tau_slot, tau_cand, J.copy(), tau_old.copy(),
                                 admits, decisions, self.kappa))
        self.epoch += 1
        return self.log[-1]

    def coefficients(self, mu):
        return stacked_coefficients(self.S, self.Sg, self.J, mu)

    def omega_g_omega(self):
        """Omega G^p Omega^T (l x l) for each p, unit-variance Omega (needs the cached Omega)."""
        s = gauss16_scale()
        Om = s * (self._Q if self._Q is not None else
                  omega_rows(self.p.seed, np.arange(self.p.ell), self.p.row_begin, self.p.row_begin + self.p.m_loc))
        return [Om @ (Gp @ Om.T) for Gp in self.G]

    def gcv(self, mu, OGO=None):
        occ = np.nonzero(self.J >= 0)[0]
        OGO = self.omega_g_omega() if OGO is None else OGO
        SJ = self.S[:, self.J[occ]]
        SgJ = [Sp[:, self.J[occ]] for Sp in self.Sg]
        return gcv(self.S, self.Sg, SJ, SgJ, OGO, mu)

    def finalize(self, lo=-3.0, hi=3.0, tol=1e-3):
        """mu* = 10^argmin GCV by golden section on log10 mu in [lo, hi]; P(mu*)."""
        OGO = self.omega_g_omega()
        x = golden_section(lambda lm: self.gcv(10.0 ** lm, OGO), lo, hi, tol)
        mu_star = 10.0 ** x
        self.P = self.coefficients(mu_star)
        return mu_star, self.P
