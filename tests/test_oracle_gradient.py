"""Pins of the gradient-variant oracle (oracle/gradient.py, paper P:625-719) against
what the mathematics fixes, not against the oracle's own formulas."""

import math

import numpy as np
import pytest

from oracle import OracleParams
from oracle.oid import alg4_coefficients
from oracle.gradient import grid_gradient_operators, stacked_coefficients, gcv, golden_section, OracleGradOID


def _coords(nx, ny, hx, hy):
    i, j = np.meshgrid(np.arange(nx), np.arange(ny), indexing="ij")
    return (i * hx).ravel(), (j * hy).ravel()


def test_linear_fields_exact_gradient_everywhere():
    """Least squares on exact linear data returns the exact gradient at every node, boundary and
    corner nodes included (K_q has full column rank there)."""
    nf, nx, ny = 2, 7, 5
    hx, hy = 1.0 / (nx - 1), 1.0 / (ny - 1)
    G1, G2 = grid_gradient_operators(nf, nx, ny)
    x, y = _coords(nx, ny, hx, hy)
    a = np.concatenate([3.0 * x - 2.0 * y + 0.5, -1.25 * x + 4.0 * y - 7.0])
    g1, g2 = G1 @ a, G2 @ a
    np.testing.assert_allclose(g1[: nx * ny], 3.0, rtol=0, atol=1e-12)
    np.testing.assert_allclose(g2[: nx * ny], -2.0, rtol=0, atol=1e-12)
    np.testing.assert_allclose(g1[nx * ny:], -1.25, rtol=0, atol=1e-12)
    np.testing.assert_allclose(g2[nx * ny:], 4.0, rtol=0, atol=1e-12)


def test_stencils_central_interior_one_sided_boundary():
    """Interior rows are the central difference (+-1/(2h)); an x-boundary node's x-row is the
    one-sided difference (+-1/h); constants have zero gradient (rows sum to zero)."""
    nx, ny = 6, 6
    h = 1.0 / (nx - 1)
    G1, G2 = grid_gradient_operators(1, nx, ny)
    q = 2 * ny + 3                                     # interior node (2, 3)
    row = G1.getrow(q).toarray().ravel()
    assert row[3 * ny + 3] == pytest.approx(1 / (2 * h)) and row[1 * ny + 3] == pytest.approx(-1 / (2 * h))
    assert abs(row[q]) < 1e-12 and np.count_nonzero(np.abs(row) > 1e-12) == 2
    q0 = 0 * ny + 3                                    # x = 0 boundary node
    row0 = G1.getrow(q0).toarray().ravel()
    assert row0[1 * ny + 3] == pytest.approx(1 / h) and row0[q0] == pytest.approx(-1 / h)
    ones = np.ones(nx * ny)
    assert np.max(np.abs(G1 @ ones)) < 1e-12 and np.max(np.abs(G2 @ ones)) < 1e-12


def test_stacked_coefficients_mu0_is_alg4_and_normal_equations():
    rng = np.random.default_rng(3)
    ell, n, t = 20, 30, 6
    S = rng.standard_normal((ell, n))
    Sg = [rng.standard_normal((ell, n)), rng.standard_normal((ell, n))]
    J = np.array([4, -1, 11, 0, 23, 7])
    P0 = stacked_coefficients(S, Sg, J, 0.0)
    Pa, _ = alg4_coefficients(S, J)
    np.testing.assert_allclose(P0, Pa, rtol=1e-12, atol=1e-12)
    mu = 0.7
    P = stacked_coefficients(S, Sg, J, mu)
    occ = J >= 0
    # normal equations of min ||S_J X - S||^2 + mu sum ||S^p_J X - S^p||^2
    lhs = S[:, J[occ]].T @ (S[:, J[occ]] @ P[occ] - S)
    lhs += mu * sum(Sp[:, J[occ]].T @ (Sp[:, J[occ]] @ P[occ] - Sp) for Sp in Sg)
    assert np.max(np.abs(lhs)) < 1e-9 * np.max(np.abs(S)) ** 2
    assert np.all(P[~occ] == 0)


def test_gcv_mu0_closed_form():
    """At mu = 0, C(0) is the orthogonal projector onto range(S_J): GCV(0) = ||(I - Pi) S||^2 / (l - t)^2."""
    rng = np.random.default_rng(4)
    ell, n, t = 16, 40, 5
    S = rng.standard_normal((ell, n))
    SJ = S[:, :t]
    Sg = [rng.standard_normal((ell, n))]
    SgJ = [Sg[0][:, :t]]
    OGO = [rng.standard_normal((ell, ell))]
    Q, _ = np.linalg.qr(SJ)
    E = S - Q @ (Q.T @ S)
    want = np.sum(E * E) / (ell - t) ** 2
    assert gcv(S, Sg, SJ, SgJ, OGO, 0.0) == pytest.approx(want, rel=1e-10)


def test_golden_section_finds_minimum():
    f = lambda x: (x - 0.8137) ** 2 + 3.0
    assert golden_section(f, -3.0, 3.0, tol=1e-6) == pytest.approx(0.8137, abs=1e-5)
    assert golden_section(lambda x: abs(x + 2.5), -3.0, 3.0, tol=1e-6) == pytest.approx(-2.5, abs=1e-5)


def test_constant_fields_reduce_to_plain_scores():
    """Columns that are constant on each field have zero simplex gradients, so the augmented
    sketches add nothing: the selection equals the plain Algorithm 3 oracle's."""
    from oracle import OracleOID
    nf, nx, ny = 2, 6, 5
    m = nf * nx * ny
    rng = np.random.default_rng(5)
    A = np.repeat(rng.standard_normal((nf, 24)), nx * ny, axis=0)   # field-wise constant columns
    prm = OracleParams(m=m, k=3, ell=8, ell1=2, ell2=3, ell3=3, lam=0.1, seed=9)
    og = OracleGradOID(prm, grid_gradient_operators(nf, nx, ny))
    o = OracleOID(prm)
    for j in range(0, 24, 8):
        og.ingest_block(A[:, j:j + 8])
        o.ingest_block(A[:, j:j + 8])
        assert np.array_equal(og.J, o.J)


def test_gradient_variant_end_to_end_small():
    """Smooth fields: the gradient-aware coefficients at mu* reconstruct gradients at least as
    well as the mu = 0 coefficients (the purpose of the variant), and mu* lies in
    [1e-3, 1e3]."""
    nf, nx, ny = 1, 12, 10
    m = nf * nx * ny
    x, y = _coords(nx, ny, 1 / (nx - 1), 1 / (ny - 1))
    rng = np.random.default_rng(6)
    cols = []
    for s in range(40):
        a, b, c = rng.standard_normal(3)
        cols.append(np.sin(3 * x + a) * np.cos(2 * y + b) + 0.2 * c * x * y + 1e-3 * rng.standard_normal(m))
    A = np.stack(cols, axis=1)
    Gs = grid_gradient_operators(nf, nx, ny)
    prm = OracleParams(m=m, k=8, ell=24, ell1=6, ell2=8, ell3=10, lam=-1.0, seed=2)
    og = OracleGradOID(prm, Gs)
    for j in range(0, 40, 8):
        og.ingest_block(A[:, j:j + 8])
    mu_star, P = og.finalize()
    assert 1e-3 * 0.99 <= mu_star <= 1e3 * 1.01
    occ = og.J >= 0
    AJ = A[:, og.J[occ]]
    P0 = og.coefficients(0.0)
    def grad_err(PP):
        return sum(np.linalg.norm(G @ (AJ @ PP[occ]) - G @ A) for G in Gs)
    assert grad_err(P) <= grad_err(P0) * (1 + 1e-9)


def test_3d_gradient_operators_exact_on_linear_fields():
    """NEXT-4: the 3-D simplex gradients of a linear field a x + b y + c z are exact at every node
    (interior central differences, one-sided at faces, edges and corners), per field, and every
    row sums to zero."""
    from oracle.gradient import grid_gradient_operators_3d
    nf, nx, ny, nz = 2, 5, 4, 3
    G = grid_gradient_operators_3d(nf, nx, ny, nz)
    hx, hy, hz = 1 / (nx - 1), 1 / (ny - 1), 1 / (nz - 1)
    i, j, l = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    x, y, z = (i * hx).ravel(), (j * hy).ravel(), (l * hz).ravel()
    coef = [(0.7, -1.3, 2.1), (-0.2, 0.5, -3.0)]
    a = np.concatenate([c[0] * x + c[1] * y + c[2] * z + 4.0 for c in coef])
    for p in range(3):
        g = G[p] @ a
        want = np.concatenate([np.full(x.size, c[p]) for c in coef])
        assert np.allclose(g, want, atol=1e-12)
        assert np.allclose(np.asarray(G[p].sum(axis=1)).ravel(), 0.0, atol=1e-12)
    # the 2-D operators are the nz = 1 slice of the same construction
    from oracle.gradient import grid_gradient_operators
    G2 = grid_gradient_operators(1, nx, ny)
    G3 = grid_gradient_operators_3d(1, nx, ny, 2, hz=1.0)
    b = np.random.default_rng(0).standard_normal(nx * ny)
    b3 = np.repeat(b, 2)                      # constant along z: l = 0, 1 hold the same values
    for p in range(2):
        assert np.allclose((G3[p] @ b3)[::2], G2[p] @ b, atol=1e-12)
