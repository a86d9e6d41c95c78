"""Sketch entries Omega(r, i): the Gauss-16 quantised Gaussian (reading R2).

Paper: Omega is a Gaussian random matrix, Omega = randn(l, m);
Hutchinson / NA-Hutch++ need i.i.d. centered entries with mean 0 and variance 1
(P:558); the ridge-leverage sketch needs a JL-type embedding,
which any i.i.d. centered sub-Gaussian law provides.

Reading R2: each entry is drawn from the 16-level equiprobable
discretisation of N(0, 1) by bin centroids.  With Phi the normal CDF and phi its
density, the 8 positive bins [Phi^-1((k+8)/16), Phi^-1((k+9)/16)), k = 0..7, have
centroids c_k = 16 (phi(Phi^-1((k+8)/16)) - phi(Phi^-1((k+9)/16))); the integer
magnitudes are m_k = round(56 c_k - 1/2) = [4, 13, 22, 32, 43, 56, 74, 110] and the
16 levels are +-(m_k + 1/2).  A 4-bit draw n (nibble) maps to
    L(n) = (m_{n & 7} + 1/2) * (1 - 2 (n >> 3)),   Omega(r, i) = s * L(n(r, i)),
    s = 1 / sqrt(mean_n L(n)^2),
so E[Omega] = 0 exactly (L is odd in the sign bit) and E[Omega^2] = 1.  Every
level is an integer plus 1/2 with |L| <= 110.5, which is what lets the GPU path
run the contraction exactly on int8 tensor cores (q = L - 1/2 in [-111, 110]).
Every m_k lies >= 0.19 from a rounding boundary, so any Phi^-1 / phi accurate to
1e-3 gives the same table (pinned by an independent erfc bisection in tests).

The nibble n(r, i) is nibble (i & 7) (bits 4(i & 7) .. 4(i & 7) + 3) of word
((i & 31) >> 3) of the 128-bit Philox block at counter (i >> 5, r, 0, tag=0).

Oracle implementation: Phi^-1 is scipy's ndtri and phi scipy's norm.pdf (library
routines).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""

import numpy as np
from scipy.special import ndtri
from scipy.stats import norm

from .philox import philox4x32_10, seed_key, TAG_OMEGA


def gauss16_magnitudes():
    """int64 m_k, k = 0..7 (reading R2)."""
    k = np.arange(8, dtype=np.float64)
    c = 16.0 * (norm.pdf(ndtri((k + 8) / 16.0)) - norm.pdf(ndtri((k + 9) / 16.0)))
    return np.round(56.0 * c - 0.5).astype(np.int64)


def gauss16_levels():
    """float64 L(n), n = 0..15: half-integers (m_{n&7} + 1/2)(1 - 2 (n >> 3))."""
    m = gauss16_magnitudes().astype(np.float64)
    n = np.arange(16)
    return (m[n & 7] + 0.5) * (1.0 - 2.0 * (n >> 3))


def gauss16_scale():
    """s = 1 / sqrt(mean L^2) in fp64."""
    L = gauss16_levels()
    return 1.0 / np.sqrt(float(np.sum(L * L)) / 16.0)


def omega_nibbles(seed, rows, i0, i1):
    """uint8 array [len(rows), i1 - i0] of the Philox nibbles n(r, i)."""
    rows = np.asarray(rows, dtype=np.int64)
    k0, k1 = seed_key(seed)
    q0, q1 = i0 >> 5, (i1 + 31) >> 5
    blocks = np.arange(q0, q1, dtype=np.int64)
    C0 = np.broadcast_to(blocks[None, :], (rows.size, blocks.size))
    C1 = np.broadcast_to(rows[:, None], (rows.size, blocks.size))
    w = philox4x32_10(C0, C1, 0, TAG_OMEGA, k0, k1)
    words = np.stack(w, axis=-1).astype(np.uint32)                    # [R, B, 4]
    shifts = (4 * np.arange(8, dtype=np.uint32))
    nib = (words[..., None] >> shifts) & np.uint32(0xF)               # [R, B, 4, 8]: entry 8 w + j
    nib = nib.reshape(rows.size, blocks.size * 32).astype(np.uint8)
    off = i0 - q0 * 32
    return nib[:, off:off + (i1 - i0)]


def omega_rows(seed, rows, i0, i1):
    """Unscaled sketch entries L(n(r, i)) (float64 half-integers), rows x [i0, i1).

    Omega = gauss16_scale() * omega_rows(...).
    """
    return gauss16_levels()[omega_nibbles(seed, rows, i0, i1)]
