"""Sketch entries Omega(r, i): the Gauss-256 equiprobable quantized Gaussian.

Paper: Omega is a Gaussian random matrix, Omega = randn(l, m);
Hutchinson / NA-Hutch++ need i.i.d. centered (sub-)Gaussian entries with mean 0
and variance 1.

Reading R2: each entry is drawn from the 256-point equiprobable
quantile discretisation of N(0, 1),
    q(u) = round(44 * Phi^{-1}((u + 1/2) / 256)),  u in {0..255},
    Omega(r, i) = s * q(u(r, i)),  s = 16 / sqrt(sum_u q(u)^2),
so that E[Omega] = 0 exactly (q is odd about u = 127.5) and E[Omega^2] = 1
(s^2 * mean q^2 = 1).  q fits int8 exactly, which is what lets the GPU
contraction run exactly on int8 tensor cores.  The byte u(r, i) is byte
(i & 15) of the 16-byte Philox block at counter (i >> 4, r, 0, tag=0):
little-endian bytes of w0, w1, w2, w3 in that order.

Oracle implementation: Phi^{-1} is scipy's ndtri (a library routine); every
q(u) lies >= 0.006 away from a rounding boundary, so any Phi^{-1} accurate to
1e-4 yields the same table (pinned in tests by an independent erfc bisection).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""

import numpy as np
from scipy.special import ndtri

from .philox import philox4x32_10, seed_key, TAG_OMEGA


def gauss256_table():
    """int64 array q[0..255]."""
    u = np.arange(256, dtype=np.float64)
    return np.round(44.0 * ndtri((u + 0.5) / 256.0)).astype(np.int64)


def gauss256_scale():
    """s = 16 / sqrt(sum q^2) in fp64 (two correctly rounded IEEE ops)."""
    q = gauss256_table()
    return 16.0 / np.sqrt(float(np.sum(q * q)))


def omega_bytes(seed, rows, i0, i1):
    """uint8 array [len(rows), i1 - i0] of the Philox bytes u(r, i)."""
    rows = np.asarray(rows, dtype=np.int64)
    k0, k1 = seed_key(seed)
    q0, q1 = i0 >> 4, (i1 + 15) >> 4
    blocks = np.arange(q0, q1, dtype=np.int64)
    C0 = np.broadcast_to(blocks[None, :], (rows.size, blocks.size))
    C1 = np.broadcast_to(rows[:, None], (rows.size, blocks.size))
    w = philox4x32_10(C0, C1, 0, TAG_OMEGA, k0, k1)
    # bytes in order: w0 b0..b3, w1 b0..b3, w2 ..., w3 ...  -> 16 per block
    words = np.stack(w, axis=-1).astype("<u4")          # [R, B, 4]
    by = words.view(np.uint8).reshape(rows.size, blocks.size * 16)
    off = i0 - q0 * 16
    return by[:, off:off + (i1 - i0)]


def omega_rows(seed, rows, i0, i1):
    """Integer sketch entries q(u(r, i)) (int64), rows x [i0, i1).

    Omega = gauss256_scale() * omega_rows(...).
    """
    q = gauss256_table()
    return q[omega_bytes(seed, rows, i0, i1)]
