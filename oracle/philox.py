"""Philox4x32-10 counter-based generator, plain numpy (oracle side).

The paper only says Omega = randn(l, m) and that the Hutchinson probes
are i.i.d. mean-0 variance-1; it names no generator.  Reading R1
(DESIGN.md): every random number of the method comes from Philox4x32-10
(Salmon et al., SC'11) with key = (seed & 0xffffffff, seed >> 32) and a
counter whose 4th word is a stream tag (0 = sketch entries, 1 = selection
draws).  Being counter-based, any entry can be regenerated independently,
which is what lets the oracle and the GPU path reproduce the same stream
without sharing code.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""

import numpy as np

_M0 = np.uint64(0xD2511F53)
_M1 = np.uint64(0xCD9E8D57)
_W0 = np.uint64(0x9E3779B9)
_W1 = np.uint64(0xBB67AE85)
_MASK = np.uint64(0xFFFFFFFF)
_SH = np.uint64(32)


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Ten Philox rounds on broadcastable uint32 arrays; returns 4 uint32 arrays.

    One round: (hi0, lo0) = M0*c0, (hi1, lo1) = M1*c2,
    c' = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0); then the key is bumped by
    the Weyl constants (W0, W1).
    """
    c0, c1, c2, c3 = (np.asarray(x, dtype=np.uint64) & _MASK for x in (c0, c1, c2, c3))
    k0 = np.asarray(k0, dtype=np.uint64) & _MASK
    k1 = np.asarray(k1, dtype=np.uint64) & _MASK
    for _ in range(10):
        p0 = _M0 * c0
        p1 = _M1 * c2
        hi0, lo0 = p0 >> _SH, p0 & _MASK
        hi1, lo1 = p1 >> _SH, p1 & _MASK
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
        k0 = (k0 + _W0) & _MASK
        k1 = (k1 + _W1) & _MASK
    return tuple(x.astype(np.uint32) for x in (c0, c1, c2, c3))


def seed_key(seed):
    seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    return seed & 0xFFFFFFFF, seed >> 32


TAG_OMEGA = 0
TAG_SELECT = 1
EVICT = 0xFFFFFFFF


def uniform24(seed, epoch, slot, x):
    """Selection draw u(e, i, x) in [0, 1) on a 2^-24 grid (reading R6).

    Counter = (epoch, slot, x, tag=1); u = (w0 >> 8) * 2^-24, exact in fp64.
    x = 0xffffffff for the eviction draw of slot i, x = r for the admission
    draw of candidate r (0-based position in the current block).
    """
    k0, k1 = seed_key(seed)
    w0, _, _, _ = philox4x32_10(epoch, slot, x, TAG_SELECT, k0, k1)
    return (np.asarray(w0, dtype=np.uint64) >> np.uint64(8)).astype(np.float64) * 2.0 ** -24
