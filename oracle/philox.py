"""Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11 "Parallel random numbers: as easy as
1, 2, 3"), the counter-based generator north_star names for the relabel sampler.  The
paper itself is silent on the RNG (reading A-18).

Pinned in tests/test_oracle_philox.py by the Random123 known-answer vectors
(tests/golden/philox_kat.txt).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
import numpy as np

M0 = 0xD2511F53
M1 = 0xCD9E8D57
W0 = 0x9E3779B9
W1 = 0xBB67AE85
MASK32 = 0xFFFFFFFF


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """One Philox4x32-10 block per element.

    Arguments are integers or uint64 numpy arrays holding 32-bit values (broadcastable).
    Round (applied 10 times, key bumped by (W0, W1) between rounds):
        (c0,c1,c2,c3) -> (hi(M1*c2) ^ c1 ^ k0, lo(M1*c2), hi(M0*c0) ^ c3 ^ k1, lo(M0*c0))
    Returns (x0, x1, x2, x3) as uint64 arrays of 32-bit values.
    """
    u = np.uint64
    c0, c1, c2, c3 = (np.asarray(x, dtype=u) & u(MASK32) for x in (c0, c1, c2, c3))
    k0 = np.asarray(k0, dtype=u) & u(MASK32)
    k1 = np.asarray(k1, dtype=u) & u(MASK32)
    for r in range(10):
        if r > 0:
            k0 = (k0 + u(W0)) & u(MASK32)
            k1 = (k1 + u(W1)) & u(MASK32)
        p0 = u(M0) * c0          # < 2^64, exact in uint64
        p1 = u(M1) * c2
        hi0, lo0 = p0 >> u(32), p0 & u(MASK32)
        hi1, lo1 = p1 >> u(32), p1 & u(MASK32)
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
    return c0, c1, c2, c3
