"""Philox4x32-10 (Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as easy
as 1, 2, 3", SC'11), written out from its definition.  Test infrastructure only.

The paper draws destinations with `choice(world_size, roulette=..., seed=rseed)`
(§3.2 Alg. 2 l.7).  Reading C-4: draws are
counter-based, keyed by the shared seed and indexed by (step, segment, attempt,
rank, domain tag), so every process computes the same topology with no
communication ("rseed: random seed which is shared by every process",
PAPER.md:127).

Pinned by the Random123 known-answer vectors (tests/golden/philox4x32_10_kat.txt).
"""
from __future__ import annotations

import numpy as np

M0 = 0xD2511F53
M1 = 0xCD9E8D57
W0 = 0x9E3779B9
W1 = 0xBB67AE85
MASK32 = 0xFFFFFFFF


def philox4x32_10(ctr, key):
    """One block: ctr = 4 uint32 words, key = 2 uint32 words -> 4 uint32 words.

    Round (Salmon et al. §4.2): (hi0,lo0) = M0*c0, (hi1,lo1) = M1*c2,
    c' = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0); the key is bumped by the
    Weyl constants (W0, W1) between rounds; 10 rounds.
    """
    c0, c1, c2, c3 = (int(v) & MASK32 for v in ctr)
    k0, k1 = (int(v) & MASK32 for v in key)
    for r in range(10):
        if r > 0:
            k0 = (k0 + W0) & MASK32
            k1 = (k1 + W1) & MASK32
        p0 = M0 * c0
        p1 = M1 * c2
        hi0, lo0 = p0 >> 32, p0 & MASK32
        hi1, lo1 = p1 >> 32, p1 & MASK32
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
    return (c0, c1, c2, c3)


def philox4x32_10_np(c0, c1, c2, c3, k0, k1):
    """Vectorised form of `philox4x32_10` over numpy arrays of counters (same arithmetic)."""
    m32 = np.uint64(MASK32)
    c0, c1, c2, c3 = (np.asarray(v, dtype=np.uint64) & m32 for v in (c0, c1, c2, c3))
    k0 = np.uint64(int(k0) & MASK32)
    k1 = np.uint64(int(k1) & MASK32)
    for r in range(10):
        if r > 0:
            k0 = np.uint64((int(k0) + W0) & MASK32)
            k1 = np.uint64((int(k1) + W1) & MASK32)
        p0 = np.uint64(M0) * c0
        p1 = np.uint64(M1) * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & m32
        hi1, lo1 = p1 >> np.uint64(32), p1 & m32
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
    return c0, c1, c2, c3
