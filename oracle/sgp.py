"""SGP's directed exponential graph as a topology for the same gossip step: the
baseline the paper compares against (Fig. 9 at PAPER.md:300).
Test infrastructure only.

SGP (Assran et al. 2019) uses "model-wise communication and directed exponential
network topology": at round t worker i pushes half of its
(value, weight) to one peer:

    exponential_peer(i, t, n) = (i + 2^(t mod log2 n)) mod n,   n a power of two.

Halving and pushing is the same arithmetic as the merge of Alg. 1 l.17 with
receive-from src(i) = (i - 2^(t mod log2 n)) mod n (reading C-1), so SGP runs
through gossip.gossip_step with this topology and k = 1 (model-wise); with k > 1
every segment uses the same peer.
"""
from __future__ import annotations

import numpy as np


def _log2(n: int) -> int:
    if n < 2 or n & (n - 1):
        raise ValueError("SGP's exponential graph needs a power-of-two world size (SPEC.md:138)")
    return n.bit_length() - 1


def exponential_peer(rank: int, rnd: int, n: int) -> int:
    """the rank worker `rank` sends to at round `rnd`."""
    return (rank + (1 << (rnd % _log2(n)))) % n


def exponential_topology(step: int, n: int, k: int) -> np.ndarray:
    """src[s][i] = the rank worker i receives from at `step` (inverse of exponential_peer)."""
    off = 1 << (step % _log2(n))
    row = [(i - off) % n for i in range(n)]
    return np.array([row] * k, dtype=np.int32)
