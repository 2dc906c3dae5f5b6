"""Load-balanced random topology (§3.2, Algorithm 2) and the
segment plan.  Test infrastructure only.

Algorithm 2 as printed:
    for i in world_size:
        for j in dest_list: roulettes[i][j] = 0          (l.2-4)
        roulettes[i] /= sum(roulettes[i])                 (l.5-6)
        selected_rank = choice(world_size, roulette=roulettes[i], seed=rseed)  (l.7)
        dest_list.append(selected_rank)                   (l.8)
with the initial roulettes "a stochastic matrix with its major diagonal elements
having zero value".

Readings:
  C-1  dest_list[i] is the rank that i RECEIVES segment s from
       (Alg.1 l.5 "receive_from = destinations[my rank]").
  C-4  `choice(..., seed=rseed)` = one counter-based Philox draw per (step,
       segment, attempt, rank, domain tag).
  C-5  the shared roulettes table is copied per call (l.3 mutates it).
  C-6  dead end (only rank i itself left, row sum 0) -> discard, restart with
       attempt+1; give up after 10,000 attempts (TopologyError).
  C-7  uniform off-diagonal roulettes renormalised over the remaining
       candidates are uniform over them, so the roulette wheel is "the c-th
       remaining candidate in ascending rank order", c = floor(u * |cand|),
       u = u32 / 2**32  ->  c = (u32 * |cand|) >> 32 (integer, exact).
"""
from __future__ import annotations

import numpy as np

from .philox import philox4x32_10_np

TAG_FLAT = 0
TAG_HIER = 1
MAX_ATTEMPTS = 10_000
QUANTUM = 32  # segment bounds are multiples of 32 elements (reading C-2)


class TopologyError(RuntimeError):
    pass


def draws(seed: int, step: int, seg: int, attempt: int, n: int, tag: int) -> list[int]:
    """u32 draw for ranks i = 0..n-1 of one attempt.

    draw(i) = Philox4x32-10(ctr = [i>>2, attempt | tag<<16, seg, step],
                            key = [seed lo32, seed hi32])[i & 3]
    """
    nb = (n + 3) // 4
    q = np.arange(nb, dtype=np.uint64)
    w = philox4x32_10_np(q, np.full(nb, attempt | (tag << 16)), np.full(nb, seg), np.full(nb, step),
                         seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)
    out = []
    for i in range(n):
        out.append(int(w[i & 3][i >> 2]))
    return out


def alg2(seed: int, step: int, seg: int, n: int, tag: int = TAG_FLAT, return_attempts: bool = False):
    """One load-balanced topology: src[i] = the rank worker i receives from.

    Follows PAPER.md Alg. 2 rank by rank (i = 0..n-1) with readings C-1, C-4..C-7.
    With return_attempts, returns (src, number of attempts used).
    """
    if n < 2:
        raise ValueError("world_size < 2: no peer exists (SPEC.md:113)")
    for attempt in range(MAX_ATTEMPTS):
        u = draws(seed, step, seg, attempt, n, tag)
        avail = list(range(n))            # ranks not yet in dest_list
        src = []
        for i in range(n):
            cand = [r for r in avail if r != i]   # l.2-4: zero the picked ranks and i itself
            if not cand:                          # C-6: dead end -> restart
                break
            c = (u[i] * len(cand)) >> 32          # C-7: l.5-7 roulette over uniform row
            src.append(cand[c])                   # l.8
            avail.remove(cand[c])
        else:
            return (src, attempt + 1) if return_attempts else src
    raise TopologyError("Alg.2 restart limit (10,000) exceeded")


def topology(seed: int, step: int, n: int, k: int, tag: int = TAG_FLAT) -> np.ndarray:
    """int32 [k][n]: row s = alg2(seed, step, s, n, tag) — one topology per segment
    ("we set different random network topologies for each segment")."""
    return np.array([alg2(seed, step, s, n, tag) for s in range(k)], dtype=np.int32)


def inverse(src) -> list[int]:
    """send_to for every rank: Alg.1 l.6 `send_to = destinations.index[my rank]`."""
    src = list(src)
    return [src.index(r) for r in range(len(src))]


def segment_bounds(d: int, k: int) -> np.ndarray:
    """Reading C-2: b_s = min(d, 32*floor(s*ceil(d/32)/k)), b_k = d  (int64 [k+1]).

    The paper's segments are "blocks and FC layer of ResNet" over
    flattened tensors (Alg.1 l.3); the north_star splits one flat
    vector into k contiguous segments.  Requires ceil(d/32) >= k (non-empty segments).
    """
    nq = -(-d // QUANTUM)
    if k < 1 or nq < k:
        raise ValueError("need 1 <= k <= ceil(d/32)")
    b = [min(d, QUANTUM * ((s * nq) // k)) for s in range(k)] + [d]
    return np.array(b, dtype=np.int64)


def segment_of_columns(bounds: np.ndarray, cols: np.ndarray) -> np.ndarray:
    """Segment index of each column j: the s with b_s <= j < b_{s+1}."""
    return np.searchsorted(bounds, np.asarray(cols), side="right") - 1
