"""Hierarchical Crossover-SGD (§3.3, Fig. 5).  Test infrastructure only.

"The first step is to reduce the gradients of the worker nodes in each group
... the L node, which is the leader node in each group, collects gradients
from each worker and reduces them to apply a reduced gradient to the model.
The second step is the communication of the inter-group by utilizing
Crossover-SGD. Subsequently, the gossiped model parameter of the leader node
propagates to other workers in each group."

Readings: C-12 groups are contiguous blocks of n/G workers, the
leader is the lowest rank of its block, "reduce" = mean
(sum in ascending member order, fp32, then * fp32(1/|G|)); momentum is defined
at leaders only.  C-13 the leader topology is Alg. 2 over the L = G leaders
(dense leader index) with domain tag HIER; L = 1 skips mixing.
"""
from __future__ import annotations

import numpy as np

from .gossip import local_update, mix
from .topology import TAG_HIER, topology

F32 = np.float32


def group_mean(g: np.ndarray, groups: int) -> np.ndarray:
    """h1: per group, fl(fl(...fl(g_l + g_{l+1}) ...) * fp32(1/|G|)); returns [groups, J]."""
    n = g.shape[0]
    gs = n // groups
    inv = F32(1.0 / gs)
    out = np.empty((groups, g.shape[1]), dtype=F32)
    for G in range(groups):
        acc = g[G * gs].astype(F32)
        for r in range(1, gs):
            acc = (acc + g[G * gs + r]).astype(F32)
        out[G] = (acc * inv).astype(F32)
    return out


def hier_step(x, m, g, w, groups: int, seed: int, step: int, k: int, seg_of_col, lr, mu):
    """One hierarchical step over all n workers.  Returns (x', m', w', leader_src).

    Members' momentum rows are returned unchanged (momentum is defined at leaders only).
    """
    n = x.shape[0]
    if groups < 1 or n % groups:
        raise ValueError("groups must divide world")
    gs = n // groups
    leaders = [G * gs for G in range(groups)]
    gbar = group_mean(g, groups)                                    # h1
    m_new = m.copy()
    mL, yL = local_update(x[leaders], m[leaders], gbar, lr, mu)     # leaders apply
    m_new[leaders] = mL
    wL = w[leaders]
    if groups >= 2:                                                 # h2
        srcL = topology(seed, step, groups, k, TAG_HIER)
        xL, wL = mix(yL, wL, srcL, seg_of_col)
    else:                                                           # L = 1: no gossip
        srcL = None
        xL = yL
    x_new = np.repeat(xL, gs, axis=0)                               # h3
    w_new = np.repeat(wL, gs, axis=0)
    return x_new, m_new, w_new, srcL
