"""LARS in the flat step, with a layer table and a layer-aligned segment plan.
Test infrastructure only.

Sources:
  PAPER.md:35 (section 1): LARS "adapts the learning rate of each layer by the ratio
      of the weight norm to the gradient norm".
  PAPER.md:197 (section 3.3): the gradient norm LARS uses must be the reduced one.
  Table 1: LARS coefficient 0.0025, weight decay 5e-5,
      momentum 0.96, "Segmenting blocks and FC layer of ResNet".
  SPEC.md:368-376: lars_local_lr and the momentum step with per-layer scales.
  SPEC.md:40-47: build_segment_plan, contiguous and balanced.

Readings (C-18, C-19):
  scale_l = eta * |x_l| / (|g_l| + wd * |x_l| + eps), or 1 if |x_l| = 0 or |g_l| = 0,
      in fp64; |v| = sqrt(sum_j v_j^2) over the layer's columns, in fp64.
  lrs_l   = fp32(lr * scale_l)                                 (one rounding)
  a3'     m <- fl(fl(mu * m) + fl(g + fl(wd * x)));  y <- fl(x - fl(lrs_l * m))
  a4, a5  unchanged (gossip.mix), with the segment bounds of the layer plan.
  Segment plan: among the contiguous partitions of the layers into k non-empty
      segments, those with the smallest largest segment (elements); of these, the
      one whose segment ends are lexicographically largest (each segment takes as
      many layers as it can, left to right).
"""
from __future__ import annotations

import itertools

import numpy as np

from .gossip import mix

F32 = np.float32


# ---- segment plan (SPEC build_segment_plan; Table 1 "blocks and FC layer") ---------

def _feasible(sizes, k, cap):
    """Can `sizes` be cut into at most k contiguous pieces of total <= cap each?"""
    pieces, cur = 1, 0
    for s in sizes:
        if s > cap:
            return False
        if cur + s > cap:
            pieces, cur = pieces + 1, s
        else:
            cur += s
    return pieces <= k


def segment_plan(sizes, k):
    """seg_of_layer for the plan defined above.  sizes: element counts per layer."""
    L = len(sizes)
    if L == 0 or not 1 <= k <= L:
        raise ValueError("need 1 <= k <= number of layers")
    # the smallest feasible cap is one of the contiguous sums
    cands = sorted({sum(sizes[i:j]) for i in range(L) for j in range(i + 1, L + 1)})
    cap = next(c for c in cands if _feasible(sizes, k, c))
    seg, start = [], 0
    for s in range(k):
        left = k - s - 1  # segments still to fill after this one
        if left == 0:
            end = L
        else:
            # the largest end whose segment stays <= cap while the >= `left` remaining
            # layers can still be cut into `left` pieces of <= cap
            end = max(e for e in range(start + 1, L - left + 1)
                      if sum(sizes[start:e]) <= cap and _feasible(sizes[e:], left, cap))
        seg.extend([s] * (end - start))
        start = end
    return seg


def segment_plan_bruteforce(sizes, k):
    """Reference for the pins: enumerate every contiguous partition."""
    L = len(sizes)
    best = None
    for cuts in itertools.combinations(range(1, L), k - 1):
        b = (0,) + cuts + (L,)
        mx = max(sum(sizes[b[i]:b[i + 1]]) for i in range(k))
        key = (mx, tuple(-c for c in cuts))  # smaller max first, then larger cut positions
        if best is None or key < best[0]:
            best = (key, b)
    b = best[1]
    return [s for s in range(k) for _ in range(b[s + 1] - b[s])]


def plan_bounds(layer_bounds, seg_of_layer):
    """Segment bounds (k+1) from layer bounds (L+1) and seg_of_layer (L)."""
    k = seg_of_layer[-1] + 1
    out = [0]
    for li in range(1, len(seg_of_layer)):
        if seg_of_layer[li] != seg_of_layer[li - 1]:
            out.append(int(layer_bounds[li]))
    out.append(int(layer_bounds[-1]))
    assert len(out) == k + 1
    return np.array(out, dtype=np.int64)


# ---- LARS (SPEC lars_local_lr) ----------------------------------------

def lars_local_lr(weight_norm, grad_norm, eta, weight_decay, eps):
    """SPEC.md:370-371, in fp64."""
    if weight_norm == 0.0 or grad_norm == 0.0:
        return 1.0
    return (eta * weight_norm) / ((grad_norm + weight_decay * weight_norm) + eps)


def layer_lr(x, g, layer_bounds, lr, eta, weight_decay, eps):
    """lrs[i][l] = fp32(lr * scale_il), the norms over layer l of worker i's x and g."""
    n, L = x.shape[0], len(layer_bounds) - 1
    out = np.zeros((n, L), F32)
    eta64, wd64, eps64 = float(F32(eta)), float(F32(weight_decay)), float(F32(eps))
    for i in range(n):
        for li in range(L):
            a, b = layer_bounds[li], layer_bounds[li + 1]
            nw = float(np.sqrt(np.sum(x[i, a:b].astype(np.float64) ** 2)))
            ng = float(np.sqrt(np.sum(g[i, a:b].astype(np.float64) ** 2)))
            out[i, li] = F32(float(F32(lr)) * lars_local_lr(nw, ng, eta64, wd64, eps64))
    return out


def lars_update(x, m, g, lrs, layer_of_col, mu, weight_decay):
    """a3 with per-layer rates: returns (m', y).  x, m, g: fp32 [n, J]."""
    mu, wd = F32(mu), F32(weight_decay)
    gw = g + wd * x
    m_new = mu * m + gw
    rate = lrs[:, layer_of_col]                     # [n, J]
    y = x - rate * m_new
    return m_new.astype(F32), y.astype(F32)


def lars_gossip_step(x, m, g, w, src, seg_of_col, layer_bounds, lr, mu, eta, weight_decay, eps):
    """One flat step with LARS on full rows (J = d).  Returns (x', m', w', lrs)."""
    lrs = layer_lr(x, g, layer_bounds, lr, eta, weight_decay, eps)
    d = x.shape[1]
    layer_of_col = np.searchsorted(np.asarray(layer_bounds), np.arange(d), side="right") - 1
    m_new, y = lars_update(x, m, g, lrs, layer_of_col, mu, weight_decay)
    x_new, w_new = mix(y, w, src, seg_of_col)
    return x_new, m_new, w_new, lrs


def lars_hier_step(x, m, g, w, groups, seed, step, k, seg_of_col, layer_bounds, lr, mu, eta, weight_decay, eps):
    """Hierarchical step with LARS (LARS needs the gradient norm synchronised,
    so the leader applies it to the group-reduced gradient).  h1 group mean; the leaders'
    rates come from their x and the group mean gbar (C-18); h2 leader gossip; h3 members
    take the leader's x and w.  Full rows only.  Returns (x', m', w', lrs_of_leaders)."""
    from .hierarchical import group_mean
    from .topology import TAG_HIER, topology
    n = x.shape[0]
    gs = n // groups
    leaders = [G * gs for G in range(groups)]
    gbar = group_mean(g, groups)
    lrs = layer_lr(x[leaders], gbar, layer_bounds, lr, eta, weight_decay, eps)
    d = x.shape[1]
    layer_of_col = np.searchsorted(np.asarray(layer_bounds), np.arange(d), side="right") - 1
    mL, yL = lars_update(x[leaders], m[leaders], gbar, lrs, layer_of_col, mu, weight_decay)
    m_new = m.copy()
    m_new[leaders] = mL
    wL = w[leaders]
    if groups >= 2:
        xL, wL = mix(yL, wL, topology(seed, step, groups, k, TAG_HIER), seg_of_col)
    else:
        xL = yL
    return np.repeat(xL, gs, axis=0), m_new, np.repeat(wL, gs, axis=0), lrs
