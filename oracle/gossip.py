"""One flat Crossover-SGD step: local momentum-SGD update, then the segment-wise
gossip exchange and merge.  Test infrastructure only.

Order (reading C-8): "parameter averaging is processed after the
gradient is applied to the weight parameters" (§3.1), i.e.
adapt-then-combine:

  a3  m_i <- fl(fl(mu * m_i) + g_i);   y_i <- fl(x_i - fl(lr * m_i))
      (reading C-9: heavy-ball momentum SGD, no dampening/Nesterov/wd)
  a4  worker i receives segment s of y from src_s(i)   (Alg.1 l.4-8)
  a5  x_i[R_s] <- fl(fl(y_i[R_s] + y_{src_s(i)}[R_s]) * 0.5)
      "layer = (layer + received_layer) / 2"  (Alg.1 l.17; reading C-10)
      w_{i,s}  <- fl(fl(w_{i,s} + w_{src_s(i),s}) * 0.5)
      push-sum weight mixed like x (reading C-11)

Every merge reads the pre-merge snapshot y / w ("wait until communication of all
segments are completed" before merging).  All arithmetic is
fp32 with one rounding per operation (numpy never contracts to FMA).

Arrays are restricted to a column subset: x, m, g are fp32 [n, J] and
seg_of_col[J] gives each column's segment, so the same code runs on full
vectors (J = d) and on the sampled columns of full-size parity runs (the update
is column-separable given the topology).
"""
from __future__ import annotations

import numpy as np

F32 = np.float32
HALF = np.float32(0.5)


def local_update(x: np.ndarray, m: np.ndarray, g: np.ndarray, lr, mu):
    """a3: returns (m', y) — separate fp32 ops, no FMA."""
    lr = F32(lr)
    mu = F32(mu)
    m_new = (mu * m).astype(F32) + g
    m_new = m_new.astype(F32)
    y = (x - (lr * m_new).astype(F32)).astype(F32)
    return m_new, y


def mix(y: np.ndarray, w: np.ndarray, src: np.ndarray, seg_of_col: np.ndarray, wire=None):
    """a4+a5 over a snapshot: x'[i, j] = (y[i, j] + y[src[seg(j), i], j]) * 0.5;
    w'[i, s] = (w[i, s] + w[src[s, i], s]) * 0.5.
    wire="bf16": the received y is rounded to bf16 first (oracle/wire.py, reading C-20)."""
    k = src.shape[0]
    x_new = np.empty_like(y)
    w_new = np.empty_like(w)
    for s in range(k):
        cols = np.nonzero(seg_of_col == s)[0]
        received = y[src[s]][:, cols]              # row i holds y_{src_s(i)}
        if wire == "bf16":
            from .wire import bf16_round
            received = bf16_round(received)
        x_new[:, cols] = ((y[:, cols] + received).astype(F32) * HALF).astype(F32)
        w_new[:, s] = ((w[:, s] + w[src[s], s]).astype(F32) * HALF).astype(F32)
    return x_new, w_new


def gossip_step(x, m, g, w, src, seg_of_col, lr, mu, wire=None):
    """One flat step (a3 -> a4 -> a5).  Returns (x', m', w')."""
    m_new, y = local_update(x, m, g, lr, mu)
    x_new, w_new = mix(y, w, src, seg_of_col, wire)
    return x_new, m_new, w_new
