"""Consensus distance and mean checksum, fp64.
Test infrastructure only.

With push-sum numerators x and weights w (reading C-11), the
de-biased estimate is z_ij = x_ij / w_{i,s(j)} and the network average is
z̄_j = Σ_i x_ij / Σ_i w_{i,s(j)}.

  CD = sqrt( (1/n) Σ_i Σ_j (z_ij - z̄_j)^2 )        consensus distance
  M  = Σ_j z̄_j                                      mean checksum

Written out directly (two passes, fp64).
"""
from __future__ import annotations

import numpy as np


def consensus(x: np.ndarray, w: np.ndarray, seg_of_col: np.ndarray):
    n = x.shape[0]
    x64 = x.astype(np.float64)
    wcol = w.astype(np.float64)[:, seg_of_col]          # [n, J]: w_{i, s(j)}
    z = x64 / wcol
    zbar = x64.sum(axis=0) / wcol.sum(axis=0)
    cd = float(np.sqrt(((z - zbar) ** 2).sum() / n))
    mean_sum = float(zbar.sum())
    return cd, mean_sum
