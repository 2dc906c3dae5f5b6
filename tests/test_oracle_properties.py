"""Randomised (hypothesis) checks of the oracle's invariants over shapes, seeds and steps,
complementing the fixed pins P10, P11 and P14 in test_oracle_gossip.py.  CPU only."""
import numpy as np
from hypothesis import given, settings
from hypothesis import strategies as st

from oracle import topology as T
from oracle.gossip import gossip_step

F32 = np.float32


@st.composite
def problems(draw):
    n = draw(st.integers(2, 12))
    k = draw(st.integers(1, 4))
    d = draw(st.integers(32 * k, 32 * k + 100))
    seed = draw(st.integers(0, 2**63 - 1))
    step = draw(st.integers(0, 2**32 - 1))
    return n, k, d, seed, step


@settings(max_examples=60, deadline=None)
@given(problems())
def test_topology_rows_are_derangements(p):
    n, k, _, seed, step = p
    src = T.topology(seed, step, n, k)
    for row in src:
        assert sorted(row.tolist()) == list(range(n)) and np.all(row != np.arange(n))


@settings(max_examples=40, deadline=None)
@given(problems(), st.integers(0, 2**31 - 1))
def test_mixing_conserves_weight_sums_and_contracts(p, data_seed):
    # dyadic values with few significant bits keep every add and halving exact, so:
    #   sum_i w' = sum_i w per segment (push-sum mass), sum_i x' = sum_i y per column, and
    #   S - S' = 1/4 sum_i |x_i - x_src(i)|^2 for S = sum_i |x_i - mean|^2 (P11)
    n, k, d, seed, step = p
    rng = np.random.default_rng(data_seed)
    y = (rng.integers(-256, 256, (n, d)) * 2.0 ** -8).astype(F32)
    w = (rng.integers(1, 64, (n, k)) * 2.0 ** -5).astype(F32)
    z = np.zeros_like(y)
    src = T.topology(seed, step, n, k)
    seg = T.segment_of_columns(T.segment_bounds(d, k), np.arange(d))
    x, _, w2 = gossip_step(y, z, z, w, src, seg, 0.0, 0.0)
    assert np.array_equal(w2.astype(np.float64).sum(0), w.astype(np.float64).sum(0))
    assert np.array_equal(x.astype(np.float64).sum(0), y.astype(np.float64).sum(0))
    y64 = y.astype(np.float64)
    S = ((y64 - y64.mean(0)) ** 2).sum()
    S2 = ((x.astype(np.float64) - y64.mean(0)) ** 2).sum()
    recv = np.stack([y64[src[seg[j]], j] for j in range(d)], axis=1)
    assert abs((S - S2) - 0.25 * ((y64 - recv) ** 2).sum()) <= 1e-9 * max(1.0, S)
