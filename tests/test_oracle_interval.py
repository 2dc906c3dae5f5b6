"""Pins for oracle/interval.py (communication-interval mode, Table 1
PAPER.md:230) against values the paper, SPEC's examples and the
mathematics fix."""
from fractions import Fraction

import numpy as np
import pytest

from oracle.interval import Accumulator

F32 = np.float32


def test_interval_one_is_identity():
    # comm_interval=1 -> every call flushes the input gradient unchanged
    rng = np.random.default_rng(1)
    acc = Accumulator((3, 17), 1)
    for _ in range(4):
        g = rng.standard_normal((3, 17)).astype(F32)
        out = acc.push(g)
        assert out is not None and np.array_equal(out, g)


def test_42_equal_gradients_flush_g():
    # SPEC.md:401 / Table 1 "Communication Interval 42": 42 equal gradients -> g.
    # dyadic values with <= 16 significant bits keep every partial sum exact
    rng = np.random.default_rng(2)
    g = (rng.integers(-2**15, 2**15, size=(4, 33)) * 2.0**-12).astype(F32)
    acc = Accumulator(g.shape, 42)
    for i in range(41):
        assert acc.push(g) is None
        assert acc.count == i + 1
    out = acc.push(g)
    assert np.array_equal(out, g)
    assert acc.count == 0 and not acc.acc.any()


def test_linear_regression_shards_equal_full_batch_gradient():
    # mean-loss linear model; the flushed average over K equal shards
    # equals the gradient of the concatenated batch, X^T (X w - y) / N  (fp64, 1e-12)
    rng = np.random.default_rng(3)
    K, b, p = 6, 20, 9
    X = rng.standard_normal((K * b, p))
    y = rng.standard_normal(K * b)
    w = rng.standard_normal(p)
    full = X.T @ (X @ w - y) / (K * b)
    acc = Accumulator((p,), K, dtype=np.float64)
    out = None
    for s in range(K):
        Xs, ys = X[s * b:(s + 1) * b], y[s * b:(s + 1) * b]
        out = acc.push(Xs.T @ (Xs @ w - ys) / b)
    assert out is not None
    assert np.max(np.abs(out - full)) <= 1e-12 * np.max(np.abs(full))


def test_fp32_mean_within_recursive_summation_bound():
    # exact rational mean vs the fp32 result: |err| <= gamma_I * sum|g| / I + u |mean|
    rng = np.random.default_rng(4)
    I, J = 42, 64
    gs = [rng.standard_normal(J).astype(F32) for _ in range(I)]
    acc = Accumulator((J,), I)
    for g in gs[:-1]:
        acc.push(g)
    out = acc.push(gs[-1])
    u = 2.0**-24
    gamma = I * u / (1 - I * u)
    for j in range(J):
        exact = sum(Fraction(float(g[j])) for g in gs) / I
        bound = gamma * sum(abs(float(g[j])) for g in gs) / I + u * abs(float(exact))
        assert abs(float(Fraction(float(out[j])) - exact)) <= bound


def test_sequential_order_and_reset():
    # accumulator += grad, left to right: (1 + 2^24) rounds to 2^24 in fp32, so the
    # sequence [1, 2^24, -2^24] sums to 0 (a pairwise sum would give 1)
    acc = Accumulator((1,), 3)
    assert acc.push(np.array([1.0], F32)) is None
    assert acc.push(np.array([2.0**24], F32)) is None
    assert acc.push(np.array([-(2.0**24)], F32))[0] == 0.0
    # after a flush the next interval starts from zero: same result as a fresh state
    rng = np.random.default_rng(5)
    gs = [rng.standard_normal(8).astype(F32) for _ in range(3)]
    fresh = Accumulator((8,), 3)
    r_fresh = [fresh.push(g) for g in gs][-1]
    used = Accumulator((8,), 3)
    for _ in range(3):
        used.push(rng.standard_normal(8).astype(F32) * F32(1e6))
    r_after = [used.push(g) for g in gs][-1]
    assert np.array_equal(r_fresh, r_after)


def test_negative_zero_becomes_positive_zero():
    # the accumulator starts at +0: +0 + (-0) = +0
    acc = Accumulator((1,), 1)
    out = acc.push(np.array([-0.0], F32))
    assert out[0] == 0.0 and not np.signbit(out[0])


def test_bad_interval():
    with pytest.raises(ValueError):
        Accumulator((1,), 0)
