"""Pins for oracle/wire.py (bf16 wire format, reading C-20): bf16 rounding against
hand values and torch's bf16 conversion, and the step against closed forms."""
import numpy as np
import pytest
import torch

from oracle import topology as T
from oracle.gossip import gossip_step
from oracle.wire import bf16_round

F32 = np.float32


def test_bf16_round_hand_values():
    # bf16 keeps 8 significand bits: the ulp of [1, 2) is 2^-7
    cases = [(1.0, 1.0), (1 + 2**-8, 1.0),                  # exact half: ties to even (1.0)
             (1 + 3 * 2**-8, 1 + 2**-6),                      # half above 1+2^-7 (odd): up to even
             (1 + 2**-8 + 2**-20, 1 + 2**-7),                 # just above half: up
             (-(1 + 2**-8 + 2**-20), -(1 + 2**-7)),           # symmetric
             (0.0, 0.0), (3.0, 3.0), (2.0**-130, 2.0**-130)]  # representable (incl. subnormal)
    for v, want in cases:
        assert bf16_round(np.array([v], F32))[0] == F32(want), v
    assert np.signbit(bf16_round(np.array([-0.0], F32))[0])


def test_bf16_round_matches_torch_and_nearest():
    rng = np.random.default_rng(0)
    v = (rng.standard_normal(200_000) * np.exp(rng.uniform(-30, 30, 200_000))).astype(F32)
    got = bf16_round(v)
    assert np.array_equal(got, torch.from_numpy(v).to(torch.bfloat16).float().numpy())
    # nearest: |v - r| <= half an ulp of r's binade
    e = np.floor(np.log2(np.abs(got.astype(np.float64))))
    assert np.all(np.abs(v.astype(np.float64) - got) <= 2.0 ** (e - 8) * (1 + 1e-12))


def test_bf16_representable_values_make_wire_a_no_op():
    # y with <= 8 significant bits: bf16(y) == y, so the bf16 wire step equals the fp32 step
    rng = np.random.default_rng(1)
    n, d, k = 6, 200, 3
    x = (rng.integers(-128, 128, (n, d)) * 2.0**-4).astype(F32)
    z = np.zeros_like(x)
    w = np.ones((n, k), F32)
    src = T.topology(2, 0, n, k)
    seg = T.segment_of_columns(T.segment_bounds(d, k), np.arange(d))
    a = gossip_step(x, z, z, w, src, seg, 0.0, 0.0, wire="bf16")
    b = gossip_step(x, z, z, w, src, seg, 0.0, 0.0)
    for u, v in zip(a, b):
        assert np.array_equal(u, v)


def test_two_worker_swap_closed_form():
    # n = 2: x0' = (y0 + bf16(y1)) / 2 and x1' = (y1 + bf16(y0)) / 2; 1 + 2^-9 rounds to 1
    y = np.array([[1.0 + 2**-9], [3.0]], F32)
    z = np.zeros_like(y)
    x, _, w = gossip_step(y, z, z, np.ones((2, 1), F32), np.array([[1, 0]]), np.zeros(1, np.int64), 0.0, 0.0,
                          wire="bf16")
    assert x[0, 0] == F32((1.0 + 2**-9 + 3.0) / 2) and x[1, 0] == F32((3.0 + 1.0) / 2)
    assert np.all(w == 1)


@pytest.mark.parametrize("n,k", [(4, 1), (9, 4)])
def test_mean_drift_bounded_by_rounding(n, k):
    # bf16 rounding is off by at most half an ulp = 2^-8 relative; halved by the merge, the
    # column mean moves by at most 2^-9 * mean(|y|) per step, plus fp32 rounding
    rng = np.random.default_rng(n)
    d = 300
    y = rng.standard_normal((n, d)).astype(F32)
    z = np.zeros_like(y)
    src = T.topology(4, 1, n, k)
    seg = T.segment_of_columns(T.segment_bounds(d, k), np.arange(d))
    x, _, _ = gossip_step(y, z, z, np.ones((n, k), F32), src, seg, 0.0, 0.0, wire="bf16")
    drift = np.abs(x.astype(np.float64).mean(0) - y.astype(np.float64).mean(0))
    assert np.all(drift <= 2.0**-9 * np.abs(y).astype(np.float64).mean(0) + 4 * 2.0**-24 * np.abs(y).max(0))
