"""Pins for oracle/lars.py against SPEC's worked examples,
brute-force enumeration, closed forms and exact special cases."""
import numpy as np
import pytest

import synth
from oracle import topology as T
from oracle.gossip import gossip_step
from oracle.lars import (lars_gossip_step, lars_local_lr, layer_lr, plan_bounds, segment_plan,
                         segment_plan_bruteforce)

F32 = np.float32


def test_lars_local_lr_spec_examples():
    # SPEC.md:373-375
    assert lars_local_lr(0.0, 1.0, 0.0025, 5e-5, 1e-9) == 1.0
    assert lars_local_lr(1.0, 0.0, 0.0025, 5e-5, 1e-9) == 1.0
    assert lars_local_lr(1.0, 1.0, 0.0025, 0.0, 0.0) == 0.0025        # Table 1 coefficient, ratio 1
    assert lars_local_lr(2.0, 1.0, 0.0025, 5e-5, 1e-9) == 0.0025 * 2 / (1 + 1e-4 + 1e-9)


def test_segment_plan_spec_examples():
    # SPEC.md:45-47
    assert segment_plan([2, 2, 2, 2], 2) == [0, 0, 1, 1]
    assert segment_plan([5, 3, 9], 1) == [0, 0, 0]
    assert segment_plan([10, 1, 1], 2) == [0, 1, 1]
    with pytest.raises(ValueError):
        segment_plan([1, 2], 3)
    with pytest.raises(ValueError):
        segment_plan([], 1)


def test_segment_plan_matches_bruteforce():
    rng = np.random.default_rng(0)
    for _ in range(300):
        L = int(rng.integers(1, 9))
        sizes = [int(v) for v in rng.integers(1, 6, size=L) * 4]
        for k in range(1, L + 1):
            assert segment_plan(sizes, k) == segment_plan_bruteforce(sizes, k), (sizes, k)


def test_segment_plan_resnet50_blocks():
    sizes, block = synth.resnet50_layers()
    assert len(sizes) == 161 and sum(sizes) == 25_557_032       # torchvision ResNet-50
    lb = np.concatenate([[0], np.cumsum(sizes)])
    b = plan_bounds(lb, block)                                   # Table 1: blocks and FC layer
    assert len(b) == 19 and b[-1] == 25_557_032 and b[-2] == 25_557_032 - 2_049_000
    seg = segment_plan(sizes, 18)
    mx = max(sum(s for s, g in zip(sizes, seg) if g == q) for q in range(18))
    assert mx >= max(sizes) and sorted(set(seg)) == list(range(18))
    assert plan_bounds([0, 4, 8, 20], [0, 0, 1]).tolist() == [0, 8, 20]


def test_pythagorean_norms():
    # ||(3,4)|| = 5, ||(6,8)|| = 10 -> scale = eta/2 (wd = eps = 0); lr = 1, eta = 0.5 -> 0.25
    x = np.array([[3, 4, 0, 0]], F32)
    g = np.array([[6, 8, 0, 0]], F32)
    assert layer_lr(x, g, [0, 4], 1.0, 0.5, 0.0, 0.0)[0, 0] == F32(0.25)


def test_scale_invariance_bitwise():
    # mu = 0, wd = 0, eps = 0: the update lrs * g is invariant under g -> c g
    rng = np.random.default_rng(1)
    n, d, k = 4, 64, 2
    lb = [0, 20, 44, 64]
    x = rng.standard_normal((n, d)).astype(F32)
    g = rng.standard_normal((n, d)).astype(F32)
    m = np.zeros_like(x)
    w = np.ones((n, k), F32)
    src = T.topology(0, 0, n, k)
    seg = T.segment_of_columns(T.segment_bounds(d, k), np.arange(d))
    base = lars_gossip_step(x, m, g, w, src, seg, lb, 0.5, 0.0, 0.01, 0.0, 0.0)
    for c in [2.0, 0.25, 1024.0]:
        out = lars_gossip_step(x, m, (g * F32(c)).astype(F32), w, src, seg, lb, 0.5, 0.0, 0.01, 0.0, 0.0)
        assert np.array_equal(out[0], base[0]), c


def test_zero_weights_reduce_to_plain_step():
    # |x_l| = 0 -> scale 1 -> lrs = lr; with wd = 0 the step is the plain flat step (pinned in
    # test_oracle_gossip.py)
    rng = np.random.default_rng(2)
    n, d, k = 5, 96, 3
    x = np.zeros((n, d), F32)
    m = rng.standard_normal((n, d)).astype(F32)
    g = rng.standard_normal((n, d)).astype(F32)
    w = np.ones((n, k), F32)
    src = T.topology(3, 1, n, k)
    seg = T.segment_of_columns(T.segment_bounds(d, k), np.arange(d))
    lr, mu = F32(2.0 ** -6), F32(0.96)
    a = lars_gossip_step(x, m, g, w, src, seg, [0, 32, 96], lr, mu, 0.0025, 0.0, 1e-9)
    b = gossip_step(x, m, g, w, src, seg, lr, mu)
    for u, v in zip(a[:3], b):
        assert np.array_equal(u, v)
    assert np.all(a[3] == lr)


def test_weight_decay_term_closed_form():
    # g = 0 -> scale 1; mu = 0: m' = wd x, y = x - lr wd x; x = 1, wd = 2^-4, lr = 2^-2 -> 1 - 2^-6
    x = np.ones((2, 4), F32)
    g = np.zeros((2, 4), F32)
    m = np.full((2, 4), 7.0, F32)
    w = np.ones((2, 1), F32)
    src = np.array([[1, 0]])
    seg = np.zeros(4, dtype=np.int64)
    xn, mn, wn, lrs = lars_gossip_step(x, m, g, w, src, seg, [0, 4], 0.25, 0.0, 0.0025, 2.0 ** -4, 0.0)
    assert np.all(mn == F32(2.0 ** -4)) and np.all(xn == F32(1 - 2.0 ** -6)) and np.all(lrs == F32(0.25))


def test_layer_rates_are_per_worker_and_per_layer():
    # doubling one layer of one worker's x (g fixed, wd = eps = 0) doubles only that rate
    rng = np.random.default_rng(3)
    x = rng.standard_normal((3, 40)).astype(F32)
    g = rng.standard_normal((3, 40)).astype(F32)
    lb = [0, 8, 24, 40]
    a = layer_lr(x, g, lb, 1.0, 2.0 ** -8, 0.0, 0.0)
    x2 = x.copy()
    x2[1, 8:24] *= F32(2)
    b = layer_lr(x2, g, lb, 1.0, 2.0 ** -8, 0.0, 0.0)
    expect = a.copy()
    expect[1, 1] = a[1, 1] * F32(2)
    assert np.array_equal(b, expect)


def test_lars_hier_groups_equal_world_is_flat_lars():
    # G = n: each group is one worker, the group mean is its own gradient and the leader
    # topology (tag HIER) is used: equal to the flat LARS step with that topology
    from oracle.lars import lars_hier_step
    rng = np.random.default_rng(9)
    n, d, k = 4, 48, 2
    lb = [0, 16, 48]
    x = rng.standard_normal((n, d)).astype(F32)
    g = rng.standard_normal((n, d)).astype(F32)
    m = rng.standard_normal((n, d)).astype(F32)
    w = np.ones((n, k), F32)
    seg = T.segment_of_columns(T.segment_bounds(d, k), np.arange(d))
    a = lars_hier_step(x, m, g, w, n, 3, 5, k, seg, lb, 0.5, 0.9, 0.01, 1e-3, 1e-9)
    src = T.topology(3, 5, n, k, T.TAG_HIER)
    b = lars_gossip_step(x, m, g, w, src, seg, lb, 0.5, 0.9, 0.01, 1e-3, 1e-9)
    for u, v in zip(a, b):
        assert np.array_equal(u, v)


def test_lars_hier_one_group_uses_the_synchronised_norm():
    # G = 1: every worker ends with the same x, updated with the rate of the MEAN gradient's
    # norm, not any single worker's; with identical gradients it equals flat LARS
    from oracle.lars import lars_hier_step
    rng = np.random.default_rng(10)
    n, d = 4, 32
    lb = [0, 32]
    x = np.repeat(rng.standard_normal((1, d)).astype(F32), n, axis=0)
    g1 = rng.standard_normal((1, d)).astype(F32)
    g = np.repeat(g1, n, axis=0) * F32(2)   # identical gradients, exact mean
    z = np.zeros_like(x)
    xh, _, _, lrs = lars_hier_step(x, z, g, np.ones((n, 1), F32), 1, 0, 0, 1, np.zeros(d, np.int64), lb,
                                   1.0, 0.0, 0.01, 0.0, 0.0)
    assert lrs.shape == (1, 1) and np.all(xh == xh[0])
    assert lrs[0, 0] == layer_lr(x[:1], g[:1], lb, 1.0, 0.01, 0.0, 0.0)[0, 0]
