"""Pins of the hierarchical variant and the fp64 diagnostics."""
import json
import os

import numpy as np
import pytest

import synth
from conftest import GOLDEN
from oracle import topology as T
from oracle.diagnostics import consensus
from oracle.gossip import gossip_step, local_update
from oracle.hierarchical import group_mean, hier_step

F32 = np.float32


def test_p12_hand_kat():
    gold = json.load(open(os.path.join(GOLDEN, "p12_hier_kat.json")))
    n, G, k, d = gold["n"], gold["groups"], gold["k"], gold["d"]
    x = np.repeat(np.array(gold["x0_per_worker"], F32)[:, None], d, 1)
    g = np.repeat(np.array(gold["grad_per_worker"], F32)[:, None], d, 1)
    m = np.zeros_like(x)
    w = np.ones((n, k), F32)
    seg = np.zeros(d, int)
    for t in ("0", "1"):
        x, m, w, srcL = hier_step(x, m, g, w, G, 0, int(t), k, seg, gold["lr"], gold["momentum"])
        assert srcL.tolist() == [[1, 0]]
        assert np.all(x == np.array(gold["expected_x"][t], F32)[:, None])
        assert m[[0, 2], 0].tolist() == gold["expected_leader_m"][t]
        assert np.all(w == 1.0)


def _rand(n, d, seed):
    x = synth.init_params(seed, range(n), d)
    g = synth.init_params(seed + 100, range(n), d) * F32(0.0625)
    return x, g


def test_group_size_one_is_flat():
    # G = n  ->  optimizer step then crossover round (same topology)
    n, d, k = 6, 256, 4
    x, g = _rand(n, d, 1)
    m = synth.init_params(7, range(n), d) * F32(0.1)
    w = np.ones((n, k), F32)
    seg = T.segment_of_columns(T.segment_bounds(d, k), np.arange(d))
    xh, mh, wh, srcL = hier_step(x, m, g, w, n, 9, 4, k, seg, 0.015625, 0.96)
    xf, mf, wf = gossip_step(x, m, g, w, T.topology(9, 4, n, k, T.TAG_HIER), seg, 0.015625, 0.96)
    assert np.array_equal(xh, xf) and np.array_equal(mh, mf) and np.array_equal(wh, wf)


def test_one_group_is_allreduce_sgd():
    # one group of n -> gradient allreduce + one SGD step, no gossip
    n, d = 4, 128
    x, g = _rand(n, d, 2)
    x[:] = x[0]
    m = np.zeros_like(x)
    w = np.ones((n, 1), F32)
    xh, mh, _, srcL = hier_step(x, m, g, w, 1, 0, 0, 1, np.zeros(d, int), 0.5, 0.9)
    assert srcL is None
    mean = (((g[0] + g[1]).astype(F32) + g[2]).astype(F32) + g[3]).astype(F32) * F32(0.25)
    assert np.array_equal(mh[0], mean)
    assert np.array_equal(xh, np.repeat((x[0] - F32(0.5) * mean)[None].astype(F32), n, 0))


@pytest.mark.parametrize("n,G", [(8, 2), (8, 4), (12, 3), (16, 8)])
def test_intra_group_bitwise_equality_and_leader_mean(n, G):
    d, k = 320, 4
    x, g = _rand(n, d, n + G)
    m = np.zeros_like(x)
    w = np.ones((n, k), F32)
    seg = T.segment_of_columns(T.segment_bounds(d, k), np.arange(d))
    gs = n // G
    for t in range(5):
        x, m, w, srcL = hier_step(x, m, g, w, G, 3, t, k, seg, 0.015625, 0.96)
        for grp in range(G):
            blk = x[grp * gs:(grp + 1) * gs]
            assert np.all(blk == blk[0])
        if G == 2:  # L = 2: forced swap -> both groups identical
            assert np.all(x == x[0])
    # leader-level mean preservation of the gossip phase
    lead = list(range(0, n, gs))
    gbar = group_mean(g, G)
    _, yL = local_update(x[lead], m[lead], gbar, 0.015625, 0.96)
    x2, _, _, _ = hier_step(x, m, g, w, G, 3, 99, k, seg, 0.015625, 0.96)
    assert np.allclose(x2[lead].astype(np.float64).mean(0), yL.astype(np.float64).mean(0),
                       atol=2.0**-22 * np.abs(yL).max())


def test_group_mean_is_sum_times_reciprocal():
    g = np.array([[1.0], [3.0], [-1.0], [0.0], [2.0], [2.0]], F32)
    assert group_mean(g, 2)[:, 0].tolist() == [1.0, F32(4.0) * F32(1 / 3)]


def test_hier_rejects_indivisible_groups():
    with pytest.raises(ValueError):
        hier_step(np.zeros((6, 32), F32), np.zeros((6, 32), F32), np.zeros((6, 32), F32),
                  np.ones((6, 1), F32), 4, 0, 0, 1, np.zeros(32, int), 0.1, 0.9)


# ---- diagnostics -------------------------------------------------------------------------

def test_consensus_distance_spec_examples():
    # two workers [0] and [2] -> 1; all equal -> 0
    w = np.ones((2, 1), F32)
    assert consensus(np.array([[0.0], [2.0]], F32), w, np.zeros(1, int)) == (1.0, 1.0)
    assert consensus(np.full((3, 5), 7.0, F32), np.ones((3, 1), F32), np.zeros(5, int)) == (0.0, 35.0)


def test_consensus_brute_force_with_weights():
    rng = np.random.default_rng(4)
    n, d, k = 5, 40, 3
    x = rng.standard_normal((n, d)).astype(F32)
    w = rng.uniform(0.5, 2, (n, k)).astype(F32)
    seg = T.segment_of_columns(np.array([0, 10, 25, 40]), np.arange(d))
    acc, msum = 0.0, 0.0
    for j in range(d):
        s = seg[j]
        zbar = sum(float(x[i, j]) for i in range(n)) / sum(float(w[i, s]) for i in range(n))
        msum += zbar
        for i in range(n):
            acc += (float(x[i, j]) / float(w[i, s]) - zbar) ** 2
    cd, ms = consensus(x, w, seg)
    assert abs(cd - (acc / n) ** 0.5) <= 1e-12 * cd
    assert abs(ms - msum) <= 1e-12 * abs(msum) + 1e-12
