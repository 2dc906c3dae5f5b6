"""Pins of the oracle's flat step (Alg. 1 + PAPER.md:122 ordering)."""
import json
import os

import numpy as np
import pytest
import torch

import synth
from conftest import GOLDEN
from oracle import topology as T
from oracle.diagnostics import consensus
from oracle.gossip import gossip_step, local_update, mix

F32 = np.float32


def _state(n, d, seed=0):
    x = synth.init_params(seed, range(n), d)
    return x, np.zeros_like(x), np.ones((n, 1), F32)


def _segcols(d, k):
    return T.segment_of_columns(T.segment_bounds(d, k), np.arange(d))


def test_p6_worked_kat():
    gold = json.load(open(os.path.join(GOLDEN, "p6_worked_kat.json")))
    n, k, d = gold["n"], gold["k"], gold["d"]
    seg = _segcols(d, k)
    x = np.repeat(np.array(gold["x0_per_worker"], F32)[:, None], d, axis=1)
    g = np.repeat(np.array(gold["grad_per_worker"], F32)[:, None], d, axis=1)
    m = np.zeros_like(x)
    w = np.ones((n, k), F32)
    for t in ("0", "1"):
        src = np.array(gold["topology"][t], np.int32)
        x, m, w = gossip_step(x, m, g, w, src, seg, gold["lr"], gold["momentum"])
        e = gold["expected"][t]
        assert np.array_equal(m[:, 0], np.array(e["m"], F32))
        assert np.array_equal(x[:, :32], np.repeat(np.array(e["seg0"], F32)[:, None], 32, 1))
        assert np.array_equal(x[:, 32:], np.repeat(np.array(e["seg1"], F32)[:, None], 32, 1))
        assert np.all(w == 1.0)
    cs = gold["column_sums_after_step1"]
    assert x[:, 0].sum() == cs["seg0"] and x[:, 40].sum() == cs["seg1"]


def test_spec_pairwise_merge_n2():
    # n=2, params [0] and [2] -> both [1]
    x = np.array([[0.0] * 32, [2.0] * 32], F32)
    xo, _, _ = gossip_step(x, np.zeros_like(x), np.zeros_like(x), np.ones((2, 1), F32),
                           T.topology(0, 0, 2, 1), np.zeros(32, int), 0.0, 0.0)
    assert np.all(xo == 1.0)


def test_consensus_is_a_fixed_point():
    # SPEC.md:214
    n, d, k = 5, 256, 4
    x = np.repeat(synth.hash_uniform(1, 0, 0, d)[None], n, 0)
    xo, _, _ = gossip_step(x, np.zeros_like(x), np.zeros_like(x), np.ones((n, k), F32),
                           T.topology(1, 3, n, k), _segcols(d, k), 0.0, 0.96)
    assert np.array_equal(xo, x)


@pytest.mark.parametrize("r", [1, 2, 3, 4, 5, 6])
def test_p7_xor_butterfly_is_allreduce(r):
    # complete-graph reduction: after r exchange rounds over XOR partners, every worker
    # holds the butterfly mean (bitwise equal everywhere), within 2^-23 max|x| of the exact mean
    n, d = 2**r, 512
    x, m, _ = _state(n, d, seed=r)
    w = np.ones((n, 1), F32)
    seg = np.zeros(d, int)
    exact = x.astype(np.float64).mean(0)
    for t in range(r):
        src = np.array([[i ^ (1 << t) for i in range(n)]], np.int32)
        x, m, w = gossip_step(x, m, np.zeros_like(x), w, src, seg, 0.0, 0.96)
    assert np.all(x == x[0])
    assert np.max(np.abs(x[0] - exact)) <= 2.0**-23 * np.abs(exact).max() + 2.0**-23
    assert consensus(x, w, seg)[0] == 0.0


def _pushsum_round(vals, wts, t):
    """SPEC.md:270-278, written independently: split (value, weight) in half, keep one
    half, send the other to exponential_peer(i, t) = (i + 2^(t mod log2 n)) mod n."""
    n = len(vals)
    off = 1 << (t % (n.bit_length() - 1))
    nv = [v * F32(0.5) for v in vals]
    nw = [w * F32(0.5) for w in wts]
    outv, outw = list(nv), list(nw)
    for i in range(n):
        peer = (i + off) % n
        outv[peer] = outv[peer] + nv[i]
        outw[peer] = outw[peer] + nw[i]
    return outv, outw


@pytest.mark.parametrize("n", [2, 4, 8, 16])
def test_p8_k1_exponential_equals_sgp_pushsum(n):
    d = 96
    x, m, _ = _state(n, d, seed=n)
    w = np.ones((n, 1), F32)
    vals, wts = [x[i].copy() for i in range(n)], [w[i].copy() for i in range(n)]
    seg = np.zeros(d, int)
    from oracle.sgp import exponential_topology
    for t in range(7):
        src = exponential_topology(t, n, 1)
        x, m, w = gossip_step(x, m, np.zeros_like(x), w, src, seg, 0.0, 0.96)
        vals, wts = _pushsum_round(vals, wts, t)
        assert np.array_equal(x, np.stack(vals))
        assert np.array_equal(w, np.stack(wts))
    zbar = x.astype(np.float64).sum(0) / w.astype(np.float64).sum()
    assert np.allclose((x / w)[0], zbar, atol=1e-3) or n > 2


@pytest.mark.parametrize("n,k", [(2, 1), (3, 2), (8, 4), (16, 8), (33, 5)])
def test_p9_routing_probe(n, k):
    # x_i[j] = i, m = g = 0, lr = 0  ->  2 x'_i[j] - i == src_s(i) exactly
    d = 32 * k + 17
    b = T.segment_bounds(d, k)
    seg = T.segment_of_columns(b, np.arange(d))
    x = np.repeat(np.arange(n, dtype=F32)[:, None], d, 1)
    src = T.topology(7, 2, n, k)
    xo, _, _ = gossip_step(x, np.zeros_like(x), np.zeros_like(x), np.ones((n, k), F32), src, seg, 0.0, 0.5)
    decoded = 2 * xo - np.arange(n, dtype=F32)[:, None]
    for s in range(k):
        assert np.all(decoded[:, b[s]:b[s + 1]] == src[s][:, None])


@pytest.mark.parametrize("n", [2, 3, 4, 8, 32])
def test_p10_mean_invariance(n):
    d, k = 2048, 4
    x, m, _ = _state(n, d, seed=n + 1)
    w = np.ones((n, k), F32)
    seg = _segcols(d, k)
    for t in range(20):
        mean0 = x.astype(np.float64).mean(0)
        x, m, w = gossip_step(x, m, np.zeros_like(x), w, T.topology(0, t, n, k), seg, 0.0, 0.96)
        assert np.all(np.abs(x.astype(np.float64).mean(0) - mean0) <= 2.0**-23 * np.abs(x).max(0) + 1e-45)
        assert np.all(w == 1.0)   # P14: push-sum weights stay exactly 1 under permutation mixing
    # random weights: sum of w conserved within n 2^-24 max w; z-bar invariant
    rng = np.random.default_rng(0)
    w = rng.uniform(0.5, 2.0, size=(n, k)).astype(F32)
    x, m, _ = _state(n, d, seed=99)
    zb0 = x.astype(np.float64).sum(0) / w.astype(np.float64)[:, seg].sum(0)
    sw0 = w.astype(np.float64).sum(0)
    x2, _, w2 = gossip_step(x, m, np.zeros_like(x), w, T.topology(5, 0, n, k), seg, 0.0, 0.96)
    assert np.all(np.abs(w2.astype(np.float64).sum(0) - sw0) <= n * 2.0**-24 * w.max())
    zb1 = x2.astype(np.float64).sum(0) / w2.astype(np.float64)[:, seg].sum(0)
    assert np.allclose(zb1, zb0, rtol=1e-5, atol=1e-6)


@pytest.mark.parametrize("n", [2, 3, 8, 64])
def test_p11_consensus_contraction_identity(n):
    # S - S' = 1/4 sum_i ||x_i - x_src(i)||^2 per column (exact arithmetic); here in fp64 on fp32
    d, k = 1024, 4
    x, m, _ = _state(n, d, seed=3 * n)
    seg = _segcols(d, k)
    src = T.topology(1, 1, n, k)
    xo, _, _ = gossip_step(x, m, np.zeros_like(x), np.ones((n, k), F32), src, seg, 0.0, 0.96)
    x64, xo64 = x.astype(np.float64), xo.astype(np.float64)
    S = ((x64 - x64.mean(0)) ** 2).sum()
    S1 = ((xo64 - xo64.mean(0)) ** 2).sum()
    xs = np.empty_like(x64)
    for s in range(k):
        cols = seg == s
        xs[:, cols] = x64[src[s]][:, cols]
    rhs = 0.25 * ((x64 - xs) ** 2).sum()
    assert abs((S - S1) - rhs) <= 1e-6 * S
    assert S1 <= S
    if n == 2:
        assert S1 == 0.0


@pytest.mark.parametrize("n", [3, 8, 64])
def test_p11_expected_contraction_ratio(n):
    # iid worker values with variance v: E[S] = (n-1) v and, for any derangement, each
    # x'_i = (x_i + x_src(i))/2 has E[x'_i^2] = v/2, so E[S'] = n v/2 - v and
    # E[S'] / E[S] = (n-2) / (2(n-1)).  A wrong weight or a fixed point moves the ratio
    # (weights (2/3, 1/3) -> (5n-9)/(9(n-1)); src(i) = i -> 1).  For n = 3 every derangement
    # is a 3-cycle C and (I + C)/2 scales the mean-free subspace by |1 + e^{2 pi i/3}|/2 =
    # 1/2, so there S'/S = 1/4 holds column by column, not only on average.
    d, k = 65536, 8
    x = synth.init_params(7 + n, range(n), d)
    seg = _segcols(d, k)
    xo, _, _ = gossip_step(x, np.zeros_like(x), np.zeros_like(x), np.ones((n, k), F32),
                           T.topology(5, 2, n, k), seg, 0.0, 0.96)
    x64, xo64 = x.astype(np.float64), xo.astype(np.float64)
    ratio = ((xo64 - xo64.mean(0)) ** 2).sum() / ((x64 - x64.mean(0)) ** 2).sum()
    assert abs(ratio - (n - 2) / (2 * (n - 1))) <= 0.02 * (n - 2) / (2 * (n - 1))
    if n == 3:
        S = ((x64 - x64.mean(0)) ** 2).sum(0)
        S1 = ((xo64 - xo64.mean(0)) ** 2).sum(0)
        big = S > 1e-3
        assert np.all(np.abs(S1[big] / S[big] - 0.25) <= 1e-5)


def test_p13_identical_workers_follow_torch_sgd():
    # consensus fixed point + equal grads: gossip is the identity, so the trajectory is SGD
    n, d, k, steps = 4, 300, 3, 25
    x0 = synth.hash_uniform(0, 0, 0, d)
    x = np.repeat(x0[None], n, 0)
    m = np.zeros_like(x)
    w = np.ones((n, k), F32)
    seg = _segcols(d, k)
    p = torch.nn.Parameter(torch.from_numpy(x0.copy()))
    opt = torch.optim.SGD([p], lr=0.015625, momentum=0.96)
    for t in range(steps):
        g = synth.hash_uniform(0, 1, t, d) * F32(0.0625)
        x, m, w = gossip_step(x, m, np.repeat(g[None], n, 0), w, T.topology(0, t, n, k), seg, 0.015625, 0.96)
        p.grad = torch.from_numpy(g.copy())
        opt.step()
        assert np.all(x == x[0])
        ref = p.detach().numpy()
        assert np.linalg.norm(x[0] - ref) <= 1e-6 * np.linalg.norm(ref)


def test_local_update_is_heavy_ball_without_fma():
    # mu = 1 - 2^-24, m = 1 + 2^-23, g = -1: exact mu*m = 1 + 2^-24 - 2^-47 rounds to 1.0 in
    # fp32, so the separately-rounded m' is exactly 0; a fused multiply-add would give
    # 2^-24 - 2^-47.  Reading C-10 / SURVEY §7 "bit-exact fp32 op order".
    x = np.array([[1.0]], F32)
    m = np.array([[1.0 + 2.0**-23]], F32)
    g = np.array([[-1.0]], F32)
    m2, y = local_update(x, m, g, 1.0, 1.0 - 2.0**-24)
    assert m2[0, 0] == 0.0
    assert y[0, 0] == 1.0


def test_snapshot_semantics_relabel_equivariance():
    # relabelling workers by pi commutes with the round (no worker-order dependence)
    n, d, k = 7, 200, 3
    x, m, _ = _state(n, d, seed=12)
    g = synth.init_params(13, range(n), d) * F32(0.0625)
    w = np.ones((n, k), F32)
    seg = _segcols(d, k)
    src = T.topology(2, 2, n, k)
    pi = np.array([3, 0, 6, 1, 5, 2, 4])
    inv = np.argsort(pi)
    xo, mo, wo = gossip_step(x, m, g, w, src, seg, 0.015625, 0.96)
    src_r = np.array([[inv[src[s][pi[i]]] for i in range(n)] for s in range(k)], np.int32)
    xr, mr, wr = gossip_step(x[pi], m[pi], g[pi], w[pi], src_r, seg, 0.015625, 0.96)
    assert np.array_equal(xr, xo[pi]) and np.array_equal(mr, mo[pi]) and np.array_equal(wr, wo[pi])


def test_mix_reads_received_segment_of_the_right_peer():
    # a transposed operand (send_to instead of receive_from) fails this: asymmetric 3-cycle
    y = np.array([[1.0], [2.0], [4.0]], F32)
    w = np.ones((3, 1), F32)
    xo, _ = mix(y, w, np.array([[1, 2, 0]], np.int32), np.zeros(1, int))
    assert xo[:, 0].tolist() == [1.5, 3.0, 2.5]


@pytest.mark.parametrize("n", [4, 8, 32])
def test_spec_acceptance5_consensus_decay(n):
    """SPEC.md acceptance 5: pure crossover gossip with 4 segments reaches consensus
    distance < 1e-6 within 60 rounds for >= 99 of 100 seeds, and the distance never
    increases.  In exact arithmetic S' <= S (P11's identity); in fp32 each mixed
    element carries one rounding of at most 2^-24 max|x| (×0.5 is exact), which can move
    CD by at most sqrt(d)·2^-24·max|x| — the only increase allowed."""
    d, k = 128, 4
    seg = _segcols(d, k)
    reached = 0
    for seed in range(100):
        x = synth.init_params(seed, range(n), d)
        m, w = np.zeros_like(x), np.ones((n, k), F32)
        slack = np.sqrt(d) * 2.0 ** -24 * float(np.abs(x).max())
        cd, _ = consensus(x, w, seg)
        for t in range(60):
            x, m, w = gossip_step(x, m, np.zeros_like(x), w, T.topology(seed, t, n, k), seg, 0.0, 0.0)
            cd2, _ = consensus(x, w, seg)
            assert cd2 <= cd + slack, (seed, t, cd, cd2)
            cd = cd2
            if cd < 1e-6:
                reached += 1
                break
    assert reached >= 99, reached
