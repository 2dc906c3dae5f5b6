"""-m gpu: communication-interval mode (Table 1 PAPER.md:230;
SURVEY §8(f) #1).  cs_accumulate against oracle/interval.py, bitwise, and the
whole interval (I micro-steps, then one gossip round with the mean) against the
oracle's Accumulator + gossip_step."""
import numpy as np
import pytest
import torch

import synth
from oracle import topology as T
from oracle.gossip import gossip_step
from oracle.interval import Accumulator

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import __graft_entry__ as entry  # noqa: E402

entry.build()
import paper_2012_15198_b200 as cs  # noqa: E402
from gpu_util import device, device_state, grads_view  # noqa: E402

LR, MU = float(synth.DEFAULT_LR), float(synth.DEFAULT_MOMENTUM)
F32 = np.float32


def _bind(n, d, k, seed, ld):
    cs.cs_init(n, n, k, seed)
    m = torch.zeros(n, ld, device=device())
    cs.cs_bind(m, d, ld, 0, 1, torch.cuda.current_stream())
    return m


def _grads(rng, n, d, ld):
    g = np.zeros((n, ld), F32)
    g[:, :d] = rng.standard_normal((n, d)).astype(F32) * F32(rng.choice([1e-3, 1.0, 1e3]))
    g[0, :min(d, 5)] = [-0.0, 0.0, 2.0**24, -(2.0**24), 1.0][:min(d, 5)]  # signed zeros, cancellation
    return g


@pytest.mark.parametrize("n,d,ld,interval", [(5, 4099, 4100, 3), (3, 1, 4, 1), (8, 1_000_000, 1_000_000, 42),
                                             (2, 33, 36, 2), (2, 300_001, 300_004, 5)])
def test_accumulate_bitwise_padding_untouched(n, d, ld, interval):
    rng = np.random.default_rng(d + interval)
    _bind(n, d, 1, 0, ld)
    acc = torch.full((n, ld), float("nan"), device=device())
    acc[:, :d] = 123.0  # count == 0 must not read it
    orc = Accumulator((n, d), interval)
    for rep in range(2):
        for c in range(interval):
            g = _grads(rng, n, d, ld)
            cs.cs_accumulate(acc, torch.from_numpy(g).to(device()), c, interval)
            out = orc.push(g[:, :d])
            got = acc.cpu().numpy()
            want = orc.acc if out is None else out
            assert np.array_equal(got[:, :d], want), (rep, c)
            assert np.array_equal(np.signbit(got[:, :d]), np.signbit(want)), (rep, c)
            assert np.all(np.isnan(got[:, d:]))


def test_interval_then_gossip_bitwise():
    # I = 3 micro-steps of synthetic gradients, then one flat step with the mean, 3 intervals
    n, d, k, seed, I = 8, 50_003, 4, 7, 3
    ld = (d + 3) // 4 * 4
    cs.cs_init(n, n, k, seed)
    x, m, w, bank2 = device_state(cs, n, d, k, seed, ld=ld)
    cs.cs_bind(m, d, ld, 0, 1, torch.cuda.current_stream())
    acc = torch.empty(n, ld, device=device())
    X = synth.init_params(seed, range(n), d, None)
    M = np.zeros_like(X)
    W = np.ones((n, k), F32)
    bank = synth.grad_bank(seed, n, d)
    seg = T.segment_of_columns(T.segment_bounds(d, k), np.arange(d))
    orc = Accumulator((n, d), I)
    for t in range(3):
        for u in range(I):
            cs.cs_accumulate(acc, grads_view(bank2, n, t * I + u), u, I)
            gbar = orc.push(synth.grads_at(bank, n, t * I + u))
        cs.cs_gossip_step(x, acc, w, LR, MU)
        X, M, W = gossip_step(X, M, gbar, W, T.topology(seed, t, n, k), seg, LR, MU)
        cs.cs_sync()
        assert np.array_equal(acc.cpu().numpy()[:, :d], gbar), t
        assert np.array_equal(m.cpu().numpy()[:, :d], M), t
        assert np.array_equal(x.cpu().numpy()[:, :d], X), t
        assert np.array_equal(w.cpu().numpy(), W), t
    assert cs.cs_get_step() == 3  # one gossip round per interval


def test_accumulate_errors():
    _bind(2, 64, 1, 0, 64)
    acc = torch.zeros(2, 64, device=device())
    g = torch.zeros(2, 64, device=device())
    for count, interval in [(3, 3), (-1, 3), (0, 0), (0, 1 << 24)]:
        with pytest.raises(cs.CSError) as e:
            cs.cs_accumulate(acc, g, count, interval)
        assert e.value.code == -11
    flat = torch.zeros(2 * 64 + 1, device=device())
    with pytest.raises(cs.CSError) as e:
        cs.cs_accumulate(flat[1:], g, 0, 2)
    assert e.value.code == -4
