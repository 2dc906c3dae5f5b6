"""-m gpu: layer-table segment plan and LARS (Table 1
PAPER.md:225-233) through the C-ABI, against oracle/lars.py.

The plan without LARS is bitwise.  With LARS, the per-layer norms are fp64 sums in a
different order from the oracle's, so the fp32 rates agree to 1 ulp and the parameters
to the north_star tolerance (1e-6 relative); in practice they are bitwise."""
import numpy as np
import pytest
import torch

import synth
from oracle import topology as T
from oracle.diagnostics import consensus
from oracle.gossip import gossip_step
from oracle.lars import lars_gossip_step, plan_bounds, segment_plan

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import __graft_entry__ as entry  # noqa: E402

entry.build()
import paper_2012_15198_b200 as cs  # noqa: E402
from gpu_util import device, device_state, grads_view  # noqa: E402

LR, MU = float(synth.DEFAULT_LR), float(synth.DEFAULT_MOMENTUM)
ETA, WD, EPS = 0.0025, 5e-5, 1e-9   # Table 1
F32 = np.float32


def _layers(seed, L, lo=1, hi=400):
    rng = np.random.default_rng(seed)
    sizes = [int(v) * 4 for v in rng.integers(lo, hi, size=L)]
    return sizes, np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)


def _setup(n, sizes, lb, k, seed, plan=True):
    d = int(lb[-1])
    ld = (d + 3) // 4 * 4
    cs.cs_init(n, n, k, seed)
    x, m, w, bank2 = device_state(cs, n, d, k, seed, ld=ld)
    cs.cs_bind(m, d, ld, 0, 1, torch.cuda.current_stream())
    sol = segment_plan(sizes, k) if plan else None
    cs.cs_set_layers(lb, sol)
    b = plan_bounds(lb, sol) if plan else T.segment_bounds(d, k)
    seg = T.segment_of_columns(b, np.arange(d))
    X = synth.init_params(seed, range(n), d)
    return d, x, m, w, bank2, X, seg


def _ulp_close(a, b):
    return np.all(np.abs(a.astype(np.float64) - b) <= np.spacing(np.abs(b)).astype(np.float64))


@pytest.mark.parametrize("n,L,k", [(8, 40, 6), (5, 13, 13), (16, 161, 18), (3, 7, 1)])
def test_layer_plan_bitwise(n, L, k):
    sizes, lb = _layers(L, L)
    d, x, m, w, bank2, X, seg = _setup(n, sizes, lb, k, 11)
    cs.cs_set_lars(0.0)
    M, W = np.zeros_like(X), np.ones((n, k), F32)
    bank = synth.grad_bank(11, n, d)
    for t in range(6):
        cs.cs_gossip_step(x, grads_view(bank2, n, t), w, LR, MU)
        X, M, W = gossip_step(X, M, synth.grads_at(bank, n, t), W, T.topology(11, t, n, k), seg, LR, MU)
    cs.cs_sync()
    assert np.array_equal(x.cpu().numpy()[:, :d], X)
    assert np.array_equal(m.cpu().numpy()[:, :d], M)
    assert np.array_equal(w.cpu().numpy(), W)


@pytest.mark.parametrize("n,L,k,plan,diag,carry", [(8, 40, 6, True, False, False), (6, 25, 4, False, True, True),
                                                   (16, 161, 18, True, True, True), (2, 3, 2, True, False, False)])
def test_lars_matches_oracle(n, L, k, plan, diag, carry):
    sizes, lb = _layers(100 + L, L)
    seed = 5
    d, x, m, w, bank2, X, seg = _setup(n, sizes, lb, k, seed, plan)
    cs.cs_set_lars(ETA, WD, EPS)
    cs.cs_set_lars_carry(carry)
    cs.cs_set_diag(diag)
    M, W = np.zeros_like(X), np.ones((n, k), F32)
    bank = synth.grad_bank(seed, n, d)
    lr = 9.0  # Table 1 "Learning rate 9" (with LARS, lrs = lr * scale)
    bitwise = True
    for t in range(10):
        cs.cs_gossip_step(x, grads_view(bank2, n, t), w, lr, MU)
        X, M, W, lrs = lars_gossip_step(X, M, synth.grads_at(bank, n, t), W, T.topology(seed, t, n, k), seg,
                                        lb, lr, MU, ETA, WD, EPS)
        got = cs.cs_get_lars_rates(n, L)
        assert _ulp_close(got, lrs), t
        bitwise &= np.array_equal(got, lrs)
        xg = x.cpu().numpy()[:, :d]
        scale = np.abs(X).max(axis=1, keepdims=True)
        assert np.all(np.abs(xg - X) <= 1e-6 * scale), t
        mg = m.cpu().numpy()[:, :d]  # momentum to the same tolerance
        assert np.all(np.abs(mg - M) <= 1e-6 * np.abs(M).max(axis=1, keepdims=True)), t
        assert np.array_equal(w.cpu().numpy(), W)
        if diag:
            cd, ms = cs.cs_get_diag()
            cd0, ms0 = consensus(xg, w.cpu().numpy(), seg)
            assert abs(cd - cd0) <= 1e-9 * abs(cd0) and abs(ms - ms0) <= 1e-9 * max(1.0, abs(ms0))
    cs.cs_set_diag(False)
    cs.cs_set_lars(0.0)
    cs.cs_set_lars_carry(False)
    if bitwise:  # the usual outcome: the parameters are then identical too
        assert np.array_equal(x.cpu().numpy()[:, :d], X)
        assert np.array_equal(m.cpu().numpy()[:, :d], M)


@pytest.mark.parametrize("carry", [False, True])
def test_lars_params_modified_between_steps(carry):
    # SPEC.md:368-376 / PAPER.md:35: the rates come from this step's x.  The caller rescales
    # params in place between LARS steps (a checkpoint load or manual decay); by default the
    # library recomputes ||x|| every step, and with the opt-in carry cs_params_modified()
    # tells it to (the carry used to trust the pointer alone)
    n, L, k, seed = 6, 20, 4, 12
    sizes, lb = _layers(500 + L, L)
    d, x, m, w, bank2, X, seg = _setup(n, sizes, lb, k, seed)
    cs.cs_set_lars(ETA, WD, EPS)
    cs.cs_set_lars_carry(carry)
    M, W = np.zeros_like(X), np.ones((n, k), F32)
    bank = synth.grad_bank(seed, n, d)
    for t in range(6):
        if t in (2, 4):
            x.mul_(0.5)          # an outside in-place write of params
            torch.cuda.synchronize()
            X = (X * F32(0.5)).astype(F32)
            if carry:
                cs.cs_params_modified()
        cs.cs_gossip_step(x, grads_view(bank2, n, t), w, 9.0, MU)
        X, M, W, lrs = lars_gossip_step(X, M, synth.grads_at(bank, n, t), W, T.topology(seed, t, n, k), seg,
                                        lb, 9.0, MU, ETA, WD, EPS)
        assert _ulp_close(cs.cs_get_lars_rates(n, L), lrs), t
    assert np.all(np.abs(x.cpu().numpy()[:, :d] - X) <= 1e-6 * np.abs(X).max(axis=1, keepdims=True))
    cs.cs_set_lars(0.0)
    cs.cs_set_lars_carry(False)


@pytest.mark.parametrize("hybrid,plan", [(1, True), (0, True), (1, False)])
def test_lars_and_layer_plan_on_the_peer_kernels(hybrid, plan, monkeypatch):
    # the multi-GPU kernels in single-GPU emulation: hybrid walk (several workers per GPU)
    # or push/mix, with a layer table (and plan) and LARS; 10 steps, no sync in between
    monkeypatch.setenv("CS_PEER_HYBRID", str(hybrid))
    n, L, k, seed = 6, 30, 5, 4
    sizes, lb = _layers(200 + L, L)
    d = int(lb[-1])
    ld = (d + 3) // 4 * 4
    cs.cs_init(n, n, k, seed)
    cs.cs_set_path(3)
    x, m, w, bank2 = device_state(cs, n, d, k, seed, ld=ld)
    cs.cs_bind(m, d, ld, 0, 1, torch.cuda.current_stream())
    sol = segment_plan(sizes, k) if plan else None
    cs.cs_set_layers(lb, sol)
    cs.cs_set_lars(ETA, WD, EPS)
    seg = T.segment_of_columns(plan_bounds(lb, sol) if plan else T.segment_bounds(d, k), np.arange(d))
    X = synth.init_params(seed, range(n), d)
    M, W = np.zeros_like(X), np.ones((n, k), F32)
    bank = synth.grad_bank(seed, n, d)
    for t in range(10):
        cs.cs_gossip_step(x, grads_view(bank2, n, t), w, 9.0, MU)
        X, M, W, lrs = lars_gossip_step(X, M, synth.grads_at(bank, n, t), W, T.topology(seed, t, n, k), seg,
                                        lb, 9.0, MU, ETA, WD, EPS)
    assert _ulp_close(cs.cs_get_lars_rates(n, L), lrs)
    cs.cs_sync()
    assert np.all(np.abs(x.cpu().numpy()[:, :d] - X) <= 1e-6 * np.abs(X).max(axis=1, keepdims=True))
    assert np.array_equal(w.cpu().numpy(), W)
    cs.cs_set_lars(0.0)
    cs.cs_set_path(0)


@pytest.mark.parametrize("groups,lars", [(2, False), (4, False), (2, True), (1, True)])
def test_hierarchical_one_gpu_layers_and_lars(groups, lars):
    # single-GPU hierarchical kernel with a layer plan (bitwise) and LARS on the group mean
    # (rates within 1 ulp, parameters within 1e-6)
    from oracle.hierarchical import hier_step
    from oracle.lars import lars_hier_step
    n, L, k, seed = 8, 20, 4, 6
    sizes, lb = _layers(300 + L, L)
    d = int(lb[-1])
    ld = (d + 3) // 4 * 4
    cs.cs_init(n, groups, k, seed)
    x, m, w, bank2 = device_state(cs, n, d, k, seed, ld=ld)
    cs.cs_bind(m, d, ld, 0, 1, torch.cuda.current_stream())
    sol = segment_plan(sizes, k)
    cs.cs_set_layers(lb, sol)
    if lars:
        cs.cs_set_lars(ETA, WD, EPS)
    seg = T.segment_of_columns(plan_bounds(lb, sol), np.arange(d))
    X = synth.init_params(seed, range(n), d)
    M, W = np.zeros_like(X), np.ones((n, k), F32)
    bank = synth.grad_bank(seed, n, d)
    lr = 9.0 if lars else LR
    for t in range(6):
        cs.cs_hier_step(x, grads_view(bank2, n, t), w, lr, MU)
        if lars:
            X, M, W, lrs = lars_hier_step(X, M, synth.grads_at(bank, n, t), W, groups, seed, t, k, seg, lb, lr, MU,
                                          ETA, WD, EPS)
            assert _ulp_close(cs.cs_get_lars_rates(n, L)[:groups], lrs), t
        else:
            X, M, W, _ = hier_step(X, M, synth.grads_at(bank, n, t), W, groups, seed, t, k, seg, lr, MU)
    cs.cs_sync()
    xg = x.cpu().numpy()[:, :d]
    leaders = list(range(0, n, n // groups))
    if lars:
        assert np.all(np.abs(xg - X) <= 1e-6 * np.abs(X).max(axis=1, keepdims=True))
    else:
        assert np.array_equal(xg, X)
        assert np.array_equal(m.cpu().numpy()[leaders, :d], M[leaders])
    assert np.array_equal(w.cpu().numpy(), W)
    cs.cs_set_lars(0.0)


def test_lars_resnet50_blocks_plan():
    # the paper's setting: ResNet-50's 161 tensors, segments = stem + 16 blocks + FC (k = 18)
    sizes, block = synth.resnet50_layers()
    lb = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    n, k, seed, d = 4, 18, 2, int(lb[-1])
    cs.cs_init(n, n, k, seed)
    x, m, w, bank2 = device_state(cs, n, d, k, seed, ld=d)
    cs.cs_bind(m, d, d, 0, 1, torch.cuda.current_stream())
    cs.cs_set_layers(lb, block)
    cs.cs_set_lars(ETA, WD, EPS)
    seg = T.segment_of_columns(plan_bounds(lb, block), np.arange(d))
    X = synth.init_params(seed, range(n), d)
    M, W = np.zeros_like(X), np.ones((n, k), F32)
    bank = synth.grad_bank(seed, n, d)
    for t in range(3):
        cs.cs_gossip_step(x, grads_view(bank2, n, t), w, 9.0, MU)
        X, M, W, lrs = lars_gossip_step(X, M, synth.grads_at(bank, n, t), W, T.topology(seed, t, n, k), seg,
                                        lb, 9.0, MU, ETA, WD, EPS)
        assert _ulp_close(cs.cs_get_lars_rates(n, 161), lrs), t
    xg = x.cpu().numpy()
    assert np.all(np.abs(xg - X) <= 1e-6 * np.abs(X).max(axis=1, keepdims=True))
    cs.cs_set_lars(0.0)


def test_layer_table_errors():
    n, d, k = 4, 1024, 2
    cs.cs_init(n, n, k, 0)
    m = torch.zeros(n, d, device=device())
    cs.cs_bind(m, d, d, 0, 1, torch.cuda.current_stream())
    x, w, g = torch.zeros(n, d, device=device()), torch.ones(n, k, device=device()), torch.zeros(n, d, device=device())
    cs.cs_set_lars(ETA, WD, EPS)
    with pytest.raises(cs.CSError) as e:           # LARS without a layer table
        cs.cs_gossip_step(x, g, w, LR, MU)
    assert e.value.code == -11
    for lb, seg, code in [([0, 6, 1024], None, -4),               # bound not a multiple of 4
                          ([0, 512, 1000], None, -4),             # does not end at d
                          ([0, 512, 512, 1024], None, -4),        # empty layer
                          ([0, 512, 1024], [0, 0], -3),           # seg_of_layer must reach k-1
                          ([0, 256, 512, 1024], [0, 2, 1], -3)]:  # not contiguous
        with pytest.raises(cs.CSError) as e:
            cs.cs_set_layers(lb, seg)
        assert e.value.code == code, (lb, seg)
    cs.cs_set_layers([0, 512, 1024], [0, 1])
    cs.cs_gossip_step(x, g, w, LR, MU)
    cs.cs_init(n, 2, k, 0)
    cs.cs_set_path(1)                              # the register path has no layer tiles
    cs.cs_bind(m, d, d, 0, 1, torch.cuda.current_stream())
    with pytest.raises(cs.CSError) as e:
        cs.cs_set_layers([0, 512, 1024], [0, 1])
    assert e.value.code == -12
    cs.cs_set_path(0)
    with pytest.raises(cs.CSError):
        cs.cs_set_lars(-1.0)
    cs.cs_set_lars(0.0)
