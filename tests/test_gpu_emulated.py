"""-m gpu, ONE GPU: the multi-GPU protocol for V ranks emulated on one B200
(cs_test_emulate_ranks).  Same kernels, exchange regions, epoch flags and peer
addressing as across GPUs; every kernel is one cooperative launch whose CTAs are split
among the ranks, so ranks that wait on one another are co-resident.  Compared with the
oracle bit for bit.  This is how the driver's one-GPU box sees the
multi-GPU kernels (VERDICT r01 "What's missing" 1)."""
import numpy as np
import pytest
import torch

import synth
from oracle import topology as T

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import __graft_entry__ as entry  # noqa: E402

entry.build()
import paper_2012_15198_b200 as cs  # noqa: E402
from gpu_util import OracleRun, device_state, grads_view  # noqa: E402

LR, MU = float(synth.DEFAULT_LR), float(synth.DEFAULT_MOMENTUM)


def _bind_emulated(V, n, d, k, seed, groups=None, ld=None, schedule=None):
    ld = (d + 3) // 4 * 4 if ld is None else ld
    cs.cs_init(n, groups or n, k, seed)
    cs.cs_test_emulate_ranks(V)
    if schedule is not None:
        cs.cs_set_schedule(schedule)
    x, m, w, bank2 = device_state(cs, n, d, k, seed, ld=ld)
    cs.cs_bind(m, d, x.shape[1], 0, 1, torch.cuda.current_stream())
    return x, m, w, bank2


def _check(x, m, w, orc, d, cols=None):
    xg, mg = x.cpu().numpy(), m.cpu().numpy()
    if cols is None:
        assert np.array_equal(xg[:, :d], orc.x)
        assert np.array_equal(mg[:, :d], orc.m)
    else:
        assert np.array_equal(xg[:, cols], orc.x)
        assert np.array_equal(mg[:, cols], orc.m)
    assert np.array_equal(w.cpu().numpy(), orc.w)


@pytest.mark.parametrize("V,d,k,ld", [(2, 7, 1, 8), (2, 4099, 3, 4100), (4, 100_003, 4, 100_004),
                                      (8, 65_536, 8, 65_536), (8, 200_001, 16, 200_008), (3, 12_345, 5, 12_348)])
def test_in_step_merge_one_worker_per_rank_bitwise(V, d, k, ld):
    # k_push_merge (default schedule): after each step's work completes -- a plain stream
    # synchronize, no cs_flush / cs_sync -- params and psw hold the merged x', w'
    x, m, w, bank2 = _bind_emulated(V, V, d, k, 17, ld=ld)
    x[:, d:] = 3.0
    orc = OracleRun(V, d, k, 17)
    for t in range(5):
        cs.cs_gossip_step(x, grads_view(bank2, V, t), w, LR, MU)
        orc.step(LR, MU)
        torch.cuda.current_stream().synchronize()
        _check(x, m, w, orc, d)
    name, launches = cs.cs_kernel_info()
    assert name == "k_push_merge" and launches == 1
    assert np.all(x.cpu().numpy()[:, d:] == 3.0)
    cs.cs_sync()
    cs.cs_finalize()


def test_in_step_merge_many_steps_unsynchronised():
    # 40 steps enqueued back to back: the epoch parity ping-pong and the done check
    V, d, k = 4, 30_011, 6
    x, m, w, bank2 = _bind_emulated(V, V, d, k, 5)
    orc = OracleRun(V, d, k, 5)
    for t in range(40):
        cs.cs_gossip_step(x, grads_view(bank2, V, t), w, LR, MU)
        orc.step(LR, MU)
    torch.cuda.synchronize()
    _check(x, m, w, orc, d)
    cs.cs_sync()
    cs.cs_finalize()


@pytest.mark.parametrize("schedule", [1, 2])
@pytest.mark.parametrize("n_loc", [1, 3])
def test_emulated_opt_in_schedules_bitwise(schedule, n_loc):
    # the deferred (merge inside the next step, flushed by cs_sync) and split (push kernel +
    # merge kernel) schedules give the same bits; n_loc = 3 runs the hybrid walk
    V, d, k = 2, 10_007, 3
    n = V * n_loc
    x, m, w, bank2 = _bind_emulated(V, n, d, k, 9, schedule=schedule)
    orc = OracleRun(n, d, k, 9)
    for t in range(6):
        cs.cs_gossip_step(x, grads_view(bank2, n, t), w, LR, MU)
        orc.step(LR, MU)
    cs.cs_sync()
    _check(x, m, w, orc, d)
    cs.cs_finalize()


@pytest.mark.parametrize("V,n_loc,d,k", [(2, 3, 50_001, 5), (4, 4, 30_011, 8), (2, 8, 20_000, 16), (4, 2, 7, 1),
                                         (2, 40, 30_001, 8)])  # world 80 > 64: k_topology tables
def test_emulated_walk_merge_bitwise(V, n_loc, d, k):
    # several workers per rank (default schedule, k_push_merge): the walk mixes local cycles
    # and chains in registers, pushes chain heads to other ranks' inboxes with trailers and
    # merges chain tails in the same kernel -- merged when the step's work completes
    n = V * n_loc
    x, m, w, bank2 = _bind_emulated(V, n, d, k, 4)
    orc = OracleRun(n, d, k, 4)
    for t in range(5):
        cs.cs_gossip_step(x, grads_view(bank2, n, t), w, LR, MU)
        orc.step(LR, MU)
        torch.cuda.current_stream().synchronize()
        _check(x, m, w, orc, d)
    assert cs.cs_kernel_info()[0] == "k_push_merge"
    cs.cs_finalize()


def _hier_check(x, m, w, orc, V, groups, d, cols=None):
    # members hold exact replicas of their leader's params, momentum and psw (reading B-6)
    xg, mg, wg = x.cpu().numpy(), m.cpu().numpy(), w.cpu().numpy()
    cols = np.arange(d) if cols is None else cols
    gs = V // groups
    assert np.array_equal(xg[:, cols], orc.x)
    assert np.array_equal(wg, orc.w)
    for r in range(V):
        lead = (r // gs) * gs
        assert np.array_equal(mg[r, cols], orc.m[lead]), r


@pytest.mark.parametrize("V,groups,d,k", [(2, 1, 100_003, 3), (2, 2, 50_000, 4), (4, 1, 65_536, 2), (4, 2, 70_001, 5),
                                          (4, 4, 40_003, 6), (8, 2, 1_000_003, 16), (8, 4, 30_001, 3)])
def test_emulated_hierarchical_bitwise(V, groups, d, k):
    # PAPER.md:197 across ranks: reduce-scatter of the gradient (k_hier_scatter), ascending
    # sum x fp32(1/|G|) and all-gather (k_hier_reduce), replica sync (k_hier_sync), then the
    # leaders' exchange merged in the same kernel (k_push_merge) or, with one group, the
    # update alone.  (8, 2): BASELINE configs[3]'s 2 groups x 4 layout.
    x, m, w, bank2 = _bind_emulated(V, V, d, k, 11, groups=groups)
    orc = OracleRun(V, d, k, 11, groups=groups)
    for t in range(4):
        cs.cs_hier_step(x, grads_view(bank2, V, t), w, LR, MU)
        orc.step(LR, MU)
        torch.cuda.current_stream().synchronize()
        _hier_check(x, m, w, orc, V, groups, d)
    cs.cs_finalize()


def test_emulated_hierarchical_configs3_full_size_sampled():
    # BASELINE configs[3] exactly: 8 ranks as 2 groups x 4, ResNet-50-sized (25,557,032), k = 16
    V, groups, d, k = 8, 2, 25_557_032, 16
    x, m, w, bank2 = _bind_emulated(V, V, d, k, 0, groups=groups)
    cols = synth.sample_columns(d, T.segment_bounds(d, k))
    orc = OracleRun(V, d, k, 0, cols=cols, groups=groups)
    for t in range(3):
        cs.cs_hier_step(x, grads_view(bank2, V, t), w, LR, MU)
        orc.step(LR, MU)
    torch.cuda.synchronize()
    _hier_check(x, m, w, orc, V, groups, d, cols=cols)
    cs.cs_finalize()


def test_emulated_flat_after_hierarchical_resyncs_members():
    # a flat step between hierarchical steps gives members their own state; the
    # next hierarchical step must re-replicate the leaders before using member replicas
    V, groups, d, k = 4, 2, 20_011, 3
    x, m, w, bank2 = _bind_emulated(V, V, d, k, 2, groups=groups)
    orc = OracleRun(V, d, k, 2, groups=groups)
    from oracle.gossip import gossip_step
    from oracle.hierarchical import hier_step
    for t, kind in enumerate(["h", "f", "h", "h"]):
        g = synth.grads_at(orc.bank, V, t)
        if kind == "h":
            cs.cs_hier_step(x, grads_view(bank2, V, t), w, LR, MU)
            orc.x, orc.m, orc.w, _ = hier_step(orc.x, orc.m, g, orc.w, groups, 2, t, k, orc.seg, LR, MU)
            # reading B-6: across ranks every member holds its leader's momentum (the oracle
            # leaves members' rows untouched), so the flat step after it starts from replicas
            gs = V // groups
            orc.m = np.repeat(orc.m[::gs], gs, axis=0)
        else:
            cs.cs_gossip_step(x, grads_view(bank2, V, t), w, LR, MU)
            orc.x, orc.m, orc.w = gossip_step(orc.x, orc.m, g, orc.w, T.topology(2, t, V, k), orc.seg, LR, MU)
        orc.t += 1
    torch.cuda.synchronize()
    assert np.array_equal(x.cpu().numpy()[:, :d], orc.x)
    assert np.array_equal(w.cpu().numpy(), orc.w)
    cs.cs_finalize()


@pytest.mark.parametrize("V,n_loc,groups", [(2, 1, 0), (4, 3, 0), (4, 1, 2), (2, 1, 1)])
def test_emulated_diagnostics(V, n_loc, groups):
    # multi-rank diagnostics (k_diag_scatter/reduce/final): column chunks per rank,
    # rank-ordered partials, within 1e-9 of the oracle (fp64, another summation order)
    from oracle.diagnostics import consensus
    n, d, k = V * n_loc, 40_003, 4
    x, m, w, bank2 = _bind_emulated(V, n, d, k, 6, groups=groups or None)
    orc = OracleRun(n, d, k, 6, groups=groups or None)
    cs.cs_set_diag(True)
    step = cs.cs_hier_step if groups else cs.cs_gossip_step
    for t in range(3):
        step(x, grads_view(bank2, n, t), w, LR, MU)
        orc.step(LR, MU)
        cd, ms = cs.cs_get_diag()
        cd0, ms0 = consensus(orc.x, orc.w, orc.seg)
        assert abs(cd - cd0) <= 1e-9 * abs(cd0), (t, cd, cd0)
        assert abs(ms - ms0) <= 1e-9 * max(1.0, abs(ms0)) + 1e-9 * d, (t, ms, ms0)
    cs.cs_set_diag(False)
    cs.cs_finalize()


@pytest.mark.parametrize("groups", [0, 1, 2])
def test_emulated_lars(groups):
    # LARS (C-18) on the in-step merge kernel (flat) and on the hierarchical step's group
    # mean: rates within 1 ulp, params and momentum within 1e-6 (fp64 norm sums
    # in another order), layer-plan segments
    from oracle.lars import lars_gossip_step, lars_hier_step, plan_bounds, segment_plan
    V, d, k = 2, 120_000, 4
    ETA, WD, EPS, lr = 0.0025, 5e-5, 1e-9, 9.0
    x, m, w, bank2 = _bind_emulated(V, V, d, k, 8, groups=groups or None)
    rng = np.random.default_rng(10)
    lb = np.concatenate([[0], np.unique(rng.integers(1, d // 4, size=9) * 4), [d]]).astype(np.int64)
    plan = segment_plan(np.diff(lb).tolist(), k)
    cs.cs_set_layers(lb, plan)
    cs.cs_set_lars(ETA, WD, EPS)
    orc = OracleRun(V, d, k, 8)
    orc.seg = T.segment_of_columns(plan_bounds(lb, plan), orc.cols)
    for t in range(4):
        g = synth.grads_at(orc.bank, V, t)
        if groups:
            cs.cs_hier_step(x, grads_view(bank2, V, t), w, lr, MU)
            orc.x, orc.m, orc.w, lrs = lars_hier_step(orc.x, orc.m, g, orc.w, groups, 8, t, k, orc.seg, lb, lr, MU,
                                                      ETA, WD, EPS)
        else:
            cs.cs_gossip_step(x, grads_view(bank2, V, t), w, lr, MU)
            orc.x, orc.m, orc.w, lrs = lars_gossip_step(orc.x, orc.m, g, orc.w, T.topology(8, t, V, k), orc.seg, lb,
                                                        lr, MU, ETA, WD, EPS)
        orc.t += 1
        got = cs.cs_get_lars_rates(V, len(lb) - 1)
        want = lrs if not groups else np.repeat(lrs, V // groups, axis=0)
        assert np.all(np.abs(got.astype(np.float64) - want) <= np.spacing(np.abs(want))), t
        xg, mg = x.cpu().numpy()[:, :d], m.cpu().numpy()[:, :d]
        assert np.all(np.abs(xg - orc.x) <= 1e-6 * np.abs(orc.x).max(axis=1, keepdims=True)), t
        mref = orc.m if not groups else np.repeat(orc.m[::V // groups], V // groups, axis=0)
        assert np.all(np.abs(mg - mref) <= 1e-6 * np.abs(mref).max(axis=1, keepdims=True)), t
    cs.cs_set_lars(0.0)
    cs.cs_finalize()


def test_in_step_merge_resnet50_pair_sampled():
    # BASELINE configs[2] layout (25,557,032, k = 8) for two emulated ranks, 6 steps,
    # sampled columns (every segment boundary +-2, 1/1024 stride, the tail)
    V, d, k = 2, 25_557_032, 8
    x, m, w, bank2 = _bind_emulated(V, V, d, k, 0)
    cols = synth.sample_columns(d, T.segment_bounds(d, k))
    orc = OracleRun(V, d, k, 0, cols=cols)
    for t in range(6):
        cs.cs_gossip_step(x, grads_view(bank2, V, t), w, LR, MU)
        orc.step(LR, MU)
    torch.cuda.synchronize()
    idx = torch.from_numpy(cols).cuda()
    assert np.array_equal(x.index_select(1, idx).cpu().numpy(), orc.x)
    assert np.array_equal(m.index_select(1, idx).cpu().numpy(), orc.m)
    assert np.array_equal(w.cpu().numpy(), orc.w)
    cs.cs_finalize()


def test_in_step_merge_exponential_and_bf16_wire():
    V, d, k = 4, 20_003, 1
    x, m, w, bank2 = _bind_emulated(V, V, d, k, 3)
    cs.cs_set_topology_kind(cs.TOPO_EXPONENTIAL)
    cs.cs_set_wire(cs.WIRE_BF16)
    orc = OracleRun(V, d, k, 3)
    from oracle.sgp import exponential_topology
    for t in range(5):
        cs.cs_gossip_step(x, grads_view(bank2, V, t), w, LR, MU)
        orc.step(LR, MU, src=exponential_topology(t, V, k), wire="bf16")
    torch.cuda.synchronize()
    _check(x, m, w, orc, d)
    cs.cs_set_wire(cs.WIRE_FP32)
    cs.cs_set_topology_kind(cs.TOPO_CROSSOVER)
    cs.cs_finalize()
