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
def test_emulated_schedules_agree(schedule):
    # the deferred and split schedules give the same bits (they are not emulated for V > 1
    # on the push path: the library refuses them rather than running them unsafely)
    V, d, k = 2, 10_007, 3
    x, m, w, bank2 = _bind_emulated(V, V, d, k, 9, schedule=schedule)
    with pytest.raises(cs.CSError):
        cs.cs_gossip_step(x, grads_view(bank2, V, 0), w, LR, MU)
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
