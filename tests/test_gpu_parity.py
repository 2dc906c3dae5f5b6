"""-m gpu: the CUDA path (through the C-ABI) against the oracle on identical seeded inputs.

Contract: topology and routing bit-exact; flat params, momentum and
push-sum weights bit-exact (same fp32 op order, no FMA) with a norm-wise 1e-6
backstop; hierarchical bit-exact on one GPU (same ascending sum order);
diagnostics within 1e-9 relative (fp64, different reduction order)."""
import numpy as np
import pytest
import torch

import synth
from oracle import topology as T
from oracle.diagnostics import consensus
from oracle.gossip import gossip_step

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # collected on CPU boxes too; skip cleanly there
    pytest.skip("needs a CUDA device", allow_module_level=True)

import __graft_entry__ as entry  # noqa: E402

entry.build()
import paper_2012_15198_b200 as cs  # noqa: E402
from gpu_util import OracleRun, device, device_state, grads_view, rel_norm_err  # noqa: E402

LR, MU = float(synth.DEFAULT_LR), float(synth.DEFAULT_MOMENTUM)


def _bind(n, d, k, seed, groups=None, ld=None, path=None, sched=None):
    ld = (d + 3) // 4 * 4 if ld is None else ld
    cs.cs_init(n, groups or n, k, seed)
    if sched is not None:
        cs.cs_set_schedule(sched)
    if path is not None:
        cs.cs_set_path(path)
    x, m, w, bank2 = device_state(cs, n, d, k, seed, ld=ld)
    cs.cs_bind(m, d, x.shape[1], 0, 1, torch.cuda.current_stream())
    return x, m, w, bank2


def test_synth_generator_bit_exact():
    for d, rows, row0, tag in [(1000, 3, 0, 0), (4097, 2, 5, 1), (33, 7, 100, 1)]:
        out = torch.zeros(rows, d + 3, device=device())
        cs.cs_synth_fill(out, rows, d, d + 3, 11, tag, row0, 0.0625)
        got = out.cpu().numpy()
        for r in range(rows):
            assert np.array_equal(got[r, :d], synth.hash_uniform(11, tag, row0 + r, d) * np.float32(0.0625))
            assert np.all(got[r, d:] == 0)


@pytest.mark.parametrize("n,k", [(2, 3), (3, 8), (5, 4), (8, 32), (16, 8), (33, 2), (64, 32),
                                 (100, 2), (257, 1), (1024, 1)])
def test_device_topology_bit_exact(n, k):
    cs.cs_init(n, 1, k, 0x0123456789ABCDEF)
    m = torch.zeros(1, 32 * k, device=device())
    cs.cs_bind(m, 32 * k, 32 * k, 0, 1, torch.cuda.current_stream())
    for step in [0, 1, 17, 123456, 2**32 - 1]:
        dev = cs.cs_test_device_topology(step, n, k)
        assert np.array_equal(dev, cs.cs_topology(step, n, k)), (n, k, step)
        # the oracle directly for every n (n = 128, 257, 1024 were only compared
        # with the host C++ generator); pure-Python Alg. 2, a second or so at n = 1024
        assert np.array_equal(dev, T.topology(0x0123456789ABCDEF, step, n, k)), (n, k, step)


def test_device_hier_topology_bit_exact():
    cs.cs_init(32, 8, 4, 5)
    m = torch.zeros(1, 128, device=device())
    cs.cs_bind(m, 128, 128, 0, 1, torch.cuda.current_stream())
    for step in range(10):
        assert np.array_equal(cs.cs_test_device_topology(step, 8, 4, cs.CS_TAG_HIER),
                              T.topology(5, step, 8, 4, T.TAG_HIER))


def test_config1_full_bitwise_every_step():
    # BASELINE.json configs[0]: 8 workers, 1M params, k=4, 10 steps, seed 0
    n, d, k, seed, steps = 8, 1_000_000, 4, 0, 10
    x, m, w, bank2 = _bind(n, d, k, seed)
    orc = OracleRun(n, d, k, seed)
    assert np.array_equal(x.cpu().numpy(), orc.x)
    for t in range(steps):
        cs.cs_gossip_step(x, grads_view(bank2, n, t), w, LR, MU)
        cs.cs_sync()
        orc.step(LR, MU)
        xg, mg, wg = x.cpu().numpy(), m.cpu().numpy(), w.cpu().numpy()
        assert np.array_equal(mg, orc.m), t
        assert np.array_equal(xg, orc.x), t
        assert np.array_equal(wg, orc.w), t
    assert rel_norm_err(xg, orc.x).max() <= 1e-6


@pytest.mark.parametrize("n,d,k,ld", [(2, 1, 1, 4), (2, 7, 1, 8), (3, 95, 3, 96), (5, 4099, 7, 4100),
                                      (33, 1000, 4, 1024), (4, 33, 2, 36), (16, 32 * 8, 8, 256),
                                      (7, 12345, 5, 12348)])
def test_ragged_shapes_bitwise_and_padding_untouched(n, d, k, ld):
    x, m, w, bank2 = _bind(n, d, k, 3, ld=ld)
    x[:, d:] = 7.0
    m[:, d:] = -7.0
    orc = OracleRun(n, d, k, 3)
    for t in range(5):
        cs.cs_gossip_step(x, grads_view(bank2, n, t), w, LR, MU)
        orc.step(LR, MU)
    cs.cs_sync()
    xg, mg = x.cpu().numpy(), m.cpu().numpy()
    assert np.array_equal(xg[:, :d], orc.x)
    assert np.array_equal(mg[:, :d], orc.m)
    assert np.array_equal(w.cpu().numpy(), orc.w)
    assert np.all(xg[:, d:] == 7.0) and np.all(mg[:, d:] == -7.0)


@pytest.mark.parametrize("n,k", [(2, 1), (3, 2), (8, 4), (16, 8), (33, 5), (64, 32)])
def test_p9_routing_probe_on_device(n, k):
    d = 32 * k * 3 + 12
    cs.cs_init(n, n, k, 21)
    x = torch.arange(n, dtype=torch.float32, device=device())[:, None].repeat(1, d).contiguous()
    m = torch.zeros_like(x)
    g = torch.zeros_like(x)
    w = torch.ones(n, k, device=device())
    cs.cs_bind(m, d, d, 0, 1, torch.cuda.current_stream())
    b = T.segment_bounds(d, k)
    for step in range(3):
        x[:] = torch.arange(n, dtype=torch.float32, device=device())[:, None]
        cs.cs_gossip_step(x, g, w, 0.0, 0.5)
        cs.cs_sync()
        dec = 2 * x.cpu().numpy() - np.arange(n, dtype=np.float32)[:, None]
        src = cs.cs_topology(step, n, k)
        assert np.array_equal(src, T.topology(21, step, n, k))
        for s in range(k):
            assert np.all(dec[:, b[s]:b[s + 1]] == src[s][:, None]), (step, s)


def test_p6_worked_kat_with_injected_topology():
    import json, os
    from conftest import GOLDEN
    gold = json.load(open(os.path.join(GOLDEN, "p6_worked_kat.json")))
    n, k, d = gold["n"], gold["k"], gold["d"]
    cs.cs_init(n, n, k, 0)
    dev = device()
    x = torch.tensor(gold["x0_per_worker"], device=dev)[:, None].repeat(1, d).contiguous()
    g = torch.tensor(gold["grad_per_worker"], device=dev)[:, None].repeat(1, d).contiguous()
    m = torch.zeros_like(x)
    w = torch.ones(n, k, device=dev)
    cs.cs_bind(m, d, d, 0, 1, torch.cuda.current_stream())
    for t in ("0", "1"):
        cs.cs_test_set_topology(np.array(gold["topology"][t], np.int32))
        cs.cs_gossip_step(x, g, w, gold["lr"], gold["momentum"])
        cs.cs_sync()
        e = gold["expected"][t]
        xg = x.cpu().numpy()
        assert np.all(xg[:, :32] == np.array(e["seg0"], np.float32)[:, None])
        assert np.all(xg[:, 32:] == np.array(e["seg1"], np.float32)[:, None])
        assert np.all(m.cpu().numpy()[:, 0] == np.array(e["m"], np.float32))
    cs.cs_test_set_topology(None)
    with pytest.raises(cs.CSError) as err:
        cs.cs_test_set_topology(np.array([[0, 2, 1], [1, 2, 0]], np.int32))
    assert err.value.code == -6


def test_xor_butterfly_is_allreduce_on_device():
    # P7 through the C-ABI: after log2(n) injected XOR rounds all workers are bitwise equal
    n, d, r = 16, 4096, 4
    x, m, w, _ = _bind(n, d, 1, 8)
    zero = torch.zeros_like(x)
    exact = x.double().mean(0).cpu().numpy()
    for t in range(r):
        cs.cs_test_set_topology(np.array([[i ^ (1 << t) for i in range(n)]], np.int32))
        cs.cs_gossip_step(x, zero, w, 0.0, 0.96)
    cs.cs_sync()
    xg = x.cpu().numpy()
    assert np.all(xg == xg[0])
    assert np.abs(xg[0] - exact).max() <= 2.0**-23 * np.abs(exact).max()


@pytest.mark.parametrize("n,d,k", [(8, 100_000, 4), (3, 5000, 2), (16, 65536 + 7, 8)])
def test_diagnostics_match_oracle(n, d, k):
    x, m, w, bank2 = _bind(n, d, k, 4)
    orc = OracleRun(n, d, k, 4)
    cs.cs_set_diag(True)
    for t in range(4):
        cs.cs_gossip_step(x, grads_view(bank2, n, t), w, LR, MU)
        orc.step(LR, MU)
        cd, ms = cs.cs_get_diag()
        cd0, ms0 = consensus(orc.x, orc.w, orc.seg)
        assert abs(cd - cd0) <= 1e-9 * abs(cd0), (t, cd, cd0)
        assert abs(ms - ms0) <= 1e-9 * max(1.0, abs(ms0)) + 1e-9 * d, (t, ms, ms0)
    cs.cs_set_diag(False)


def test_diagnostics_with_nonunit_weights_and_consensus():
    n, d, k = 6, 3000, 3
    x, m, w, bank2 = _bind(n, d, k, 6)
    rng = np.random.default_rng(0)
    w0 = rng.uniform(0.5, 2.0, size=(n, k)).astype(np.float32)
    w.copy_(torch.from_numpy(w0))
    orc = OracleRun(n, d, k, 6)
    orc.w = w0.copy()
    cs.cs_set_diag(True)
    for t in range(3):
        cs.cs_gossip_step(x, grads_view(bank2, n, t), w, LR, MU)
        orc.step(LR, MU)
    cd, ms = cs.cs_get_diag()
    cd0, ms0 = consensus(orc.x, orc.w, orc.seg)
    assert np.array_equal(w.cpu().numpy(), orc.w)
    assert abs(cd - cd0) <= 1e-9 * cd0 and abs(ms - ms0) <= 1e-9 * abs(ms0) + 1e-9
    # consensus input, lr = 0 -> CD = 0 exactly
    x[:] = x[0:1].clone()
    w.fill_(1.0)
    cs.cs_gossip_step(x, torch.zeros_like(x), w, 0.0, 0.0)
    cd, _ = cs.cs_get_diag()
    assert cd == 0.0
    cs.cs_set_diag(False)


@pytest.mark.parametrize("n,G,k", [(8, 2, 4), (16, 4, 8), (12, 3, 2), (6, 1, 2), (6, 6, 3), (4, 2, 1)])
def test_hierarchical_single_gpu_bitwise(n, G, k):
    d = 20_000 + 3
    x, m, w, bank2 = _bind(n, d, k, 12, groups=G, ld=d + 1)
    orc = OracleRun(n, d, k, 12, groups=G)
    gs = n // G
    lead = list(range(0, n, gs))
    for t in range(4):
        cs.cs_hier_step(x, grads_view(bank2, n, t), w, LR, MU)
        orc.step(LR, MU)
    cs.cs_sync()
    xg = x.cpu().numpy()[:, :d]
    assert np.array_equal(xg, orc.x)
    assert np.array_equal(m.cpu().numpy()[lead, :d], orc.m[lead])
    assert np.array_equal(w.cpu().numpy(), orc.w)
    for grp in range(G):
        assert np.all(xg[grp * gs:(grp + 1) * gs] == xg[grp * gs])


def test_p12_hier_hand_kat_on_device():
    import json, os
    from conftest import GOLDEN
    gold = json.load(open(os.path.join(GOLDEN, "p12_hier_kat.json")))
    n, G, k, d = gold["n"], gold["groups"], gold["k"], gold["d"]
    cs.cs_init(n, G, k, 0)
    dev = device()
    x = torch.tensor(gold["x0_per_worker"], device=dev)[:, None].repeat(1, d).contiguous()
    g = torch.tensor(gold["grad_per_worker"], device=dev)[:, None].repeat(1, d).contiguous()
    m = torch.zeros_like(x)
    w = torch.ones(n, k, device=dev)
    cs.cs_bind(m, d, d, 0, 1, torch.cuda.current_stream())
    for t in ("0", "1"):
        cs.cs_hier_step(x, g, w, gold["lr"], gold["momentum"])
        cs.cs_sync()
        assert np.all(x.cpu().numpy() == np.array(gold["expected_x"][t], np.float32)[:, None])
        assert m.cpu().numpy()[[0, 2], 0].tolist() == gold["expected_leader_m"][t]


def test_nonfinite_gradient_reports_diverged():
    n, d, k = 4, 1024, 2
    x, m, w, bank2 = _bind(n, d, k, 1)
    g = grads_view(bank2, n, 0).clone()
    g[2, 77] = float("nan")
    cs.cs_gossip_step(x, g, w, LR, MU)
    with pytest.raises(cs.CSError) as e:
        cs.cs_sync()
    assert e.value.code == -10
    cs.cs_sync()  # flag cleared after being reported


def test_host_entry_point_matches_device_entry_point():
    n, d, k = 8, 50_000, 4
    x, m, w, bank2 = _bind(n, d, k, 2)
    x2, m2, w2 = x.clone(), m.clone(), w.clone()
    gh = grads_view(bank2, n, 0).cpu().pin_memory()
    cd, ms = cs.cs_gossip_step_host(x, gh, w, LR, MU)
    cs.cs_set_step(0)
    cs.cs_bind(m2, d, d, 0, 1, torch.cuda.current_stream())
    cs.cs_set_diag(True)
    cs.cs_gossip_step(x2, grads_view(bank2, n, 0), w2, LR, MU)
    cd2, ms2 = cs.cs_get_diag()
    cs.cs_set_diag(False)
    assert torch.equal(x, x2) and torch.equal(m, m2) and torch.equal(w, w2)
    assert cd == cd2 and ms == ms2


def test_resume_via_set_step():
    n, d, k = 5, 3000, 3
    x, m, w, bank2 = _bind(n, d, k, 9)
    for t in range(6):
        cs.cs_gossip_step(x, grads_view(bank2, n, t), w, LR, MU)
    cs.cs_sync()
    ref = x.clone()
    x2, m2, w2, _ = device_state(cs, n, d, k, 9)
    cs.cs_bind(m2, d, d, 0, 1, torch.cuda.current_stream())
    cs.cs_set_step(0)
    for t in range(3):
        cs.cs_gossip_step(x2, grads_view(bank2, n, t), w2, LR, MU)
    snap = (x2.clone(), m2.clone(), w2.clone())
    cs.cs_bind(snap[1], d, d, 0, 1, torch.cuda.current_stream())   # "restore" into fresh buffers
    cs.cs_set_step(3)
    for t in range(3, 6):
        cs.cs_gossip_step(snap[0], grads_view(bank2, n, t), snap[2], LR, MU)
    cs.cs_sync()
    assert torch.equal(snap[0], ref)


# ---- every kernel path is bit-identical to the oracle ---------------------------------

PATHS = {"reg": 1, "tma": 2, "peer": 3, "peer_pm": 3}
SCHED = {"instep": 0, "deferred": 1, "split": 2}


@pytest.mark.parametrize("sched", ["instep", "deferred", "split"])
@pytest.mark.parametrize("path", ["reg", "tma", "peer", "peer_pm"])
@pytest.mark.parametrize("n,d,k,ld", [(2, 7, 1, 8), (3, 4099, 3, 4100), (8, 100_003, 4, 100_004),
                                      (16, 65_536, 8, 65_536), (5, 12_345, 5, 12_348)])
def test_each_path_bitwise(path, n, d, k, ld, sched, monkeypatch):
    # peer: the multi-GPU exchange kernels with every receiver local (one rank); instep:
    # k_push_merge's walk + in-kernel merge; deferred: the hybrid walk (several workers) or the
    # push/mix pair (peer_pm) with each step's merge inside the next step's kernel, the last one
    # in the final cs_sync's flush; split: walk + tail / push + mix
    if path in ("reg", "tma") and sched != "instep":
        pytest.skip("the schedules apply to the peer paths only")
    if path == "peer_pm":
        monkeypatch.setenv("CS_PEER_HYBRID", "0")
    cs.cs_init(n, n, k, 17)
    cs.cs_set_schedule(SCHED[sched])
    cs.cs_set_path(PATHS[path])
    x, m, w, bank2 = device_state(cs, n, d, k, 17, ld=ld)
    cs.cs_bind(m, d, ld, 0, 1, torch.cuda.current_stream())
    x[:, d:] = 3.0
    orc = OracleRun(n, d, k, 17)
    for t in range(4):
        cs.cs_gossip_step(x, grads_view(bank2, n, t), w, LR, MU)
        orc.step(LR, MU)
    cs.cs_sync()
    name, _ = cs.cs_kernel_info()
    want = {"reg": "k_gossip_local", "tma": "k_gossip_tma"}.get(path)
    if want is None:
        want = {"instep": "k_push_merge",
                "deferred": "k_peer_push(fused merge)" if path == "peer_pm" else "k_hyb_walk(fused tail merge)",
                "split": "k_peer_push+k_peer_mix" if path == "peer_pm" else "k_hyb_walk+k_hyb_tail"}[sched]
    assert name == want, (name, want)
    xg = x.cpu().numpy()
    assert np.array_equal(xg[:, :d], orc.x)
    assert np.array_equal(m.cpu().numpy()[:, :d], orc.m)
    assert np.array_equal(w.cpu().numpy(), orc.w)
    assert np.all(xg[:, d:] == 3.0)
    cs.cs_set_schedule(0)
    cs.cs_set_path(0)


@pytest.mark.parametrize("path", ["peer", "peer_pm"])
def test_peer_paths_world_128_bitwise(path, monkeypatch):
    # world 128 = the driver's 8-GPU weak-scaling run (16 workers per GPU): topology from
    # the device fallback generator (n > 64), every receiver local in single-GPU emulation
    if path == "peer_pm":
        monkeypatch.setenv("CS_PEER_HYBRID", "0")
    n, d, k, ld = 128, 8_195, 8, 8_196
    x, m, w, bank2 = _bind(n, d, k, 23, ld=ld, path=PATHS[path])
    orc = OracleRun(n, d, k, 23)
    for t in range(3):
        cs.cs_gossip_step(x, grads_view(bank2, n, t), w, LR, MU)
        orc.step(LR, MU)
    cs.cs_sync()
    assert np.array_equal(x.cpu().numpy()[:, :d], orc.x)
    assert np.array_equal(m.cpu().numpy()[:, :d], orc.m)
    assert np.array_equal(w.cpu().numpy(), orc.w)


@pytest.mark.parametrize("pieces", [2, 3, 8])
def test_peer_path_pieces_bitwise(pieces, monkeypatch):
    # the step cut into pieces: push(p+1) on the caller's stream overlaps mix(p) on the aux stream
    monkeypatch.setenv("CS_PEER_PIECES", str(pieces))
    monkeypatch.setenv("CS_PEER_HYBRID", "0")  # pieces apply to the push/mix pair (split schedule)
    n, d, k = 3, 70_003, 5
    x, m, w, bank2 = _bind(n, d, k, 23, path=PATHS["peer"], sched=2)
    orc = OracleRun(n, d, k, 23)
    for t in range(5):
        cs.cs_gossip_step(x, grads_view(bank2, n, t), w, LR, MU)
        orc.step(LR, MU)
    cs.cs_sync()
    assert np.array_equal(x.cpu().numpy()[:, :d], orc.x)
    assert np.array_equal(m.cpu().numpy()[:, :d], orc.m)
    assert np.array_equal(w.cpu().numpy(), orc.w)


def test_peer_path_single_gpu_resnet50_pair_sampled(monkeypatch):
    # the multi-GPU exchange protocol (inbox push, flags, epochs) with both workers of
    # BASELINE configs[2] co-resident: 2 x 25,557,032, k = 8, 10 steps
    monkeypatch.setenv("CS_PEER_HYBRID", "0")
    n, d, k = 2, 25_557_032, 8
    x, m, w, bank2 = _bind(n, d, k, 0, path=PATHS["peer"])
    cols = synth.sample_columns(d, T.segment_bounds(d, k))
    orc = OracleRun(n, d, k, 0, cols=cols)
    idx = torch.from_numpy(cols).cuda()
    for t in range(10):
        cs.cs_gossip_step(x, grads_view(bank2, n, t), w, LR, MU)
        orc.step(LR, MU)
    cs.cs_sync()
    assert np.array_equal(x.index_select(1, idx).cpu().numpy(), orc.x)
    assert np.array_equal(m.index_select(1, idx).cpu().numpy(), orc.m)
    assert np.array_equal(w.cpu().numpy(), orc.w)


@pytest.mark.parametrize("hybrid", ["1", "0"])
def test_peer_path_diagnostics_match_oracle(hybrid, monkeypatch):
    # the multi-GPU diagnostics pass (column chunks per GPU, rank-ordered partials)
    monkeypatch.setenv("CS_PEER_HYBRID", hybrid)
    n, d, k = 4, 50_003, 3
    x, m, w, bank2 = _bind(n, d, k, 1, path=PATHS["peer"])
    orc = OracleRun(n, d, k, 1)
    cs.cs_set_diag(True)
    for t in range(3):
        cs.cs_gossip_step(x, grads_view(bank2, n, t), w, LR, MU)
        orc.step(LR, MU)
        cd, ms = cs.cs_get_diag()
        cd0, ms0 = consensus(orc.x, orc.w, orc.seg)
        assert abs(cd - cd0) <= 1e-9 * abs(cd0), (t, cd, cd0)
        assert abs(ms - ms0) <= 1e-9 * max(1.0, abs(ms0)) + 1e-9 * d, (t, ms, ms0)
    cs.cs_set_diag(False)


@pytest.mark.parametrize("n,d,k,ld", [(8, 100_003, 4, 100_004), (16, 65_536, 8, 65_536), (3, 4_099, 3, 4_100)])
def test_gossip_step_io_round_trip_bitwise(n, d, k, ld):
    # the end-to-end entry: gradients from pinned host memory, the merged params and psw
    # copied back to host buffers, pieces of the vector pipelined across copy engines and the
    # step kernel; every returned buffer equals the oracle bit for bit
    x, m, w, bank2 = _bind(n, d, k, 21, ld=ld)
    x[:, d:] = 3.0
    orc = OracleRun(n, d, k, 21)
    host_bank = bank2.cpu().pin_memory()
    xo = torch.empty(n, ld, pin_memory=True)
    wo = torch.empty(n, k, pin_memory=True)
    for t in range(4):
        cs.cs_gossip_step_io(x, grads_view(host_bank, n, t), w, LR, MU, xo, wo)
        orc.step(LR, MU)
        assert np.array_equal(xo.numpy()[:, :d], orc.x), t
        assert np.array_equal(wo.numpy(), orc.w), t
    assert np.array_equal(x.cpu().numpy()[:, :d], orc.x)
    assert np.array_equal(m.cpu().numpy()[:, :d], orc.m)
    assert np.all(x.cpu().numpy()[:, d:] == 3.0)
    cs.cs_finalize()
