"""-m gpu: BASELINE.json configs[1] at full size (16 workers x ResNet-18-sized
11,689,512 fp32, k=8, 100 steps) in the launch configuration bench.py times,
checked on sampled columns (every segment boundary +-2, a 1/1024 stride, the
tail and 256 random columns) that the oracle computes column by column — the
update is column-separable given the topology."""
import numpy as np
import pytest
import torch

import synth
from oracle import topology as T
from oracle.diagnostics import consensus

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import __graft_entry__ as entry  # noqa: E402

entry.build()
import paper_2012_15198_b200 as cs  # noqa: E402
from gpu_util import OracleRun, device_state, grads_view, rel_norm_err  # noqa: E402

LR, MU = float(synth.DEFAULT_LR), float(synth.DEFAULT_MOMENTUM)


@pytest.mark.parametrize("n,d,k,steps,check_at", [(16, 11_689_512, 8, 100, (1, 10, 100))])
def test_config2_sampled_bitwise(n, d, k, steps, check_at):
    seed = 0
    cs.cs_init(n, n, k, seed)
    x, m, w, bank2 = device_state(cs, n, d, k, seed)
    cs.cs_bind(m, d, d, 0, 1, torch.cuda.current_stream())
    cols = synth.sample_columns(d, T.segment_bounds(d, k))
    orc = OracleRun(n, d, k, seed, cols=cols)
    idx = torch.from_numpy(cols).cuda()
    for t in range(steps):
        cs.cs_gossip_step(x, grads_view(bank2, n, t), w, LR, MU)
        orc.step(LR, MU)
        if t + 1 in check_at:
            xg = x.index_select(1, idx).cpu().numpy()
            mg = m.index_select(1, idx).cpu().numpy()
            assert np.array_equal(xg, orc.x), t
            assert np.array_equal(mg, orc.m), t
            assert np.array_equal(w.cpu().numpy(), orc.w), t
    assert rel_norm_err(xg, orc.x).max() <= 1e-6
    xa = np.abs(orc.x).max()
    assert np.abs(xg - orc.x).max() <= 1e-6 * xa


def test_config2_invariants_at_full_size():
    # properties that hold at any size, on every column: psw stays exactly 1 (P14);
    # with lr = 0 the per-column mean is invariant within 2^-23 max|y| (P10) and the
    # consensus distance does not increase (P11)
    n, d, k, seed = 16, 11_689_512, 8, 0
    cs.cs_init(n, n, k, seed)
    x, m, w, _ = device_state(cs, n, d, k, seed)
    cs.cs_bind(m, d, d, 0, 1, torch.cuda.current_stream())
    zero = torch.zeros(n, d, device=x.device)
    cs.cs_set_diag(True)
    prev_cd = None
    for t in range(5):
        mean0 = x.double().mean(0)
        cs.cs_gossip_step(x, zero, w, 0.0, MU)
        cd, _ = cs.cs_get_diag()
        drift = (x.double().mean(0) - mean0).abs()
        bound = 2.0**-23 * x.abs().max(0).values.double() + 1e-45
        assert bool((drift <= bound).all())
        assert bool((w == 1.0).all())
        if prev_cd is not None:
            assert cd <= prev_cd * (1 + 1e-12)
        prev_cd = cd
    cs.cs_set_diag(False)
