"""-m gpu: bf16 wire format (reading C-20) on every single-GPU kernel
path, bitwise against the oracle's gossip_step(..., wire="bf16")."""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import __graft_entry__ as entry  # noqa: E402

entry.build()
import paper_2012_15198_b200 as cs  # noqa: E402
from gpu_util import OracleRun, device_state, grads_view  # noqa: E402

LR, MU = float(synth.DEFAULT_LR), float(synth.DEFAULT_MOMENTUM)


@pytest.mark.parametrize("n,d,k,path,hybrid", [(8, 100_003, 4, 0, 1), (16, 65_536, 8, 1, 1), (128, 4_099, 2, 0, 1),
                                               (6, 50_001, 5, 3, 1), (6, 50_001, 5, 3, 0), (2, 33, 1, 0, 1)])
def test_bf16_wire_bitwise(n, d, k, path, hybrid, monkeypatch):
    monkeypatch.setenv("CS_PEER_HYBRID", str(hybrid))
    seed = 13
    ld = (d + 3) // 4 * 4
    cs.cs_init(n, n, k, seed)
    cs.cs_set_path(path)
    cs.cs_set_wire(cs.WIRE_BF16)
    x, m, w, bank2 = device_state(cs, n, d, k, seed, ld=ld)
    cs.cs_bind(m, d, ld, 0, 1, torch.cuda.current_stream())
    orc = OracleRun(n, d, k, seed)
    for t in range(6):
        cs.cs_gossip_step(x, grads_view(bank2, n, t), w, LR, MU)
        orc.step(LR, MU, wire="bf16")
    cs.cs_sync()
    assert np.array_equal(x.cpu().numpy()[:, :d], orc.x)
    assert np.array_equal(m.cpu().numpy()[:, :d], orc.m)
    assert np.array_equal(w.cpu().numpy(), orc.w)
    cs.cs_set_path(0)


def test_bf16_wire_differs_from_fp32_and_hier_refuses():
    n, d, k = 4, 4096, 2
    outs = []
    for fmt in (cs.WIRE_FP32, cs.WIRE_BF16):
        cs.cs_init(n, n, k, 1)
        cs.cs_set_wire(fmt)
        x, m, w, bank2 = device_state(cs, n, d, k, 1)
        cs.cs_bind(m, d, d, 0, 1, torch.cuda.current_stream())
        cs.cs_gossip_step(x, grads_view(bank2, n, 0), w, LR, MU)
        cs.cs_sync()
        outs.append(x.cpu().numpy())
    assert not np.array_equal(outs[0], outs[1])
    assert np.max(np.abs(outs[0] - outs[1])) <= 2.0**-9 * np.abs(outs[0]).max() * 2
    cs.cs_init(n, 2, k, 1)
    cs.cs_set_wire(cs.WIRE_BF16)
    x, m, w, bank2 = device_state(cs, n, d, k, 1)
    cs.cs_bind(m, d, d, 0, 1, torch.cuda.current_stream())
    with pytest.raises(cs.CSError) as e:
        cs.cs_hier_step(x, grads_view(bank2, n, 0), w, LR, MU)
    assert e.value.code == -12
    with pytest.raises(cs.CSError):
        cs.cs_set_wire(5)
