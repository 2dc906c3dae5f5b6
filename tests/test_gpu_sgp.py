"""-m gpu: SGP's directed exponential graph on the same machinery (
PAPER.md:103, :300) through the C-ABI, bitwise against oracle/sgp.py + the oracle
step, on every single-GPU kernel path."""
import numpy as np
import pytest
import torch

import synth
from oracle.sgp import exponential_topology

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import __graft_entry__ as entry  # noqa: E402

entry.build()
import paper_2012_15198_b200 as cs  # noqa: E402
from gpu_util import OracleRun, device_state, grads_view  # noqa: E402

LR, MU = float(synth.DEFAULT_LR), float(synth.DEFAULT_MOMENTUM)


@pytest.mark.parametrize("n,d,k,path,hybrid", [(8, 100_003, 1, 0, 1), (16, 65_536, 1, 2, 1),
                                               (16, 65_536, 1, 1, 1), (64, 20_000, 2, 0, 1),
                                               (128, 4_096, 1, 0, 1), (4, 50_000, 4, 3, 1), (8, 50_000, 1, 3, 0)])
def test_exponential_topology_bitwise(n, d, k, path, hybrid, monkeypatch):
    # path 0 auto (TMA for n <= 64, k_topology + register walk for n = 128), 1 reg, 2 tma,
    # 3 peer (single-GPU emulation of the NVLink path: hybrid walk, or push/mix with hybrid 0)
    monkeypatch.setenv("CS_PEER_HYBRID", str(hybrid))
    seed = 9
    ld = (d + 3) // 4 * 4
    cs.cs_init(n, n, k, seed)
    cs.cs_set_path(path)
    cs.cs_set_topology_kind(cs.TOPO_EXPONENTIAL)
    x, m, w, bank2 = device_state(cs, n, d, k, seed, ld=ld)
    cs.cs_bind(m, d, ld, 0, 1, torch.cuda.current_stream())
    orc = OracleRun(n, d, k, seed)
    for t in range(2 * (n.bit_length() - 1) + 1):
        cs.cs_gossip_step(x, grads_view(bank2, n, t), w, LR, MU)
        orc.step(LR, MU, src=exponential_topology(t, n, k))
    cs.cs_sync()
    assert np.array_equal(x.cpu().numpy()[:, :d], orc.x)
    assert np.array_equal(m.cpu().numpy()[:, :d], orc.m)
    assert np.array_equal(w.cpu().numpy(), orc.w)
    cs.cs_set_path(0)


def test_exponential_reaches_consensus_in_log2_n_steps():
    # lr = 0: x_i <- mean of all rows after log2 n rounds (dyadic inputs: exact)
    n, d = 16, 4096
    cs.cs_init(n, n, 1, 0)
    cs.cs_set_topology_kind(cs.TOPO_EXPONENTIAL)
    x = (torch.randint(-512, 512, (n, d), dtype=torch.int32).float() * 2.0 ** -6).cuda()
    mean = x.double().mean(0).float()
    m = torch.zeros(n, d, device="cuda")
    w = torch.ones(n, 1, device="cuda")
    cs.cs_bind(m, d, d, 0, 1, torch.cuda.current_stream())
    z = torch.zeros(n, d, device="cuda")
    for _ in range(4):
        cs.cs_gossip_step(x, z, w, 0.0, 0.0)
    cs.cs_sync()
    assert torch.equal(x, mean.expand(n, d))
