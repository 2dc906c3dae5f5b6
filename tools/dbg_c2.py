# emulated c2 shape at V=2 (n_loc=16, d=11.7M, k=8): does the step finish?
import sys, os, time
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests"))
import torch
import __graft_entry__ as entry
entry.build()
import paper_2012_15198_b200 as cs
import synth
from gpu_util import device_state, grads_view
LR, MU = float(synth.DEFAULT_LR), float(synth.DEFAULT_MOMENTUM)
V, n_loc, d, k = 2, int(sys.argv[1]) if len(sys.argv) > 1 else 16, int(sys.argv[2]) if len(sys.argv) > 2 else 11_689_512, 8
n = V * n_loc
cs.cs_init(n, n, k, 0)
cs.cs_test_emulate_ranks(V)
x, m, w, bank2 = device_state(cs, n, d, k, 0)
cs.cs_bind(m, d, d, 0, 1, torch.cuda.current_stream())
for t in range(4):
    t0 = time.time()
    cs.cs_gossip_step(x, grads_view(bank2, n, t), w, LR, MU)
    try:
        cs.cs_sync()
        print("step", t, "ok", round(time.time() - t0, 3), "s", flush=True)
    except cs.CSError as e:
        print("step", t, "error", e, round(time.time() - t0, 3), "s", flush=True)
cs.cs_finalize()
