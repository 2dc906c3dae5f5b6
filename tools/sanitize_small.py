"""Small runs of every single-GPU kernel path, for `compute-sanitizer --tool memcheck`
(out-of-bounds / misaligned accesses, including the ragged tails and padding columns).
Results are not checked here (the parity tests do that); the sanitizer's report is."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__ as entry  # noqa: E402

entry.build()
import paper_2012_15198_b200 as cs  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
LR, MU = float(synth.DEFAULT_LR), float(synth.DEFAULT_MOMENTUM)


def state(n, d, k, ld, seed=1):
    x = torch.zeros(n, ld, device=dev)
    cs.cs_synth_fill(x, n, d, ld, seed, synth.TAG_INIT, 0, 1.0)
    m = torch.zeros(n, ld, device=dev)
    w = torch.ones(n, k, device=dev)
    g = torch.zeros(n, ld, device=dev)
    cs.cs_synth_fill(g, n, d, ld, seed, synth.TAG_GRAD, 0, 0.0625)
    return x, m, w, g


def run(n, d, k, ld, path=0, groups=None, diag=False, wire=0, topo=0, env=None, steps=3):
    for key, val in (env or {}).items():
        os.environ[key] = val
    cs.cs_init(n, groups or n, k, 3)
    cs.cs_set_path(path)
    cs.cs_set_wire(wire)
    if topo:
        cs.cs_set_topology_kind(topo)
    x, m, w, g = state(n, d, k, ld)
    cs.cs_bind(m, d, ld, 0, 1, torch.cuda.current_stream())
    cs.cs_set_diag(diag)
    step = cs.cs_hier_step if groups else cs.cs_gossip_step
    for _ in range(steps):
        step(x, g, w, LR, MU)
    cs.cs_sync()
    if diag:
        cs.cs_get_diag()
    for key in (env or {}):
        del os.environ[key]
    print(f"ok n={n} d={d} k={k} ld={ld} path={path} groups={groups} diag={diag} wire={wire} env={env}", flush=True)


# flat paths: TMA (0 auto), register (1), peer hybrid / push-mix emulation (3), fused or not
for (n, d, k, ld) in [(2, 7, 1, 8), (5, 4099, 3, 4100), (8, 20_001, 4, 20_004), (130, 3_000, 2, 3_000)]:
    for path in (0, 1):
        run(n, d, k, ld, path=path, diag=True)
    for fuse in ("1", "0"):
        run(n, d, k, ld, path=3, env={"CS_PEER_FUSE": fuse}) if n <= 64 else None
        run(n, d, k, ld, path=3, env={"CS_PEER_FUSE": fuse, "CS_PEER_HYBRID": "0"}) if n <= 64 else None
    run(n, d, k, ld, path=0, wire=1)
    if n <= 64:
        run(n, d, k, ld, path=3, wire=1)
# hierarchical on one GPU, SGP topology
run(8, 10_001, 3, 10_004, groups=2, diag=True)
run(8, 10_001, 1, 10_004, topo=1)
# communication interval and LARS with a layer plan
cs.cs_init(4, 4, 3, 0)
x, m, w, g = state(4, 9_998, 3, 10_000)
cs.cs_bind(m, 9_998, 10_000, 0, 1, torch.cuda.current_stream())
acc = torch.empty_like(g)
for c in range(3):
    cs.cs_accumulate(acc, g, c, 3)
sizes = [1000, 2996, 4000, 2002]
lb = np.concatenate([[0], np.cumsum(sizes)])
cs.cs_set_layers(lb, cs.cs_segment_plan(sizes, 3))
cs.cs_set_lars(0.0025, 5e-5, 1e-9)
for _ in range(3):
    cs.cs_gossip_step(x, acc, w, 9.0, MU)
cs.cs_sync()
cs.cs_get_lars_rates(4, len(sizes))
print("ok interval + LARS", flush=True)
cs.cs_finalize()
print("SANITIZE-RUN-DONE", flush=True)
