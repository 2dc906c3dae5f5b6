"""-m gpu, >= 2 GPUs: the NVLink peer-memory path (one process per GPU) against
the oracle, bit-exact on sampled (or all) columns.  Skipped on 1-GPU boxes; the
world_size-2 host logic is covered on CPU by tests/test_multiproc_cpu.py."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0


def _free_port():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(nproc, *args, timeout=600, env=None):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.join(ROOT, "tests", "mp_gossip_worker.py"),
           *[str(a) for a in args]]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT,
                       env={**os.environ, **(env or {})})
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    assert "OK" in p.stdout


@pytest.mark.skipif(NGPU < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("n_loc,d,k,steps,full", [(1, 4099, 3, 6, True), (3, 50_001, 5, 5, True),
                                                  (8, 200_000, 32, 4, True), (1, 1_000_003, 8, 8, True),
                                                  (40, 30_001, 8, 4, True)])  # world 80 > 64: k_topology tables
def test_two_gpu_parity(n_loc, d, k, steps, full):
    args = ["--workers-per-gpu", n_loc, "--vector-len", d, "--segments", k, "--num-steps", steps]
    if full:
        args.append("--compare-all")
    _run(2, *args)


@pytest.mark.skipif(NGPU < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("n_loc,d,k,extra", [(1, 100_003, 5, []), (1, 25_557_032, 8, []), (1, 50_001, 1, ["--exponential"]),
                                             (1, 70_001, 4, ["--wire-bf16"]), (1, 200_000, 6, ["--hier-groups", "2"])])
def test_two_gpu_in_step_merge_without_flush(n_loc, d, k, extra):
    # the default schedule: after each step's work -- a plain stream synchronize, no cs_flush
    # or cs_sync -- params and psw equal the oracle's merged x', w' bit for bit
    args = ["--workers-per-gpu", n_loc, "--vector-len", d, "--segments", k, "--num-steps", 8, "--stream-sync"]
    if d < 1_000_000:
        args.append("--compare-all")
    _run(2, *args, *extra)


@pytest.mark.skipif(NGPU < 4, reason="needs 4 GPUs")
@pytest.mark.parametrize("d,k,extra", [(25_557_032, 8, []), (300_001, 16, ["--hier-groups", "2"]),
                                       (100_003, 3, ["--wire-bf16"])])
def test_four_gpu_in_step_merge_without_flush(d, k, extra):
    args = ["--workers-per-gpu", 1, "--vector-len", d, "--segments", k, "--num-steps", 8, "--stream-sync"]
    if d < 1_000_000:
        args.append("--compare-all")
    _run(4, *args, *extra)


@pytest.mark.skipif(NGPU < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("schedule", ["deferred", "split"])
def test_two_gpu_opt_in_schedules_bitwise(schedule):
    _run(2, "--workers-per-gpu", 1, "--vector-len", 100_003, "--segments", 5, "--num-steps", 6, "--compare-all",
         "--schedule", schedule)


@pytest.mark.skipif(NGPU < 2, reason="needs 2 GPUs")
def test_two_gpu_resnet50_sampled():
    # BASELINE configs[2] layout (one worker per GPU, 25,557,032 fp32, k = 8)
    _run(2, "--workers-per-gpu", 1, "--vector-len", 25_557_032, "--segments", 8, "--num-steps", 10)


@pytest.mark.skipif(NGPU < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("n_loc,groups", [(3, 0), (1, 0), (1, 2)])
def test_two_gpu_diagnostics(n_loc, groups):
    # consensus distance / mean checksum across GPUs vs the oracle (<= 1e-9 relative)
    args = ["--workers-per-gpu", n_loc, "--vector-len", 100_003, "--segments", 5, "--num-steps", 3,
            "--compare-all", "--diag"]
    if groups:
        args += ["--hier-groups", groups]
    _run(2, *args)


@pytest.mark.skipif(NGPU < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("n_loc,k", [(1, 1), (4, 1), (2, 3)])
def test_two_gpu_exponential_bitwise(n_loc, k):
    # SGP's directed exponential graph across GPUs (push/mix for 1 worker/GPU, hybrid otherwise)
    _run(2, "--workers-per-gpu", n_loc, "--vector-len", 100_003, "--segments", k, "--num-steps", 5,
         "--compare-all", "--exponential")


@pytest.mark.skipif(NGPU < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("n_loc,d,k", [(1, 100_003, 3), (3, 50_001, 5), (1, 25_557_032, 8)])
def test_two_gpu_bf16_wire_bitwise(n_loc, d, k):
    # bf16 inbox rows over NVLink (push/mix for 1 worker/GPU, hybrid heads otherwise)
    args = ["--workers-per-gpu", n_loc, "--vector-len", d, "--segments", k, "--num-steps", 5, "--wire-bf16"]
    if d < 1_000_000:
        args.append("--compare-all")
    _run(2, *args)


@pytest.mark.skipif(NGPU < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("layers,plan,lars,diag", [(9, True, False, True), (25, True, True, False),
                                                   (12, False, True, True)])
def test_two_gpu_layers_and_lars(layers, plan, lars, diag):
    # layer table on the push/mix path: layer-plan segments bitwise; LARS within 1 ulp / 1e-6
    args = ["--workers-per-gpu", 1, "--vector-len", 200_000, "--segments", 6, "--num-steps", 5, "--compare-all",
            "--layers", layers]
    args += (["--layer-plan"] if plan else []) + (["--lars"] if lars else []) + (["--diag"] if diag else [])
    _run(2, *args)


@pytest.mark.skipif(NGPU < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("n_loc,plan,diag", [(3, True, True), (4, False, False)])
def test_two_gpu_hybrid_layers_and_lars(n_loc, plan, diag):
    # several workers per GPU (hybrid walk) with a layer table and LARS
    args = ["--workers-per-gpu", n_loc, "--vector-len", 180_000, "--segments", 5, "--num-steps", 5,
            "--compare-all", "--layers", 16, "--lars"]
    args += (["--layer-plan"] if plan else []) + (["--diag"] if diag else [])
    _run(2, *args)


@pytest.mark.skipif(NGPU < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("groups,plan", [(1, True), (2, False)])
def test_two_gpu_hierarchical_lars(groups, plan):
    # LARS on the group-reduced gradient: one group (AllReduce-SGD + LARS) and
    # two groups of one (leader gossip), with a layer table
    args = ["--workers-per-gpu", 1, "--vector-len", 120_000, "--segments", 4, "--num-steps", 4, "--compare-all",
            "--layers", 10, "--lars", "--hier-groups", groups] + (["--layer-plan"] if plan else [])
    _run(2, *args)


@pytest.mark.skipif(NGPU < 4, reason="needs 4 GPUs")
def test_four_gpu_hierarchical_lars():
    _run(4, "--workers-per-gpu", 1, "--vector-len", 200_000, "--segments", 6, "--num-steps", 4, "--compare-all",
         "--layers", 14, "--lars", "--hier-groups", 2, "--layer-plan")


@pytest.mark.skipif(NGPU < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("n_loc,d,k,extra", [(1, 100_003, 3, []), (1, 25_557_032, 8, []), (3, 60_001, 4, []),
                                             (1, 50_001, 2, ["--exponential"]), (1, 100_003, 5, ["--wire-bf16"])])
def test_two_gpu_deferred_merge_bitwise(n_loc, d, k, extra):
    # no cs_sync between steps: each step's merge runs inside the next step's push kernel
    # (push/mix schedule; n_loc > 1 with the hybrid walk off), flushed by the final cs_sync
    args = ["--workers-per-gpu", n_loc, "--vector-len", d, "--segments", k, "--num-steps", 7, "--sync-at-end"]
    if d < 1_000_000:
        args.append("--compare-all")
    _run(2, *args, *extra, "--schedule", "deferred", env={"CS_PEER_HYBRID": "0"})


@pytest.mark.skipif(NGPU < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("n_loc,d,k,extra", [(4, 100_003, 5, []), (8, 400_000, 16, []), (4, 50_001, 2, ["--exponential"]),
                                             (3, 70_001, 6, ["--wire-bf16"]),
                                             (40, 30_001, 8, [])])  # world 80: k_topology tables every step
def test_two_gpu_hybrid_deferred_tail_merge_bitwise(n_loc, d, k, extra):
    # several workers per GPU (hybrid walk): each step's chain tails merge inside the next walk
    _run(2, "--workers-per-gpu", n_loc, "--vector-len", d, "--segments", k, "--num-steps", 7, "--sync-at-end",
         "--compare-all", "--schedule", "deferred", *extra)


@pytest.mark.skipif(NGPU < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("n_loc,groups", [(1, 0), (3, 0), (1, 1)])
def test_two_gpu_nonfinite_gradient_reported(n_loc, groups):
    # push (1/GPU), hybrid walk (3/GPU) and the hierarchical step flag a NaN gradient
    args = ["--workers-per-gpu", n_loc, "--vector-len", 50_001, "--segments", 3, "--inject-nan"]
    if groups:
        args += ["--hier-groups", groups]
    _run(2, *args)


@pytest.mark.skipif(NGPU < 2, reason="needs 2 GPUs")
def test_two_gpu_missing_peer_times_out():
    # a peer that never pushes: the waiting GPU gives up after the ~20 s bound with CS_ETIMEOUT
    _run(2, "--workers-per-gpu", 1, "--vector-len", 50_001, "--segments", 3, "--skip-step")


@pytest.mark.skipif(NGPU < 2, reason="needs 2 GPUs")
def test_two_gpu_hier_deferred_exchange_merge_bitwise():
    # groups >= 2: the leader exchange's merge runs inside the next hierarchical push
    # (opt-in schedule, CS_HIER_FUSE=1)
    _run(2, "--workers-per-gpu", 1, "--vector-len", 150_001, "--segments", 5, "--num-steps", 6,
         "--hier-groups", 2, "--compare-all", "--sync-at-end", "--schedule", "deferred",
         env={"CS_HIER_FUSE": "1"})


@pytest.mark.skipif(NGPU < 4, reason="needs 4 GPUs")
def test_four_gpu_hier_deferred_exchange_merge_bitwise():
    _run(4, "--workers-per-gpu", 1, "--vector-len", 150_001, "--segments", 7, "--num-steps", 6,
         "--hier-groups", 2, "--compare-all", "--sync-at-end", "--schedule", "deferred",
         env={"CS_HIER_FUSE": "1"})


@pytest.mark.skipif(NGPU < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("pieces", [3, 8])
def test_two_gpu_pieces_bitwise(pieces):
    # push(p+1) / mix(p) overlap across the caller's and the aux stream, across GPUs
    _run(2, "--workers-per-gpu", 2, "--vector-len", 300_001, "--segments", 6, "--num-steps", 5,
         "--compare-all", env={"CS_PEER_PIECES": str(pieces)})
    _run(2, "--workers-per-gpu", 1, "--vector-len", 200_000, "--segments", 4, "--num-steps", 4,
         "--hier-groups", 2, "--compare-all", env={"CS_PEER_PIECES": str(pieces)})


@pytest.mark.skipif(NGPU < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("groups,d,k", [(1, 100_003, 3), (2, 50_000, 4)])
def test_two_gpu_hierarchical_bitwise(groups, d, k):
    # one worker per GPU; groups=1: gradient allreduce + SGD, groups=2: leader gossip (swap)
    _run(2, "--workers-per-gpu", 1, "--vector-len", d, "--segments", k, "--num-steps", 5,
         "--hier-groups", groups, "--compare-all")


@pytest.mark.skipif(NGPU < 4, reason="needs 4 GPUs")
@pytest.mark.parametrize("groups,d,k", [(2, 1_000_003, 16), (1, 65_536, 2), (4, 70_001, 5)])
def test_four_gpu_hierarchical_bitwise(groups, d, k):
    # BASELINE configs[3] layout at 4 GPUs: 2 groups x 2 GPUs, k = 16
    _run(4, "--workers-per-gpu", 1, "--vector-len", d, "--segments", k, "--num-steps", 4,
         "--hier-groups", groups, "--compare-all")


@pytest.mark.skipif(NGPU < 4, reason="needs 4 GPUs")
@pytest.mark.parametrize("n_loc,groups", [(2, 0), (1, 2)])
def test_four_gpu_diagnostics(n_loc, groups):
    args = ["--workers-per-gpu", n_loc, "--vector-len", 200_001, "--segments", 7, "--num-steps", 3,
            "--compare-all", "--diag"]
    if groups:
        args += ["--hier-groups", groups]
    _run(4, *args)


@pytest.mark.skipif(NGPU < 4, reason="needs 4 GPUs")
@pytest.mark.parametrize("n_loc,d,k", [(1, 25_557_032, 8), (8, 1_000_000, 16)])
def test_four_gpu_parity(n_loc, d, k):
    _run(4, "--workers-per-gpu", n_loc, "--vector-len", d, "--segments", k, "--num-steps", 6)


# ---- NVLS h1: the intra-group gradient average in the NVSwitch (cs_set_multicast) ----------
@pytest.mark.skipif(NGPU < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("groups,d,k,mc_bank", [(1, 100_003, 3, False), (1, 100_003, 3, True),
                                                (1, 4099, 1, False)])
def test_two_gpu_hierarchical_nvls(groups, d, k, mc_bank):
    # groups of 2 GPUs sum two values: order-free, so bitwise vs the oracle
    _run(2, "--workers-per-gpu", 1, "--vector-len", d, "--segments", k, "--num-steps", 5,
         "--hier-groups", groups, "--compare-all", "--nvls", *(["--mc-bank"] if mc_bank else []))


@pytest.mark.skipif(NGPU < 4, reason="needs 4 GPUs")
@pytest.mark.parametrize("groups,d,k,steps,mc_bank,full", [(1, 300_001, 5, 5, True, True),
                                                          (1, 1_000_003, 8, 100, False, False),
                                                          (2, 1_000_003, 16, 6, True, True),
                                                          (1, 25_557_032, 16, 3, True, False)])
def test_four_gpu_hierarchical_nvls(groups, d, k, steps, mc_bank, full):
    # groups of 4: the switch's summation order -> norm-wise <= 1e-6 vs the oracle (the
    # hierarchical tolerance; 100 steps: the north_star criterion); groups of 2
    # (configs[3] layout at 4 GPUs) bitwise; members bit-identical to their leader always
    _run(4, "--workers-per-gpu", 1, "--vector-len", d, "--segments", k, "--num-steps", steps,
         "--hier-groups", groups, "--nvls", *(["--mc-bank"] if mc_bank else []),
         *(["--compare-all"] if full else []))


# ---- NCCL h1: the intra-group gradient sum by ncclAllReduce (cs_set_hier_nccl) -------------
@pytest.mark.skipif(NGPU < 2, reason="needs 2 GPUs")
def test_two_gpu_hierarchical_nccl():
    # a group of 2 GPUs: NCCL's sum of two values is order-free, so bitwise vs the oracle
    _run(2, "--workers-per-gpu", 1, "--vector-len", 100_003, "--segments", 3, "--num-steps", 5,
         "--hier-groups", 1, "--compare-all", "--nccl")


@pytest.mark.skipif(NGPU < 4, reason="needs 4 GPUs")
@pytest.mark.parametrize("groups,d,k,steps,full", [(1, 1_000_003, 8, 100, False), (2, 300_001, 16, 6, True)])
def test_four_gpu_hierarchical_nccl(groups, d, k, steps, full):
    # groups of 4: NCCL's order -> norm-wise <= 1e-6 after 100 steps; 2 x 2: bitwise
    _run(4, "--workers-per-gpu", 1, "--vector-len", d, "--segments", k, "--num-steps", steps,
         "--hier-groups", groups, "--nccl", *(["--compare-all"] if full else []))
