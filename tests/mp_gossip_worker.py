"""torchrun worker for the multi-GPU parity test (tests/test_gpu_multi.py).

Each rank holds n_loc workers (global ids rank*n_loc ..), steps through the
C-ABI with segments exchanged over NVLink peer memory, and compares its rows on
sampled columns with the oracle run for all workers on the same columns.
Exit code 0 = parity; 1 = mismatch."""
import argparse
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import synth  # noqa: E402
from oracle import topology as T  # noqa: E402

import __graft_entry__ as entry  # noqa: E402

entry.build()
import paper_2012_15198_b200 as cs  # noqa: E402
from gpu_util import OracleRun  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workers-per-gpu", type=int, required=True)
    ap.add_argument("--vector-len", type=int, required=True)
    ap.add_argument("--segments", type=int, required=True)
    ap.add_argument("--num-steps", type=int, default=5)
    ap.add_argument("--rng-seed", type=int, default=0)
    ap.add_argument("--compare-all", action="store_true", help="compare every column (small d)")
    ap.add_argument("--hier-groups", type=int, default=0, help="hierarchical step with this many groups")
    ap.add_argument("--diag", action="store_true", help="check the multi-GPU diagnostics too")
    ap.add_argument("--exponential", action="store_true", help="SGP's exponential graph (cs_set_topology_kind)")
    ap.add_argument("--wire-bf16", action="store_true", help="bf16 wire format (cs_set_wire)")
    ap.add_argument("--layers", type=int, default=0, help="random layer table with this many layers")
    ap.add_argument("--layer-plan", action="store_true", help="segments from the layer plan (cs_segment_plan)")
    ap.add_argument("--lars", action="store_true", help="LARS (Table 1 constants, lr 9)")
    ap.add_argument("--inject-nan", action="store_true",
                    help="rank 0 puts a NaN in its gradient at step 1: every process must see CS_EDIVERGED")
    ap.add_argument("--skip-step", action="store_true",
                    help="rank 1 skips step 1: rank 0's merge of that step must time out (CS_ETIMEOUT), not hang")
    ap.add_argument("--sync-at-end", action="store_true",
                    help="no cs_sync between steps (deferred merges run inside the next push); compare at the end")
    ap.add_argument("--schedule", default="instep", choices=["instep", "deferred", "split"],
                    help="cs_set_schedule: instep (default) merges inside each step")
    ap.add_argument("--nvls", action="store_true",
                    help="hierarchical h1 through the NVSwitch (cs_set_multicast): tolerance parity for groups "
                         ">= 3 GPUs (switch summation order), bitwise for groups of 2; members bitwise equal")
    ap.add_argument("--nccl", action="store_true",
                    help="hierarchical h1 through NCCL (cs_set_hier_nccl): tolerance parity for groups >= 3 GPUs "
                         "(NCCL's summation order), bitwise for groups of 2; members bitwise equal")
    ap.add_argument("--mc-bank", action="store_true",
                    help="with --nvls: the gradient bank lives in multicast memory (reduced in place)")
    ap.add_argument("--stream-sync", action="store_true",
                    help="read params after a plain stream synchronize (no cs_sync / cs_flush): the step's "
                         "enqueued work alone must leave merged params (in-step schedule)")
    a = ap.parse_args()
    rank, ws, lr_ = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(lr_)
    dev = torch.device("cuda", lr_)
    dist.init_process_group("nccl", device_id=dev)
    n_loc, d, k, seed = a.workers_per_gpu, a.vector_len, a.segments, a.rng_seed
    world = n_loc * ws
    first = rank * n_loc
    lr, mu = float(synth.DEFAULT_LR), float(synth.DEFAULT_MOMENTUM)
    groups = a.hier_groups or world
    cs.cs_init(world, groups, k, seed)
    cs.cs_set_schedule({"instep": cs.CS_SCHED_INSTEP, "deferred": cs.CS_SCHED_DEFERRED,
                        "split": cs.CS_SCHED_SPLIT}[a.schedule])
    if a.wire_bf16:
        cs.cs_set_wire(cs.WIRE_BF16)
    if a.exponential:
        cs.cs_set_topology_kind(cs.TOPO_EXPONENTIAL)
        from oracle.sgp import exponential_topology
    stream = torch.cuda.current_stream(dev)
    ld = (d + 3) // 4 * 4
    x = torch.zeros(n_loc, ld, device=dev)
    m = torch.zeros(n_loc, ld, device=dev)
    w = torch.ones(n_loc, k, device=dev)
    B = world + 1
    gs_h = world // groups
    bank = torch.zeros(B + n_loc, ld, device=dev)
    cs.cs_bind(m, d, ld, rank, ws, stream)
    gcur = None
    if a.nvls and a.mc_bank:
        # the caller's gradient buffer in symmetric memory over the group, at the same offset
        # on every member (as a training loop's flat gradient buffer): reduced in place
        gcur, gcur_mc = cs.multicast_empty((n_loc, ld), gs_h, dev)
    cs.cs_synth_fill(x, n_loc, d, ld, seed, synth.TAG_INIT, first, 1.0)
    cs.cs_synth_fill(bank, B, d, ld, seed, synth.TAG_GRAD, 0, float(synth.GRAD_SCALE))
    torch.cuda.synchronize()
    bank[B:] = bank[:n_loc]
    torch.cuda.synchronize()
    cs.setup_peers()
    if a.nccl:
        cs.setup_hier_nccl(gs_h)
    if a.nvls:
        if not cs.setup_multicast(gs_h, dev):
            print("no multicast on this fabric: FAIL", flush=True)
            sys.exit(1)
        if a.mc_bank:
            cs.register_multicast_grads(gcur, gcur_mc)

    cols = np.arange(d) if a.compare_all else synth.sample_columns(d, T.segment_bounds(d, k))
    orc = OracleRun(world, d, k, seed, cols=cols, groups=a.hier_groups or None)
    lb = None
    if a.layers:
        from oracle.lars import lars_gossip_step, plan_bounds, segment_plan
        rng = np.random.default_rng(a.layers)
        cuts = np.unique(rng.integers(1, d // 4, size=a.layers - 1) * 4)
        lb = np.concatenate([[0], cuts, [d]]).astype(np.int64)
        sizes = np.diff(lb).tolist()
        plan = segment_plan(sizes, k) if a.layer_plan else None
        cs.cs_set_layers(lb, plan)
        orc.seg = T.segment_of_columns(plan_bounds(lb, plan) if plan else T.segment_bounds(d, k), cols)
    if a.lars:
        ETA, WD, EPS = 0.0025, 5e-5, 1e-9
        cs.cs_set_lars(ETA, WD, EPS)
        lr = 9.0
    step_fn = cs.cs_hier_step if a.hier_groups else cs.cs_gossip_step
    if a.skip_step:  # bounded cross-GPU waits: CS_ETIMEOUT (-13) after ~20 s, never a hang
        step_fn(x, bank[:n_loc], w, lr, mu)
        if rank == 0:
            step_fn(x, bank[:n_loc], w, lr, mu)
        code = 0
        try:
            cs.cs_sync()
        except cs.CSError as e:
            code = e.code
        ok_to = (code == -13) if rank == 0 else code == 0
        okt = torch.tensor([1 if ok_to else 0], device=dev)
        dist.all_reduce(okt, op=dist.ReduceOp.MIN)
        if rank == 0:
            print(f"skipped step: rank0 code {code}: {'OK' if okt.item() else 'FAIL'}", flush=True)
        dist.barrier()
        dist.destroy_process_group()
        sys.exit(0 if okt.item() else 1)
    if a.inject_nan:  # the flag must surface as CS_EDIVERGED (-10) on the rank that saw it
        g0 = bank[:n_loc].clone()
        if rank == 0:
            g0[0, d // 2] = float("nan")
        step_fn(x, bank[:n_loc], w, lr, mu)
        step_fn(x, g0, w, lr, mu)
        code = 0
        try:
            cs.cs_sync()
        except cs.CSError as e:
            code = e.code
        ok_nan = (code == -10) if rank == 0 else code in (0, -10)
        okt = torch.tensor([1 if ok_nan else 0], device=dev)
        dist.all_reduce(okt, op=dist.ReduceOp.MIN)
        if rank == 0:
            print(f"nan injection: rank0 code {code}: {'OK' if okt.item() else 'FAIL'}", flush=True)
        dist.barrier()
        dist.destroy_process_group()
        sys.exit(0 if okt.item() else 1)
    idx = torch.from_numpy(cols).to(dev)
    ok = True
    if a.diag:
        cs.cs_set_diag(True)
        from oracle.diagnostics import consensus
    for t in range(a.num_steps):
        o = (t + first) % B
        if gcur is not None:
            gcur.copy_(bank[o:o + n_loc])  # "backward" writes this step's gradient
            step_fn(x, gcur, w, lr, mu)
        else:
            step_fn(x, bank[o:o + n_loc], w, lr, mu)
        if a.lars:  # full rows (--compare-all): LARS needs whole layers
            g_all = synth.grads_at(orc.bank, world, orc.t)
            if a.hier_groups:  # LARS on the group-reduced gradient
                from oracle.lars import lars_hier_step
                orc.x, orc.m, orc.w, lrs = lars_hier_step(orc.x, orc.m, g_all, orc.w, a.hier_groups, seed, orc.t, k,
                                                          orc.seg, lb, lr, mu, ETA, WD, EPS)
                grp = first // (world // a.hier_groups)
                want = lrs[grp:grp + 1]
            else:
                orc.x, orc.m, orc.w, lrs = lars_gossip_step(orc.x, orc.m, g_all, orc.w,
                                                            T.topology(seed, orc.t, world, k), orc.seg, lb, lr, mu,
                                                            ETA, WD, EPS)
                want = lrs[first:first + n_loc]
            orc.t += 1
            got = cs.cs_get_lars_rates(n_loc, len(lb) - 1)
            if not np.all(np.abs(got.astype(np.float64) - want) <= np.spacing(np.abs(want))):
                print(f"rank {rank} step {t}: LARS rates differ by more than 1 ulp", flush=True)
                ok = False
                failed = True  # keep stepping in lockstep with the other ranks
        else:
            orc.step(lr, mu, src=exponential_topology(t, world, k) if a.exponential else None,
                     wire="bf16" if a.wire_bf16 else None)
        if a.sync_at_end and t < a.num_steps - 1:
            continue
        if a.stream_sync:
            stream.synchronize()
        else:
            cs.cs_sync()
        if a.diag:
            cd, msum = cs.cs_get_diag()
            cd0, ms0 = consensus(orc.x, orc.w, orc.seg)
            if not (abs(cd - cd0) <= 1e-9 * abs(cd0) and abs(msum - ms0) <= 1e-9 * max(1.0, abs(ms0)) + 1e-9 * d):
                print(f"rank {rank} step {t}: diagnostics {cd, msum} vs oracle {cd0, ms0}", flush=True)
                ok = False
                failed = True  # keep stepping in lockstep with the other ranks
        xs = x.index_select(1, idx).cpu().numpy()
        ms = m.index_select(1, idx).cpu().numpy()
        rows = slice(first, first + n_loc)
        # hierarchical: momentum is defined at leaders only (members hold a replica)
        gs = world // groups
        m_ok = np.array_equal(ms, orc.m[rows]) if (not a.hier_groups or first % gs == 0) else True
        lead = (first // gs) * gs
        if a.hier_groups and first % gs != 0:
            lead = (first // gs) * gs
            m_ok = np.array_equal(ms, orc.m[lead:lead + 1])  # the replica equals its leader's
        if a.lars:  # norms in another fp64 order: rates within 1 ulp, params within 1e-6
            xs_ok = np.all(np.abs(xs - orc.x[rows]) <= 1e-6 * np.abs(orc.x[rows]).max(axis=1, keepdims=True))
            # hierarchical members hold their leader's momentum (reading B-4)
            mref = orc.m[lead:lead + 1] if (a.hier_groups and first % gs != 0) else orc.m[rows]
            m_ok = np.all(np.abs(ms - mref) <= 1e-6 * np.abs(mref).max(axis=1, keepdims=True))
        elif (a.nvls or a.nccl) and gs > 2:  # the switch's / NCCL's summation order
            ref, refm = orc.x[rows], orc.m[lead:lead + 1] if first % gs != 0 else orc.m[rows]
            xs_ok = bool(np.all(np.linalg.norm((xs - ref).astype(np.float64), axis=1)
                                <= 1e-6 * np.linalg.norm(ref.astype(np.float64), axis=1))
                         and np.abs(xs - ref).max() <= 1e-6 * np.abs(ref).max())
            m_ok = bool(np.abs(ms - refm).max() <= 1e-6 * np.abs(refm).max())
        else:
            xs_ok = np.array_equal(xs, orc.x[rows])
        if a.hier_groups:  # members hold bit-identical replicas of their leader (P12)
            xt = torch.from_numpy(np.ascontiguousarray(xs)).to(dev)
            allx = [torch.empty_like(xt) for _ in range(ws)]
            dist.all_gather(allx, xt)
            lead_r = (first // gs) * gs // n_loc
            if not torch.equal(allx[lead_r], xt):
                print(f"rank {rank} step {t}: member differs from its leader", flush=True)
                ok = False
        if not (xs_ok and m_ok and np.array_equal(w.cpu().numpy(), orc.w[rows])):
            bad = np.argwhere(xs != orc.x[rows])
            print(f"rank {rank} step {t}: mismatch at {bad[:5].tolist()} of {bad.shape[0]}", flush=True)
            ok = False
            failed = True  # keep stepping in lockstep with the other ranks
    okt = torch.tensor([1 if ok else 0], device=dev)
    dist.all_reduce(okt, op=dist.ReduceOp.MIN)
    if rank == 0:
        print(f"mp parity world={world} groups={groups} n_loc={n_loc} d={d} k={k} steps={a.num_steps}: "
              f"{'OK' if okt.item() else 'FAIL'}", flush=True)
    dist.barrier()
    dist.destroy_process_group()
    cs.cs_finalize()
    sys.exit(0 if okt.item() else 1)


if __name__ == "__main__":
    main()
