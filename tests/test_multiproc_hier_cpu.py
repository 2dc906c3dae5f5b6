"""world_size-2 host-side checks of the hierarchical N > 1 path on CPU (gloo).

The three steps of PAPER.md:197 (§3.3, Fig. 5) run as separate processes that
each hold a contiguous block of n_loc workers, with groups that sit inside one
process (G = 4, 8 workers), one per process (G = 2) or span both (G = 1):

h1  every member's gradient reaches its leader's process; the leader sums the
    group in ascending member order and scales by fp32(1/|G|) (reading C-12);
h2  leaders apply the momentum update and gossip segment s with the leader
    permutation the library's host generator draws (`cs_topology_hier`,
    reading C-13), each leader pushing y[R_s] and w_s to send_to = dst_s(G)
    (Alg. 1 l.6-7) and mixing its inbox (l.17);
h3  the leader's x', w' propagate to its members.

Routed by the library's topology, computed on the oracle's arithmetic, and
compared bitwise with the single-process `oracle.hierarchical.hier_step`: the
contract `cs_hier_step` implements across GPUs with its own NVLink reduce-scatter /
all-gather and the in-step merge kernel (or, opt-in, NCCL for h1).  With LARS the
leader's per-layer rates come from its x and the group-reduced gradient (PAPER.md:197
"LARS needs the gradient norm synchronised", reading C-18), compared with
`oracle.lars.lars_hier_step`.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import __graft_entry__ as entry

entry.build()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, ws, port, n_loc, d, k, groups, steps, q, lars=False):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_2012_15198_b200 as cs
    import synth
    from oracle import topology as T
    from oracle.gossip import local_update
    from oracle.hierarchical import hier_step
    from oracle.lars import lars_hier_step, lars_update, layer_lr

    F32 = np.float32
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=ws)
    try:
        world, seed = n_loc * ws, 11
        first = rank * n_loc
        gs = world // groups
        leaders = [G * gs for G in range(groups)]
        proc_of = lambda i: i // n_loc  # noqa: E731
        mine = lambda i: proc_of(i) == rank  # noqa: E731
        cs.cs_init(world, groups, k, seed)
        b = T.segment_bounds(d, k)
        seg = T.segment_of_columns(b, np.arange(d))
        x_all = synth.init_params(seed, range(world), d)
        # hierarchical state starts replicated within each group (members = leader)
        x_all = np.repeat(x_all[leaders], gs, axis=0)
        bank = synth.grad_bank(seed, world, d)
        m_all = np.zeros_like(x_all)
        w_all = np.ones((world, k), F32)
        x, m, w = (a[first:first + n_loc].copy() for a in (x_all, m_all, w_all))
        lr, mu = synth.DEFAULT_LR, synth.DEFAULT_MOMENTUM
        # LARS: 3 uneven layers, Table 1-style trust ratio (eta, wd, eps); PAPER.md:197 needs the
        # leader's rate from the group-reduced gradient (reading C-18)
        eta, wd, eps = 0.01, 1e-3, 1e-9
        lb = np.array([0, d // 5, d // 2 + 3, d])
        layer_of_col = np.searchsorted(lb, np.arange(d), side="right") - 1
        topo_ok = True
        for t in range(steps):
            g_all = synth.grads_at(bank, world, t)
            if lars:
                x_all, m_all, w_all, _ = lars_hier_step(x_all, m_all, g_all, w_all, groups, seed, t, k, seg,
                                                        lb, lr, mu, eta, wd, eps)
                srcL_oracle = T.topology(seed, t, groups, k, T.TAG_HIER) if groups >= 2 else None
            else:
                x_all, m_all, w_all, srcL_oracle = hier_step(x_all, m_all, g_all, w_all, groups, seed, t, k,
                                                            seg, lr, mu)
            g = g_all[first:first + n_loc]
            srcL = cs.cs_topology_hier(t, groups, k) if groups >= 2 else None
            if srcL is not None:
                topo_ok &= np.array_equal(srcL, srcL_oracle)
            # h1: members -> leader's process, summed in ascending member order
            reqs = []
            for i in range(first, first + n_loc):
                L = (i // gs) * gs
                if not mine(L):
                    reqs.append(dist.isend(torch.from_numpy(g[i - first].copy()), proc_of(L), tag=i))
            ybox, wL, yL = {}, {}, {}
            for G, L in enumerate(leaders):
                if not mine(L):
                    continue
                acc = None
                for i in range(L, L + gs):
                    if mine(i):
                        gi = g[i - first]
                    else:
                        buf = torch.zeros(d)
                        dist.recv(buf, proc_of(i), tag=i)
                        gi = buf.numpy()
                    acc = gi.astype(F32) if acc is None else (acc + gi).astype(F32)
                gbar = (acc * F32(1.0 / gs)).astype(F32)
                if lars:
                    rates = layer_lr(x[L - first][None], gbar[None], lb, lr, eta, wd, eps)
                    mL, y = lars_update(x[L - first][None], m[L - first][None], gbar[None], rates,
                                        layer_of_col, mu, wd)
                else:
                    mL, y = local_update(x[L - first][None], m[L - first][None], gbar[None], lr, mu)
                m[L - first], yL[G], wL[G] = mL[0], y[0], w[L - first].copy()
            for rq in reqs:
                rq.wait()
            # h2: leader gossip, push to send_to = dst_s(G)
            if srcL is not None:
                reqs = []
                for s in range(k):
                    dst = T.inverse(srcL[s])
                    for G in yL:
                        payload = np.concatenate([yL[G][b[s]:b[s + 1]], wL[G][s:s + 1]])
                        to = leaders[dst[G]]
                        if mine(to):
                            ybox[(dst[G], s)] = payload
                        else:
                            reqs.append(dist.isend(torch.from_numpy(payload), proc_of(to),
                                                   tag=world + s * groups + dst[G]))
                    for G in yL:
                        frm = leaders[int(srcL[s][G])]
                        if not mine(frm):
                            buf = torch.zeros(b[s + 1] - b[s] + 1)
                            dist.recv(buf, proc_of(frm), tag=world + s * groups + G)
                            ybox[(G, s)] = buf.numpy()
                for rq in reqs:
                    rq.wait()
                xL, wLn = {}, {}
                for G in yL:
                    xi, wi = np.empty(d, F32), np.empty(k, F32)
                    for s in range(k):
                        p = ybox[(G, s)]
                        xi[b[s]:b[s + 1]] = ((yL[G][b[s]:b[s + 1]] + p[:-1]).astype(F32) * F32(0.5)).astype(F32)
                        wi[s] = F32(F32(wL[G][s] + F32(p[-1])) * F32(0.5))
                    xL[G], wLn[G] = xi, wi
            else:
                xL, wLn = yL, wL
            # h3: leader -> members
            reqs = []
            base = world + k * groups
            for G, L in enumerate(leaders):
                if not mine(L):
                    continue
                payload = torch.from_numpy(np.concatenate([xL[G], wLn[G]]))
                for i in range(L, L + gs):
                    if mine(i):
                        x[i - first], w[i - first] = xL[G], wLn[G]
                    else:
                        reqs.append(dist.isend(payload, proc_of(i), tag=base + i))
            for i in range(first, first + n_loc):
                L = (i // gs) * gs
                if not mine(L):
                    buf = torch.zeros(d + k)
                    dist.recv(buf, proc_of(L), tag=base + i)
                    x[i - first], w[i - first] = buf.numpy()[:d], buf.numpy()[d:]
            for rq in reqs:
                rq.wait()
        sl = slice(first, first + n_loc)
        same = (np.array_equal(x, x_all[sl]) and np.array_equal(m, m_all[sl])
                and np.array_equal(w, w_all[sl]))
        q.put((rank, topo_ok, same))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_loc,d,k,groups,lars", [
    (4, 96, 2, 4, False),    # two groups inside each process
    (4, 200, 3, 2, False),   # one group per process: L = 2, forced leader swap (P12)
    (2, 97, 2, 1, False),    # one group spanning both processes: allreduce-SGD, no gossip
    (3, 160, 5, 3, False),   # group {2,3} spans the process boundary
    (3, 160, 5, 3, True),    # the same with LARS on the group-reduced gradient
    (2, 97, 2, 1, True),     # LARS with one group spanning both processes
])
def test_two_process_hierarchical(n_loc, d, k, groups, lars):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_loc, d, k, groups, 3, q, lars)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, topo_ok, same in res:
        assert topo_ok, f"rank {rank}: library leader topology differs from the oracle's"
        assert same, f"rank {rank}: partitioned hierarchical step differs from the oracle"
