"""world_size-2 host-side checks of the N > 1 path on CPU (gloo).

1. Shared-seed contract: every process computes the same per-segment topology
   from (seed, step) with no communication ("rseed ... shared by
   every process"; reading C-4) — the library's host generator, compared across
   ranks.
2. Partitioned exchange semantics: workers split contiguously over ranks, each
   sender pushes y_i[R_s] to send_to = dst_s(i) (Alg.1 l.6-7) and each receiver
   mixes its inbox (l.17).  Run with gloo isend/irecv between processes on the
   oracle's arithmetic, routed by the library's topology, and compared with the
   single-process oracle step (bitwise): the contract the NVLink kernel implements.
   Also with the bf16 wire (reading C-20: the sender's y rounded by torch's own bf16
   conversion, the weight in fp32) and with SGP's exponential graph
   (cs_set_topology_kind).
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


def _worker(rank, ws, port, n_loc, d, k, steps, q, wire=None, exponential=False):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_2012_15198_b200 as cs
    import synth
    from oracle import topology as T
    from oracle.gossip import gossip_step, local_update

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=ws)
    try:
        world, seed = n_loc * ws, 5
        first = rank * n_loc
        cs.cs_init(world, world, k, seed)
        if exponential:
            cs.cs_set_topology_kind(cs.TOPO_EXPONENTIAL)
        # 1. topology agreement across processes
        topo = torch.from_numpy(np.stack([cs.cs_topology(t, world, k) for t in range(steps)]))
        allt = [torch.zeros_like(topo) for _ in range(ws)]
        dist.all_gather(allt, topo)
        agree = all(torch.equal(a, topo) for a in allt)
        # 2. partitioned push exchange vs the single-process oracle
        b = T.segment_bounds(d, k)
        seg = T.segment_of_columns(b, np.arange(d))
        x_all = synth.init_params(seed, range(world), d)
        bank = synth.grad_bank(seed, world, d)
        m_all = np.zeros_like(x_all)
        w_all = np.ones((world, k), np.float32)
        x, m, w = x_all[first:first + n_loc].copy(), m_all[first:first + n_loc].copy(), w_all[first:first + n_loc].copy()
        lr, mu = synth.DEFAULT_LR, synth.DEFAULT_MOMENTUM
        for t in range(steps):
            src = cs.cs_topology(t, world, k)
            g_all = synth.grads_at(bank, world, t)
            x_all, m_all, w_all = gossip_step(x_all, m_all, g_all, w_all, src, seg, lr, mu, wire=wire)
            m, y = local_update(x, m, g_all[first:first + n_loc], lr, mu)
            inbox = np.zeros_like(y)
            wbox = np.zeros_like(w)
            reqs = []
            for s in range(k):
                dst = T.inverse(src[s])
                for r in range(n_loc):                      # push (isend) my segments
                    i = first + r
                    peer = dst[i]
                    # the wire carries y[R_s] (bf16 via torch's own rounding when wire="bf16",
                    # reading C-20) and the fp32 push-sum weight as a second message
                    ys = torch.from_numpy(y[r, b[s]:b[s + 1]].copy())
                    if wire == "bf16":
                        ys = ys.to(torch.bfloat16)
                    ws_ = torch.from_numpy(w[r, s:s + 1].copy())
                    if peer // n_loc == rank:
                        inbox[peer - first, b[s]:b[s + 1]] = ys.float().numpy()
                        wbox[peer - first, s] = ws_.item()
                    else:
                        reqs.append(dist.isend(ys, peer // n_loc, tag=s * world + peer))
                        reqs.append(dist.isend(ws_, peer // n_loc, tag=(k + s) * world + peer))
                for r in range(n_loc):                      # irecv what my workers receive
                    i = first + r
                    sender = int(src[s][i])
                    if sender // n_loc != rank:
                        buf = torch.zeros(b[s + 1] - b[s], dtype=torch.bfloat16 if wire == "bf16" else torch.float32)
                        wbuf = torch.zeros(1)
                        dist.recv(buf, sender // n_loc, tag=s * world + i)
                        dist.recv(wbuf, sender // n_loc, tag=(k + s) * world + i)
                        inbox[r, b[s]:b[s + 1]] = buf.float().numpy()
                        wbox[r, s] = wbuf.item()
            for rq in reqs:
                rq.wait()
            x = ((y + inbox).astype(np.float32) * np.float32(0.5)).astype(np.float32)
            w = ((w + wbox).astype(np.float32) * np.float32(0.5)).astype(np.float32)
        same = (np.array_equal(x, x_all[first:first + n_loc]) and np.array_equal(m, m_all[first:first + n_loc])
                and np.array_equal(w, w_all[first:first + n_loc]))
        q.put((rank, agree, same))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_loc,d,k,wire,exponential", [
    (1, 97, 2, None, False), (3, 200, 5, None, False), (4, 64, 2, None, False),
    (3, 200, 5, "bf16", False),   # bf16 wire (C-20), rounded by torch on the sender side
    (4, 96, 3, None, True),       # SGP's exponential graph from cs_set_topology_kind
    (2, 130, 4, "bf16", True),
])
def test_two_process_partitioned_exchange(n_loc, d, k, wire, exponential):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_loc, d, k, 4, q, wire, exponential)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, agree, same in res:
        assert agree, f"rank {rank}: topologies differ across processes"
        assert same, f"rank {rank}: partitioned exchange differs from the oracle"
