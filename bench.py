#!/usr/bin/env python
"""Benchmark of the Crossover-SGD gossip step (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2|c3|c5|c1]

A "step" is one full pass of the hot path (device topology,
momentum-SGD update, segment exchange, mix, push-sum weights) over every worker.
N = 1 times BASELINE configs[1] (16 workers x 11,689,512 fp32, k = 8) on one GPU;
N > 1 keeps that per-GPU load (16 workers per GPU, world = 16 N; weak scaling)
with segments crossing GPUs over NVLink peer memory.  --config c3 is one worker
per GPU with a ResNet-50-sized vector (25,557,032), c5 eight workers per GPU.

value   = whole-job "params mixed+updated" GB/s = 4 B * world * d / step time
          (device-timed with CUDA events, max over ranks)
e2e     = the same metric through the host-buffer entry point cs_gossip_step_io (N = 1:
          grads copied host->device and the merged params + psw copied back every step,
          pipelined in column pieces); N > 1: grads H2D, cs_gossip_step, params + psw D2H
roofline = the hot kernel's algorithmic bytes / its CUDA-event duration vs the
          measured HBM copy peak (N = 1) or the measured NVLink peer bandwidth (N > 1);
          N > 1 adds the NVLink bytes the hardware counted (NVML) as `traffic`
cpu_baseline = the oracle (oracle/, plain NumPy) timed on this host on a bounded
          column sample of the same workload (rank 0, N = 1 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "gossip-step time and effective GB/s (params mixed+updated) vs HBM/NVLink roofline"
UNIT = "GB/s"
NVLINK_PEER_GBS = 770.0      # B200_PROFILING.md: measured peer copy per direction (nominal 900)
HBM_FALLBACK_GBS = 6650.0    # B200_PROFILING.md fallback when MEASURED_PEAKS.json is absent
HBM_NOMINAL_GBS = 8000.0     # north_star "~8 TB/s HBM" (B200_PROFILING.md: 7.7 HGX / 8 DGX)
NVLINK_NOMINAL_GBS = 900.0   # north_star "900 GB/s/dir NVLink"

WORKLOADS = {
    # name: (workers per GPU, d, k, description)
    "c1": (8, 1_000_000, 4, "8 workers x 1M fp32, k=4 (BASELINE configs[0])"),
    "c2": (16, 11_689_512, 8, "16 workers x ResNet-18-sized 11,689,512 fp32, k=8 (BASELINE configs[1])"),
    "c3": (1, 25_557_032, 8, "1 worker/GPU x ResNet-50-sized 25,557,032 fp32, k=8 (BASELINE configs[2])"),
    "c4": (1, 25_557_032, 16, "hierarchical: 1 worker/GPU, groups of 4 GPUs (or all GPUs if fewer), "
                              "ResNet-50-sized 25,557,032 fp32, k=16 (BASELINE configs[3])"),
    "c5": (8, 25_557_032, 8, "8 workers/GPU x ResNet-50-sized 25,557,032 fp32 (BASELINE configs[4])"),
    "c6": (16, 25_557_032, 18, "LARS (SURVEY 8(f) #2): 16 workers x ResNet-50's 161 tensors, segments = stem + "
                               "16 blocks + FC (k=18, Table 1), eta 0.0025, wd 5e-5, lr 9"),
}
LARS = {"c6": (0.0025, 5e-5, 1e-9, 9.0)}   # eta, weight decay, eps, lr (Table 1)


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic(workload: str):
    """dram bytes per launch of the hot kernel from a committed ncu --set full capture."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f).get(workload)
    return None


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons while the timed region runs."""

    def __init__(self, index: int, period_s: float = 0.01):
        self.index, self.period = index, period_s
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001
            self._nv = None
            return self
        names = {
            "hw_slowdown": getattr(self._nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "hw_thermal_slowdown": getattr(self._nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_thermal_slowdown": getattr(self._nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "sw_power_cap": getattr(self._nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake_slowdown": getattr(self._nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }

        def run():
            while not self._stop.is_set():
                try:
                    self.samples.append(self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM))
                    r = self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                    for k, bit in names.items():
                        if r & bit:
                            self.reasons.add(k)
                except Exception:  # noqa: BLE001
                    pass
                time.sleep(self.period)

        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


class NvlinkCounters:
    """Hardware NVLink byte counters of this GPU (NVML field values, summed over its links),
    read before and after the timed region: the NVLink traffic the step actually moved."""

    # (tx field, rx field, bytes per unit): byte counters, else the KiB throughput counters
    FIELDS = (("NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES", "NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES", 1),
              ("NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX", "NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX", 1024))

    def __init__(self, index: int):
        self.ok, self.source = False, None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            for tx, rx, unit in self.FIELDS:
                links = [l for l in range(18) if self._ok(tx, l) and self._ok(rx, l)]
                if links:
                    self.fields, self.links, self.unit = (tx, rx), links, unit
                    self.ok, self.source = True, f"NVML {tx}/{rx} over {len(links)} links"
                    break
        except Exception:  # noqa: BLE001
            self.ok = False

    def _ok(self, name, link):
        try:
            return self.nv.nvmlDeviceGetFieldValues(self.h, [(getattr(self.nv, name), link)])[0].nvmlReturn == 0
        except Exception:  # noqa: BLE001
            return False

    def read(self):
        """{tx, rx} bytes summed over the links, or None."""
        out = {}
        for key, name in zip(("tx", "rx"), self.fields):
            vals = self.nv.nvmlDeviceGetFieldValues(self.h, [(getattr(self.nv, name), l) for l in self.links])
            if any(v.nvmlReturn != 0 for v in vals):
                return None
            out[key] = sum(v.value.ullVal for v in vals) * self.unit
        return out


class OracleSample:
    """The oracle as it stands, on all n workers x the first `cols` columns of the workload."""

    def __init__(self, n: int, d: int, k: int, seed: int, cols: int, lars=None):
        import synth
        from oracle import topology as T
        from oracle.gossip import gossip_step
        self.synth, self.T, self.gossip_step = synth, T, gossip_step
        self.n, self.d, self.k, self.seed = n, d, k, seed
        self.lars = lars
        if lars is None:
            c = np.arange(min(cols, d))
            bounds = T.segment_bounds(d, k)
        else:
            # LARS needs whole layers: the first ResNet-50 layers that fit in `cols` (>= 1)
            from oracle.lars import lars_gossip_step, plan_bounds
            self.lars_step = lars_gossip_step
            sizes, block = synth.resnet50_layers()
            lb = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
            j = max(1, int(np.searchsorted(lb, min(cols, d), side="right")) - 1)
            self.lb = lb[:j + 1]
            c = np.arange(int(self.lb[-1]))
            bounds = plan_bounds(lb, block)
        self.cols = len(c)
        self.x = synth.init_params(seed, range(n), d, c)
        self.bank = synth.grad_bank(seed, n, d, c)
        self.seg = T.segment_of_columns(bounds, c)
        self.m = np.zeros_like(self.x)
        self.w = np.ones((n, k), np.float32)
        self.t = 0

    def step(self) -> float:
        t0 = time.perf_counter()
        src = self.T.topology(self.seed, self.t, self.n, self.k)
        g = self.synth.grads_at(self.bank, self.n, self.t)
        if self.lars is not None:
            eta, wd, eps, lr = self.lars
            self.x, self.m, self.w, _ = self.lars_step(self.x, self.m, g, self.w, src, self.seg, self.lb, lr,
                                                       self.synth.DEFAULT_MOMENTUM, eta, wd, eps)
        else:
            self.x, self.m, self.w = self.gossip_step(self.x, self.m, g, self.w, src, self.seg,
                                                      self.synth.DEFAULT_LR, self.synth.DEFAULT_MOMENTUM)
        self.t += 1
        return time.perf_counter() - t0

    def record(self, per_step: float, steps: int) -> dict:
        return {"value": 4.0 * self.n * self.cols / per_step / 1e9, "unit": UNIT, "cores": 1,
                "host_cores": len(os.sched_getaffinity(0)), "cpu_model": cpu_model(), "kind": "oracle",
                "sample": f"{self.n} workers x first {self.cols} of {self.d} columns, k={self.k}, {steps} steps, "
                          + ("LARS on whole layers, " if self.lars is not None else "")
                          + 
                          f"{per_step:.3f} s/step (NumPy elementwise, single-threaded)",
                "steps": steps, "s_per_step": per_step}


def cpu_oracle_sample(n: int, d: int, k: int, seed: int, budget_s: float, cols: int, lars=None):
    """Time the oracle for ~budget_s (at least one step) on a column sample."""
    o = OracleSample(n, d, k, seed, cols, lars)
    steps, el = 0, 0.0
    while steps == 0 or (el < budget_s and steps < 1000):
        el += o.step()
        steps += 1
    return o.record(el / steps, steps)


def emit(obj):
    print(json.dumps(obj), flush=True)


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def bench_config(args, desc, world, n_loc, d, k, lr, mu, world_size, lars):
    """The `config` object of both arms' JSON lines (the same dict for the same run)."""
    return {"workload": f"{args.config}: {desc}", "world": world, "workers_per_gpu": n_loc,
            "d": d, "k": k, "seed": 0, "lr": lr, "momentum": mu,
            "parallelism": f"workers partitioned over {world_size} GPU(s)", "scheme": args.scheme,
            "schedule": args.schedule, "wire": args.wire,
            "lars_x_norm_carry": bool(lars),
            "l2": f"inputs larger than L2 ({20.0 * n_loc * d / 1e9:.2f} GB moved per step per GPU)"}


def run_reference(args, rank, world_size):
    """The oracle as the reference arm: each of the W + K steps is one oracle step over
    all workers on a column sample sized so the whole run stays within ~90 s."""
    if rank != 0:
        return
    n_loc, d, k, desc = WORKLOADS[args.config]
    d = args.d or d
    k = args.k or k
    if args.workers_per_gpu:
        n_loc = args.workers_per_gpu
        desc += f" [{n_loc} workers per GPU]"
    n = n_loc * world_size
    total = args.steps + args.warmup
    lars = LARS.get(args.config)
    probe = OracleSample(n, d, k, 0, min(args.cpu_cols, 100_000, d), lars)
    probe.step()
    per_col = probe.step() / probe.cols
    cols = int(max(4096, min(args.cpu_cols, d, 60.0 / max(1, total) / per_col)))
    o = OracleSample(n, d, k, 0, cols, lars)
    cols = o.cols
    for _ in range(args.warmup):
        o.step()
    res = [o.record(dt, 1) for dt in (o.step() for _ in range(max(1, args.steps)))]
    v = statistics.median(r["value"] for r in res)
    ms_sample = statistics.median(r["s_per_step"] for r in res) * 1e3
    cb = dict(res[0])
    cb["value"] = v
    cb["sample"] = f"each step: one oracle step over {n} workers x the first {cols} of {d} columns, k={k}"
    lr = lars[3] if lars else float(__import__("synth").DEFAULT_LR)
    mu = float(__import__("synth").DEFAULT_MOMENTUM)
    emit({"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world_size,
          "steps": args.steps, "warmup": args.warmup,
          # measured: one timed oracle step = the column sample (the value is the same metric,
          # GB/s of params mixed and updated, so it needs no extrapolation)
          "ms_per_step": ms_sample,
          "ms_per_step_full_vector_extrapolated": ms_sample * d / cols,
          "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
          "data": "synthetic", "config": bench_config(args, desc, n, n_loc, d, k, lr, mu, world_size, lars),
          "cpu_baseline": cb,
          "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None, choices=sorted(WORKLOADS))
    ap.add_argument("--segments", dest="k", type=int, default=None, help="segment count k (default: the config's)")
    ap.add_argument("--workers-per-gpu", type=int, default=None)
    ap.add_argument("--vector-len", dest="d", type=int, default=None, help="parameters per worker (default: the config's)")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--cpu-cols", type=int, default=1_000_000)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-interval", action="store_true", help="skip the communication-interval sub-measurement")
    ap.add_argument("--hier-groups", type=int, default=0,
                    help="c4: number of groups (default: groups of 4 GPUs, or one group if fewer)")
    ap.add_argument("--wire", default="fp32", choices=["fp32", "bf16"],
                    help="SURVEY 8(f) #4: bf16 wire format for received segments (reading C-20)")
    ap.add_argument("--scheme", default="crossover", choices=["crossover", "sgp", "allreduce"],
                    help="SURVEY 8(f) #3 baselines on the same machinery: sgp = SGP's directed exponential "
                         "graph, model-wise (k=1 unless --k); allreduce = AllReduce-SGD (hierarchical, 1 group)")
    ap.add_argument("--schedule", default="instep", choices=["instep", "deferred", "split"],
                    help="multi-GPU step schedule (cs_set_schedule): instep = merged params when the step's "
                         "work completes (default); deferred = the merge runs inside the next step (opt-in, "
                         "params readable only after cs_flush); split = push kernel + merge kernel")
    ap.add_argument("--h1", default="auto", choices=["auto", "nvls", "nccl", "p2p"],
                    help="multi-GPU hierarchical gradient average: p2p = reduce-scatter + all-gather over peer "
                         "stores (bitwise); nccl = ncclAllReduce over the group's communicator "
                         "(cs_set_hier_nccl; NCCL's order, tolerance parity for groups >= 3); nvls = in-switch "
                         "reduction (cs_set_multicast), measured slower for fp32 (DESIGN §8); auto = the faster "
                         "measured route: nccl for one group of >= 3 GPUs, else p2p")
    ap.add_argument("--path", default="auto", choices=["auto", "reg", "tma", "peer"],
                    help="library kernel path (cs_set_path); peer with 1 GPU = single-GPU emulation")
    args = ap.parse_args()
    # the timing rules need W >= 3 untimed warm-up steps; the line reports the W actually run
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world_size = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.config is None:
        args.config = "c2"
    if args.impl == "reference":
        run_reference(args, rank, world_size)
        return

    import torch
    import torch.distributed as dist

    import __graft_entry__ as entry
    entry.build()
    import paper_2012_15198_b200 as cs
    import synth

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world_size > 1:
        dist.init_process_group("nccl", device_id=dev)

    n_loc, d, k, desc = WORKLOADS[args.config]
    d = args.d or d
    k = args.k or k
    if args.workers_per_gpu:
        n_loc = args.workers_per_gpu
        desc += f" [{n_loc} workers per GPU]"
    world = n_loc * world_size
    if world < 2:
        raise SystemExit(f"config {args.config} needs >= 2 workers in total")
    seed = 0
    lr, mu = float(synth.DEFAULT_LR), float(synth.DEFAULT_MOMENTUM)
    lars = LARS.get(args.config)
    if lars is not None:
        lr = lars[3]
    first = rank * n_loc
    B = world + 1

    hier = args.config == "c4" or args.scheme == "allreduce"
    groups = 1 if args.scheme == "allreduce" else (max(1, world // 4) if hier else world)
    if hier and args.hier_groups:
        groups = args.hier_groups
    if args.scheme == "sgp" and not args.k:
        k = 1
    cs.cs_init(world, groups, k, seed)
    if args.scheme == "sgp":
        cs.cs_set_topology_kind(cs.TOPO_EXPONENTIAL)
    if args.wire == "bf16":
        cs.cs_set_wire(cs.WIRE_BF16)
    cs.cs_set_schedule({"instep": cs.CS_SCHED_INSTEP, "deferred": cs.CS_SCHED_DEFERRED,
                        "split": cs.CS_SCHED_SPLIT}[args.schedule])
    step_fn = cs.cs_hier_step if hier else cs.cs_gossip_step
    cs.cs_set_path({"auto": 0, "reg": 1, "tma": 2, "peer": 3}[args.path])
    stream = torch.cuda.Stream(dev)
    with torch.cuda.stream(stream):
        x = torch.empty(n_loc, d, device=dev)
        m = torch.zeros(n_loc, d, device=dev)
        w = torch.ones(n_loc, k, device=dev)
    cs.cs_bind(m, d, d, rank, world_size, stream)
    gs_h = world // groups
    want_nvls = hier and world_size > 1 and gs_h > 1 and args.h1 == "nvls"
    with torch.cuda.stream(stream):
        bank = torch.empty(B + n_loc, d, device=dev)
    if lars is not None:
        sizes, block = synth.resnet50_layers()
        if d != sum(sizes):
            raise SystemExit("c6 needs the ResNet-50 vector (no --d)")
        cs.cs_set_layers(np.concatenate([[0], np.cumsum(sizes)]), block)
        cs.cs_set_lars(*lars[:3])
        cs.cs_set_lars_carry(True)  # the bench loop writes params only through the library
    cs.cs_synth_fill(x, n_loc, d, d, seed, synth.TAG_INIT, first, 1.0)
    cs.cs_synth_fill(bank, B, d, d, seed, synth.TAG_GRAD, 0, float(synth.GRAD_SCALE))
    stream.synchronize()
    bank[B:] = bank[:n_loc]
    torch.cuda.synchronize()
    h1 = "p2p" if hier and world_size > 1 and gs_h > 1 else None
    if world_size > 1:
        cs.setup_peers()
        if hier and gs_h > 1 and (args.h1 == "nccl" or (args.h1 == "auto" and gs_h >= 3 and groups == 1)):
            cs.setup_hier_nccl(gs_h)
            h1 = "nccl (ncclAllReduce over the group, the update scales by 1/|G|)"
        if want_nvls:
            if not cs.setup_multicast(gs_h, dev):
                raise SystemExit("--h1 nvls: this fabric gives no multicast")
            h1 = "nvls (in-switch reduce, gradient copied into the multicast workspace)"

    def grads(t):
        o = (t + first) % B
        return bank[o:o + n_loc]

    def barrier():
        if world_size > 1:
            dist.barrier()

    t = 0
    for _ in range(args.warmup):
        step_fn(x, grads(t), w, lr, mu)
        t += 1
    cs.cs_sync()
    barrier()
    torch.cuda.synchronize()

    hbm_b, nvl_b = 0.0, 0.0
    nvl_max = []
    for s in range(t, t + args.steps):
        hb, nb = cs.cs_step_bytes(s, hier)
        hbm_b += hb
        nvl_max.append(nb)
    cs.cs_set_timing(True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    nvc = NvlinkCounters(local_rank) if world_size > 1 else None
    with ClockSampler(local_rank) as clk:
        barrier()
        torch.cuda.synchronize()
        nv0 = nvc.read() if nvc and nvc.ok else None
        ev0.record(stream)
        for _ in range(args.steps):
            step_fn(x, grads(t), w, lr, mu)
            t += 1
        cs.cs_flush()  # the last step's deferred merge (multi-GPU push/mix) inside the timed region
        ev1.record(stream)
        torch.cuda.synchronize()
        nv1 = nvc.read() if nv0 is not None else None
        barrier()
    cs.cs_sync()
    ms = ev0.elapsed_time(ev1)
    kern_ms, kern_launches = cs.cs_get_timing()
    cs.cs_set_timing(False)
    hot_kernel, launches_per_step = cs.cs_kernel_info()
    nvl_b = float(sum(nvl_max))
    hw_tx = (nv1["tx"] - nv0["tx"]) / args.steps if nv1 else -1.0
    hw_rx = (nv1["rx"] - nv0["rx"]) / args.steps if nv1 else -1.0
    stats = torch.tensor([ms, kern_ms, nvl_b, hw_tx, hw_rx], dtype=torch.float64, device=dev)
    if world_size > 1:
        dist.all_reduce(stats, op=dist.ReduceOp.MAX)
    ms, kern_ms_max, nvl_b_max, hw_tx, hw_rx = stats.tolist()
    ms_step = ms / args.steps
    value = 4.0 * world * d / (ms_step * 1e-3) / 1e9

    # ---- e2e through the public API: grads from pinned host memory every step ----
    e2e = None
    if not args.no_e2e:
        esteps = max(2, args.e2e_steps)
        host_bank = torch.empty(B + n_loc, d, dtype=torch.float32, pin_memory=True)
        host_bank.copy_(bank.cpu())
        torch.cuda.synchronize()
        h2d = 4 * n_loc * d

        def hgrads(tt):
            o = (tt + first) % B
            return host_bank[o:o + n_loc]

        host_api = world_size == 1 and args.path != "peer" and lars is None
        xout = torch.empty(n_loc, d, pin_memory=True)   # the step's result: merged params and psw
        wout = torch.empty(n_loc, k, pin_memory=True)
        d2h = 4 * n_loc * d + 4 * n_loc * k
        if host_api:
            # cs_gossip_step_io: grads in from pinned host memory, merged params + psw out to
            # pinned host memory, in 8 column pieces that overlap both copy directions with
            # the step kernel; synchronous, so the events bracket complete round trips
            cs.cs_gossip_step_io(x, hgrads(t), w, lr, mu, xout, wout)   # warm the staging buffer
            t += 1
            e0 = time.perf_counter()
            torch.cuda.synchronize()
            ee0, ee1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ee0.record(stream)
            for _ in range(esteps):
                cs.cs_gossip_step_io(x, hgrads(t), w, lr, mu, xout, wout)
                t += 1
            ee1.record(stream)
            torch.cuda.synchronize()
            ems = ee0.elapsed_time(ee1)
            wall = time.perf_counter() - e0
        else:
            stage = torch.empty(n_loc, d, device=dev)
            barrier()
            torch.cuda.synchronize()
            ee0, ee1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0 = time.perf_counter()
            ee0.record(stream)
            with torch.cuda.stream(stream):
                for _ in range(esteps):
                    stage.copy_(hgrads(t), non_blocking=True)
                    step_fn(x, stage, w, lr, mu)
                    cs.cs_flush()  # no-op on the in-step schedule (a deferred merge otherwise)
                    xout.copy_(x, non_blocking=True)   # the step's result back to the host
                    wout.copy_(w, non_blocking=True)
                    stream.synchronize()
                    t += 1
            ee1.record(stream)
            torch.cuda.synchronize()
            barrier()
            ems = ee0.elapsed_time(ee1)
            wall = time.perf_counter() - e0
        et = torch.tensor([ems], dtype=torch.float64, device=dev)
        if world_size > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        ems = et.item()
        e2e = {"value": 4.0 * world * d / (ems / esteps * 1e-3) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": esteps,
               "ms_per_step": ems / esteps, "wall_s": wall,
               "api": ("cs_gossip_step_io (grads H2D, params + psw D2H, 8 pipelined column pieces)" if host_api
                       else "grads H2D + cs_gossip_step (merged in-step) + params and psw D2H, serial")}
        del host_bank, xout, wout

    hpeak, hpeak_src = hbm_peak()

    # ---- communication-interval mode (Table 1: I = 42) ------------------
    # one interval = I cs_accumulate micro-steps + one gossip round with the mean gradient;
    # the accumulate kernel is timed alone on the bound stream (12 B/param mid-interval)
    interval = None
    if not args.no_interval:
        I = 42
        acc = torch.empty(n_loc, d, device=dev)
        for u in range(I):  # warm-up interval
            cs.cs_accumulate(acc, grads(t + u), u, I)
        step_fn(x, acc, w, lr, mu)
        t += 1
        barrier()
        torch.cuda.synchronize()
        ia, ib, ic = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        ia.record(stream)
        for u in range(I):
            cs.cs_accumulate(acc, grads(t + u), u, I)
        ib.record(stream)
        step_fn(x, acc, w, lr, mu)
        t += 1
        ic.record(stream)
        torch.cuda.synchronize()
        barrier()
        acc_ms, int_ms = ia.elapsed_time(ib), ia.elapsed_time(ic)
        st = torch.tensor([acc_ms, int_ms], dtype=torch.float64, device=dev)
        if world_size > 1:
            dist.all_reduce(st, op=dist.ReduceOp.MAX)
        acc_ms, int_ms = st.tolist()
        acc_bytes = (8.0 + 12.0 * (I - 1)) * n_loc * d   # count 0 reads g only
        acc_ach = acc_bytes / (acc_ms * 1e-3) / 1e9
        interval = {"I": I, "ms_per_interval": int_ms, "accumulate_ms": acc_ms,
                    "accumulate_roofline": {"bound": "hbm", "achieved": acc_ach, "peak": hpeak, "unit": "GB/s",
                                            "frac": acc_ach / hpeak, "kernel": "k_accumulate",
                                            "bytes_formula": "(8 + 12 (I-1)) B x n_loc x d per interval"},
                    "gpu_launches": I + launches_per_step}
        del acc

    # ---- roofline of the hot kernel --------------------------------------------------
    avg_kern_s = kern_ms_max / max(1, kern_launches) * 1e-3
    hbm_per_launch = hbm_b / args.steps
    hbm_ach = hbm_per_launch / avg_kern_s / 1e9
    roof_hbm = {"bound": "hbm", "achieved": hbm_ach, "peak": hpeak, "unit": "GB/s", "frac": hbm_ach / hpeak,
                "traffic": ncu_traffic(f"{args.config}" + ("" if args.path == "auto" else f":{args.path}")
                                       + ("" if world_size == 1 else f"@{world_size}")),
                "peak_source": hpeak_src, "kernel": hot_kernel,
                "algorithmic_bytes_per_launch": hbm_per_launch, "bytes_formula": ("24 B x n_loc x d (LARS g-norm 4 B, x norms carried from the previous step, + step 20 B)"
                                                                   if lars and world_size == 1 else
                                                                   "28 B x n_loc x d (LARS norms 8 B + step 20 B)" if lars else
                                                                   "20 B x n_loc x d"),
                "avg_kernel_us": avg_kern_s * 1e6, "launches_timed": kern_launches,
                "peak_nominal": HBM_NOMINAL_GBS, "frac_nominal": hbm_ach / HBM_NOMINAL_GBS}
    if world_size == 1:
        roofline = roof_hbm
    else:
        # the step is bound by whichever resource needs longer for its algorithmic bytes
        nvl_per_launch = nvl_b_max / args.steps
        nvl_ach = nvl_per_launch / avg_kern_s / 1e9
        # traffic: the hardware NVLink counters (NVML) over the timed region, per step, on the
        # GPU that moved the most, in the direction the algorithmic bytes count (into a GPU)
        traffic = {"rx_bytes_per_step": hw_rx, "tx_bytes_per_step": hw_tx,
                   "rx_over_algorithmic": hw_rx / nvl_per_launch if nvl_per_launch else None,
                   "source": (nvc.source if nvc else "") + ", max over ranks"} \
            if hw_rx >= 0 else None
        roof_nvl = {"bound": "nvlink", "achieved": nvl_ach, "peak": NVLINK_PEER_GBS, "unit": "GB/s",
                    "frac": nvl_ach / NVLINK_PEER_GBS, "traffic": traffic,
                    "achieved_hw_rx": hw_rx / avg_kern_s / 1e9 if hw_rx >= 0 else None,
                    "peak_source": "measured peer copy per direction (B200_PROFILING.md; 900 nominal)",
                    "kernel": hot_kernel, "algorithmic_bytes_per_launch": nvl_per_launch,
                    "bytes_formula": "4 B x remote-sourced segment elements (exact from the topology), "
                                     "most-loaded GPU; hierarchical adds the in-group reduce-scatter + all-gather",
                    "avg_kernel_us": avg_kern_s * 1e6, "launches_timed": kern_launches,
                    "peak_nominal": NVLINK_NOMINAL_GBS, "frac_nominal": nvl_ach / NVLINK_NOMINAL_GBS}
        t_nvl = nvl_per_launch / (NVLINK_PEER_GBS * 1e9)
        t_hbm = hbm_per_launch / (hpeak * 1e9)
        roofline = dict(roof_nvl if t_nvl >= t_hbm else roof_hbm)
        roofline["other"] = roof_hbm if t_nvl >= t_hbm else roof_nvl

    cpu = None
    if rank == 0 and world_size == 1 and not args.no_cpu:
        cpu = cpu_oracle_sample(n_loc * world_size, d, k, seed, args.cpu_seconds, args.cpu_cols, lars)

    if rank == 0:
        emit({"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world_size, "steps": args.steps,
              "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
              "vs_baseline": None, "dtype": "f32", "data": "synthetic",
              "config": {**bench_config(args, desc, world, n_loc, d, k, lr, mu, world_size, lars),
                         **({"h1": h1, "groups": groups} if hier else {})},
              "step_us": ms_step * 1e3,
              "traffic_GBps": 20.0 * world * d / (ms_step * 1e-3) / 1e9,
              "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "interval": interval,
              "gpu_launches": launches_per_step * args.steps + (1 if "fused" in hot_kernel else 0),  # + the flush
              "clocks": clk.summary()})
    if world_size > 1:
        dist.barrier()
        dist.destroy_process_group()
    cs.cs_finalize()


if __name__ == "__main__":
    main()
