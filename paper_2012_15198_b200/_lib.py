"""ctypes binding of include/crossover_sgd.h — marshalling only.

Tensors are passed as raw device pointers (`tensor.data_ptr()`), streams as the
raw `cudaStream_t` of a `torch.cuda.Stream`.  Each wrapper raises CSError on a
negative status.  No computation happens here.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libcrossover_sgd.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
        "(there is no CPU fallback)")

lib = ctypes.CDLL(LIB_PATH)

CS_MAX_WORLD = 1024
CS_QUANTUM = 32
CS_IPC_HANDLE_BYTES = 64
CS_TAG_FLAT = 0
CS_TAG_HIER = 1
CS_PATH_AUTO, CS_PATH_REG, CS_PATH_TMA, CS_PATH_PEER = 0, 1, 2, 3
CS_SCHED_INSTEP, CS_SCHED_DEFERRED, CS_SCHED_SPLIT = 0, 1, 2

STATUS = {
    0: "CS_OK", -1: "CS_EINVAL_WORLD", -2: "CS_EINVAL_GROUPS", -3: "CS_EINVAL_SEGMENTS",
    -4: "CS_ELAYOUT", -5: "CS_ETOPOLOGY", -6: "CS_EINVAL_TOPOLOGY", -7: "CS_ENOTINIT",
    -8: "CS_ENOTBOUND", -9: "CS_ECUDA", -10: "CS_EDIVERGED", -11: "CS_EINVAL",
    -12: "CS_EUNSUPPORTED", -13: "CS_ETIMEOUT",
}

_c_int, _c_i64, _c_u64, _c_f, _vp = ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, ctypes.c_float, ctypes.c_void_p

_SIGS = {
    "cs_init": (_c_int, [_c_int, _c_int, _c_int, _c_u64]),
    "cs_finalize": (None, []),
    "cs_last_error": (ctypes.c_char_p, []),
    "cs_version": (_c_int, []),
    "cs_build_id": (ctypes.c_char_p, []),
    "cs_segment_bounds": (_c_int, [_c_i64, _vp]),
    "cs_topology": (_c_int, [_c_i64, _vp]),
    "cs_topology_hier": (_c_int, [_c_i64, _vp]),
    "cs_bind": (_c_int, [_vp, _c_i64, _c_i64, _c_int, _c_int, _vp]),
    "cs_set_stream": (_c_int, [_vp]),
    "cs_set_path": (_c_int, [_c_int]),
    "cs_set_schedule": (_c_int, [_c_int]),
    "cs_test_emulate_ranks": (_c_int, [_c_int]),
    "cs_ipc_export": (_c_int, [_vp]),
    "cs_ipc_import": (_c_int, [_vp]),
    "cs_multicast_bytes": (_c_int, [_vp]),
    "cs_nccl_unique_id": (_c_int, [_vp]),
    "cs_set_hier_nccl": (_c_int, [_vp]),
    "cs_set_multicast": (_c_int, [_vp, _vp, _c_i64]),
    "cs_add_multicast_grads": (_c_int, [_vp, _vp, _c_i64]),
    "cs_gossip_step": (_c_int, [_vp, _vp, _vp, _c_f, _c_f]),
    "cs_gossip_step_host": (_c_int, [_vp, _vp, _vp, _c_f, _c_f, _vp]),
    "cs_gossip_step_io": (_c_int, [_vp, _vp, _vp, _c_f, _c_f, _vp, _vp]),
    "cs_hier_step": (_c_int, [_vp, _vp, _vp, _c_f, _c_f]),
    "cs_accumulate": (_c_int, [_vp, _vp, _c_int, _c_int]),
    "cs_set_topology_kind": (_c_int, [_c_int]),
    "cs_set_wire": (_c_int, [_c_int]),
    "cs_flush": (_c_int, []),
    "cs_segment_plan": (_c_int, [_vp, _c_int, _c_int, _vp]),
    "cs_set_layers": (_c_int, [_vp, _c_int, _vp]),
    "cs_set_lars": (_c_int, [_c_f, _c_f, _c_f]),
    "cs_get_lars_rates": (_c_int, [_vp]),
    "cs_set_lars_carry": (_c_int, [_c_int]),
    "cs_params_modified": (_c_int, []),
    "cs_set_step": (_c_int, [_c_i64]),
    "cs_get_step": (_c_int, [_vp]),
    "cs_set_diag": (_c_int, [_c_int]),
    "cs_get_diag": (_c_int, [_vp, _vp]),
    "cs_sync": (_c_int, []),
    "cs_test_set_topology": (_c_int, [_vp]),
    "cs_test_device_topology": (_c_int, [_c_i64, _c_int, _vp]),
    "cs_synth_fill": (_c_int, [_vp, _c_i64, _c_i64, _c_i64, _c_u64, _c_int, _c_i64, _c_f]),
    "cs_step_bytes": (_c_int, [_c_i64, _c_int, _vp]),
    "cs_set_timing": (_c_int, [_c_int]),
    "cs_get_timing": (_c_int, [_vp, _vp]),
    "cs_kernel_info": (ctypes.c_char_p, [_vp]),
}

for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args


def exported_symbols():
    return sorted(_SIGS)


class CSError(RuntimeError):
    def __init__(self, code: int, where: str):
        self.code = code
        self.status = STATUS.get(code, str(code))
        super().__init__(f"{where}: {self.status} ({code}): {cs_last_error()}")


def _check(rc: int, where: str) -> int:
    if rc < 0:
        raise CSError(rc, where)
    return rc


def _ptr(t) -> int:
    if t is None:
        return None
    if isinstance(t, int):
        return t
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def _stream_handle(stream) -> int | None:
    if stream is None:
        return None
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def cs_last_error() -> str:
    return lib.cs_last_error().decode()


def cs_version() -> int:
    return lib.cs_version()


def cs_build_id() -> str:
    return lib.cs_build_id().decode()


def cs_init(world: int, groups: int, k_segments: int, seed: int) -> None:
    _check(lib.cs_init(world, groups, k_segments, seed & 0xFFFFFFFFFFFFFFFF), "cs_init")


def cs_finalize() -> None:
    lib.cs_finalize()


def cs_segment_bounds(d: int, k: int) -> np.ndarray:
    out = np.zeros(k + 1, dtype=np.int64)
    _check(lib.cs_segment_bounds(d, out.ctypes.data), "cs_segment_bounds")
    return out


def cs_topology(step: int, world: int, k: int) -> np.ndarray:
    out = np.zeros((k, world), dtype=np.int32)
    _check(lib.cs_topology(step, out.ctypes.data), "cs_topology")
    return out


def cs_topology_hier(step: int, groups: int, k: int) -> np.ndarray:
    out = np.zeros((k, groups), dtype=np.int32)
    _check(lib.cs_topology_hier(step, out.ctypes.data), "cs_topology_hier")
    return out


def cs_bind(momentum, d: int, ld: int | None = None, proc_rank: int = 0, nprocs: int = 1,
            stream=None) -> None:
    ld = d if ld is None else ld
    _check(lib.cs_bind(_ptr(momentum), d, ld, proc_rank, nprocs, _stream_handle(stream)), "cs_bind")


def cs_set_stream(stream) -> None:
    _check(lib.cs_set_stream(_stream_handle(stream)), "cs_set_stream")


def cs_ipc_export() -> bytes:
    buf = ctypes.create_string_buffer(CS_IPC_HANDLE_BYTES)
    _check(lib.cs_ipc_export(buf), "cs_ipc_export")
    return buf.raw


def cs_ipc_import(handles: list[bytes]) -> None:
    blob = b"".join(handles)
    buf = ctypes.create_string_buffer(blob, len(blob))
    _check(lib.cs_ipc_import(buf), "cs_ipc_import")


def setup_peers(group=None) -> None:
    """Exchange exchange-region IPC handles over torch.distributed and map the peers."""
    import torch.distributed as dist
    mine = cs_ipc_export()
    allh = [None] * dist.get_world_size(group)
    dist.all_gather_object(allh, mine, group=group)
    cs_ipc_import(allh)
    dist.barrier(group=group)


def cs_multicast_bytes() -> int:
    out = ctypes.c_int64(0)
    _check(lib.cs_multicast_bytes(ctypes.byref(out)), "cs_multicast_bytes")
    return int(out.value)


def cs_set_multicast(uc_ptr: int, mc_ptr: int, nbytes: int) -> None:
    _check(lib.cs_set_multicast(uc_ptr or None, mc_ptr or None, nbytes), "cs_set_multicast")


def cs_add_multicast_grads(uc_ptr: int, mc_ptr: int, nbytes: int) -> None:
    _check(lib.cs_add_multicast_grads(uc_ptr, mc_ptr, nbytes), "cs_add_multicast_grads")


# Symmetric (multicast-bound) buffers handed to the library must outlive their use.
_MC_KEEP: list = []
_MC_GROUP = {}


def _hier_group(group_size: int):
    """This process's hierarchical group (contiguous ranks) as a torch process group."""
    import torch.distributed as dist
    if group_size not in _MC_GROUP:
        _MC_GROUP[group_size], _ = dist.new_subgroups(group_size=group_size)
    return _MC_GROUP[group_size]


def multicast_empty(shape, group_size: int, device):
    """Plumbing, no arithmetic: an fp32 tensor in torch symmetric memory rendezvoused over this
    process's hierarchical group, plus its multicast address (0 if the fabric has none).
    Collective over the whole job."""
    import torch
    import torch.distributed._symmetric_memory as symm_mem
    grp = _hier_group(group_size)
    t = symm_mem.empty(*shape, dtype=torch.float32, device=device)
    h = symm_mem.rendezvous(t, grp.group_name)
    mc = h.multicast_ptr
    if mc:
        mc += t.data_ptr() - h.buffer_ptrs[h.rank]
    _MC_KEEP.append((t, h))
    return t, mc


def setup_multicast(group_size: int, device) -> bool:
    """Registers a multicast workspace over this process's hierarchical group (cs_set_multicast)
    so cs_hier_step averages gradients in the NVSwitch.  False (nothing registered) if the
    fabric gives no multicast.  Collective over the whole job; call after setup_peers()."""
    import torch.distributed as dist
    nbytes = cs_multicast_bytes()
    t, mc = multicast_empty(((nbytes + 3) // 4,), group_size, device)
    ok = mc != 0
    flags = [None] * dist.get_world_size()
    dist.all_gather_object(flags, ok)
    if not all(flags):
        return False
    cs_set_multicast(t.data_ptr(), mc, 4 * t.numel())
    dist.barrier()
    return True


CS_NCCL_ID_BYTES = 128


def cs_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(CS_NCCL_ID_BYTES)
    _check(lib.cs_nccl_unique_id(buf), "cs_nccl_unique_id")
    return buf.raw


def cs_set_hier_nccl(group_id) -> None:
    _check(lib.cs_set_hier_nccl(ctypes.c_char_p(group_id) if group_id else None), "cs_set_hier_nccl")


def setup_hier_nccl(group_size: int) -> None:
    """Plumbing, no arithmetic: each group's first member draws an NCCL id, the ids are
    all-gathered over torch.distributed and every member joins its group's communicator
    (cs_set_hier_nccl).  Collective over the whole job; call after setup_peers()."""
    import torch.distributed as dist
    r = dist.get_rank()
    lead = (r // group_size) * group_size
    ids = [None] * dist.get_world_size()
    dist.all_gather_object(ids, cs_nccl_unique_id() if r == lead else None)
    cs_set_hier_nccl(ids[lead])
    dist.barrier()


def register_multicast_grads(t, mc: int) -> None:
    """Gradient rows inside `t` (from multicast_empty) are reduced in place by cs_hier_step."""
    cs_add_multicast_grads(t.data_ptr(), mc, 4 * t.numel())


def cs_gossip_step(params, grads, psw, lr: float, momentum: float) -> None:
    _check(lib.cs_gossip_step(_ptr(params), _ptr(grads), _ptr(psw), lr, momentum), "cs_gossip_step")


def cs_gossip_step_host(params, grads_host, psw, lr: float, momentum: float) -> tuple[float, float]:
    out = np.zeros(2, dtype=np.float64)
    _check(lib.cs_gossip_step_host(_ptr(params), _ptr(grads_host), _ptr(psw), lr, momentum,
                                   out.ctypes.data), "cs_gossip_step_host")
    return float(out[0]), float(out[1])


def cs_gossip_step_io(params, grads_host, psw, lr: float, momentum: float, params_host_out, psw_host_out) -> None:
    """One step with host-resident gradients in and the merged params / psw copied back to
    host buffers (pipelined column pieces; synchronous)."""
    _check(lib.cs_gossip_step_io(_ptr(params), _ptr(grads_host), _ptr(psw), lr, momentum, _ptr(params_host_out),
                                 _ptr(psw_host_out)), "cs_gossip_step_io")


def cs_hier_step(params, grads, psw, lr: float, momentum: float) -> None:
    _check(lib.cs_hier_step(_ptr(params), _ptr(grads), _ptr(psw), lr, momentum), "cs_hier_step")


def cs_accumulate(acc, grads, count: int, interval: int) -> None:
    """Micro-step `count` of a communication interval (Table 1):
    acc = 0 + g at count 0, acc += g after, acc /= interval at count interval-1."""
    _check(lib.cs_accumulate(_ptr(acc), _ptr(grads), count, interval), "cs_accumulate")


def cs_segment_plan(layer_sizes, k: int) -> np.ndarray:
    """Layer-aligned segment plan (SPEC build_segment_plan, Table 1): seg_of_layer."""
    sz = np.ascontiguousarray(layer_sizes, dtype=np.int64)
    out = np.zeros(len(sz), dtype=np.int32)
    _check(lib.cs_segment_plan(sz.ctypes.data, len(sz), k, out.ctypes.data), "cs_segment_plan")
    return out


def cs_set_layers(layer_bounds, seg_of_layer=None) -> None:
    """Layer table [n_layers + 1] of the bound vector, optionally the segment of each layer."""
    if layer_bounds is None:
        _check(lib.cs_set_layers(None, 0, None), "cs_set_layers")
        return
    lb = np.ascontiguousarray(layer_bounds, dtype=np.int64)
    sl = None if seg_of_layer is None else np.ascontiguousarray(seg_of_layer, dtype=np.int32)
    _check(lib.cs_set_layers(lb.ctypes.data, len(lb) - 1, None if sl is None else sl.ctypes.data),
           "cs_set_layers")


def cs_set_lars(eta: float, weight_decay: float = 0.0, eps: float = 0.0) -> None:
    """LARS in the flat step (Table 1); eta == 0 disables."""
    _check(lib.cs_set_lars(eta, weight_decay, eps), "cs_set_lars")


def cs_get_lars_rates(n_loc: int, n_layers: int) -> np.ndarray:
    out = np.zeros((n_loc, n_layers), dtype=np.float32)
    _check(lib.cs_get_lars_rates(out.ctypes.data), "cs_get_lars_rates")
    return out


TOPO_CROSSOVER, TOPO_EXPONENTIAL = 0, 1
WIRE_FP32, WIRE_BF16 = 0, 1


def cs_set_wire(fmt: int) -> None:
    """WIRE_FP32 (default) or WIRE_BF16: received segments rounded to bf16 (reading C-20)."""
    _check(lib.cs_set_wire(fmt), "cs_set_wire")


def cs_set_topology_kind(kind: int) -> None:
    """TOPO_CROSSOVER (Alg. 2, default) or TOPO_EXPONENTIAL (SGP's graph)."""
    _check(lib.cs_set_topology_kind(kind), "cs_set_topology_kind")


def cs_flush() -> None:
    """Complete deferred work (the multi-GPU deferred merge) on the bound stream."""
    _check(lib.cs_flush(), "cs_flush")


def cs_set_step(step: int) -> None:
    _check(lib.cs_set_step(step), "cs_set_step")


def cs_get_step() -> int:
    v = ctypes.c_int64(0)
    _check(lib.cs_get_step(ctypes.byref(v)), "cs_get_step")
    return v.value


def cs_set_diag(enable: bool) -> None:
    _check(lib.cs_set_diag(1 if enable else 0), "cs_set_diag")


def cs_get_diag() -> tuple[float, float]:
    cd, mean = ctypes.c_double(0.0), ctypes.c_double(0.0)
    _check(lib.cs_get_diag(ctypes.byref(cd), ctypes.byref(mean)), "cs_get_diag")
    return cd.value, mean.value


def cs_sync() -> None:
    _check(lib.cs_sync(), "cs_sync")


def cs_test_set_topology(src: np.ndarray | None) -> None:
    if src is None:
        _check(lib.cs_test_set_topology(None), "cs_test_set_topology")
        return
    arr = np.ascontiguousarray(src, dtype=np.int32)
    _check(lib.cs_test_set_topology(arr.ctypes.data), "cs_test_set_topology")


def cs_test_device_topology(step: int, n: int, k: int, tag: int = CS_TAG_FLAT) -> np.ndarray:
    out = np.zeros((k, n), dtype=np.int32)
    _check(lib.cs_test_device_topology(step, tag, out.ctypes.data), "cs_test_device_topology")
    return out


def cs_synth_fill(out, rows: int, d: int, ld: int, seed: int, tag: int, row0: int, scale: float) -> None:
    _check(lib.cs_synth_fill(_ptr(out), rows, d, ld, seed & 0xFFFFFFFFFFFFFFFF, tag, row0, scale),
           "cs_synth_fill")


def cs_step_bytes(step: int, hier: bool = False) -> tuple[float, float]:
    out = np.zeros(2, dtype=np.float64)
    _check(lib.cs_step_bytes(step, 1 if hier else 0, out.ctypes.data), "cs_step_bytes")
    return float(out[0]), float(out[1])


def cs_set_timing(enable: bool) -> None:
    _check(lib.cs_set_timing(1 if enable else 0), "cs_set_timing")


def cs_get_timing() -> tuple[float, int]:
    ms, n = ctypes.c_double(0.0), ctypes.c_int64(0)
    _check(lib.cs_get_timing(ctypes.byref(ms), ctypes.byref(n)), "cs_get_timing")
    return ms.value, n.value


def cs_kernel_info() -> tuple[str, int]:
    n = ctypes.c_int(0)
    name = lib.cs_kernel_info(ctypes.byref(n))
    return name.decode(), n.value


def cs_set_path(path: int) -> None:
    _check(lib.cs_set_path(path), "cs_set_path")


def cs_set_schedule(schedule: int) -> None:
    """CS_SCHED_INSTEP (default: merged params when the step's work completes),
    CS_SCHED_DEFERRED (opt-in: the merge runs in the next step; cs_flush before reading),
    CS_SCHED_SPLIT (push kernel + merge kernel)."""
    _check(lib.cs_set_schedule(schedule), "cs_set_schedule")


def cs_test_emulate_ranks(vranks: int) -> None:
    """Test hook: the multi-GPU protocol for `vranks` ranks on this one GPU (next cs_bind)."""
    _check(lib.cs_test_emulate_ranks(vranks), "cs_test_emulate_ranks")


def cs_set_lars_carry(enable: bool) -> None:
    """Opt in to reusing the previous LARS step's x norms (caller calls cs_params_modified
    after writing params itself)."""
    _check(lib.cs_set_lars_carry(1 if enable else 0), "cs_set_lars_carry")


def cs_params_modified() -> None:
    """Params were written outside the library: the next LARS step recomputes ||x||."""
    _check(lib.cs_params_modified(), "cs_params_modified")
