"""Probe (context only, not product): does this box's NVSwitch fabric give multicast
(NVLS) to a process group, and what do NCCL and torch's multimem all-reduce reach on a
ResNet-50-sized fp32 vector?  Run under torchrun; prints one line per fact on rank 0."""
import os
import time

import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm_mem
from cuda.bindings import driver as cu

rank, ws = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
lr = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(lr)
dev = torch.device("cuda", lr)
dist.init_process_group("nccl", device_id=dev)
cu.cuInit(0)
_, cud = cu.cuDeviceGet(lr)
_, mc = cu.cuDeviceGetAttribute(cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, cud)
_, fab = cu.cuDeviceGetAttribute(cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, cud)
_, pos = cu.cuDeviceGetAttribute(
    cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED, cud)
if rank == 0:
    print(f"MULTICAST_SUPPORTED={mc} FABRIC_HANDLE={fab} POSIX_FD_HANDLE={pos}", flush=True)

d = 25_557_032
try:
    t = symm_mem.empty(d, device=dev, dtype=torch.float32)
    h = symm_mem.rendezvous(t, dist.group.WORLD.group_name)
    if rank == 0:
        print(f"symm_mem rendezvous ok: multicast_ptr={h.multicast_ptr:#x} "
              f"buffer_ptrs={[hex(p) for p in h.buffer_ptrs]}", flush=True)
    t.normal_()
    ok = h.multicast_ptr != 0
    if ok:
        for _ in range(5):
            torch.ops.symm_mem.multimem_all_reduce_(t, "sum", dist.group.WORLD.group_name)
        torch.cuda.synchronize()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            torch.ops.symm_mem.multimem_all_reduce_(t, "sum", dist.group.WORLD.group_name)
        b.record()
        torch.cuda.synchronize()
        us = a.elapsed_time(b) / 20 * 1e3
        tt = torch.tensor([us], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        if rank == 0:
            print(f"torch multimem_all_reduce_ fp32 x {d}: {tt.item():.1f} us", flush=True)
except Exception as e:  # noqa: BLE001
    if rank == 0:
        print(f"symm_mem failed: {type(e).__name__}: {e}", flush=True)

g = torch.randn(d, device=dev)
for _ in range(10):
    dist.all_reduce(g)
torch.cuda.synchronize()
dist.barrier()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(50):
    dist.all_reduce(g)
b.record()
torch.cuda.synchronize()
tt = torch.tensor([a.elapsed_time(b) / 50 * 1e3], device=dev)
dist.all_reduce(tt, op=dist.ReduceOp.MAX)
if rank == 0:
    busbw = 2 * (ws - 1) / ws * 4 * d / (tt.item() * 1e-6) / 1e9
    print(f"NCCL all_reduce fp32 x {d} over {ws} GPUs ({os.environ.get('NCCL_ALGO', 'default')}): "
          f"{tt.item():.1f} us, busbw {busbw:.0f} GB/s", flush=True)
dist.destroy_process_group()
