"""Context for the hierarchical step: NCCL all_reduce of a ResNet-50-sized fp32 vector
(25,557,032) over every GPU of the box, CUDA-event timed, max over ranks."""
import os

import torch
import torch.distributed as dist

rank, ws = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
d = 25_557_032
g = torch.randn(d, device="cuda")
for _ in range(10):
    dist.all_reduce(g)
torch.cuda.synchronize()
dist.barrier()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
steps = 50
a.record()
for _ in range(steps):
    dist.all_reduce(g)
b.record()
torch.cuda.synchronize()
t = torch.tensor([a.elapsed_time(b) / steps * 1e3], device="cuda")
dist.all_reduce(t, op=dist.ReduceOp.MAX)
if rank == 0:
    busbw = 2 * (ws - 1) / ws * 4 * d / (t.item() * 1e-6) / 1e9
    print(f"NCCL all_reduce fp32 x {d} over {ws} GPUs: {t.item():.1f} us, busbw {busbw:.0f} GB/s")
dist.destroy_process_group()
