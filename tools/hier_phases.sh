# Per-phase times of the multi-GPU hierarchical step (CS_PHASE_TIMING=1), plus NCCL all_reduce
# of the same vector for context.  Run under gpurun --gpus N.
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
CS_PHASE_TIMING=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
  --master-addr 127.0.0.1 --master-port 29911 bench.py --gpus $N --steps 50 --warmup 5 --config c4 --no-e2e \
  --no-interval > gpurun_out/phases_c4_n$N.log 2>&1
CS_PHASE_TIMING=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
  --master-addr 127.0.0.1 --master-port 29912 bench.py --gpus $N --steps 50 --warmup 5 --config c3 \
  --scheme allreduce --no-e2e --no-interval > gpurun_out/phases_ar_n$N.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
  --master-port 29913 tools/nccl_allreduce.py > gpurun_out/nccl_ar_n$N.log 2>&1
echo done
