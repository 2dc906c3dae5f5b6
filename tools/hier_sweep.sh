# Hierarchical step with one group (AllReduce-SGD, c3 vector) for CS_HIER_PIECES = 1, 2, 4, 8
# (column pieces: the update of piece q on a second stream overlaps h1 of piece q+1).
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
for P in 1 2 4 8; do
  CS_HIER_PIECES=$P timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port 29921 bench.py --gpus $N --steps 50 --warmup 5 --config c3 \
    --scheme allreduce --no-e2e --no-interval > gpurun_out/hsweep_p$P.log 2>&1
done
echo done
