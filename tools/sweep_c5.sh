# BASELINE configs[4] scaling sweep on the GPUs of this box: 8 workers per GPU, segment count
# k = 1..32, vector 25.6M and 100M fp32 (bench.py --config c5 --segments K --vector-len D).
mkdir -p gpurun_out/sweep
N=$(nvidia-smi -L | wc -l)
for D in 25557032 100000000; do
  for K in 1 2 4 8 16 32; do
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port 29951 bench.py --gpus $N --steps 30 --warmup 5 --config c5 --segments $K --vector-len $D --no-e2e \
      --no-interval > gpurun_out/sweep/c5_n${N}_d${D}_k${K}.log 2>&1
  done
done
echo done
