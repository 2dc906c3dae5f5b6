# multi-GPU validation + benches (run under gpurun --gpus N)
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 1500 python -m pytest tests/test_gpu_multi.py -m gpu -q > gpurun_out/pytest_multi_n$N.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_multi_n$N.log
for c in c3 c4 c2 c5; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2970${#c} bench.py --gpus $N --steps 50 --warmup 5 --config $c --no-e2e > gpurun_out/bench_n${N}_$c.log 2>&1
done
echo done
