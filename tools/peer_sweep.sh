# peer-exchange tuning sweep (run under gpurun --gpus 2)
mkdir -p gpurun_out
CS_PEER_ALGO=5 timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_parity.py -k "peer or two_gpu" -m gpu -q > gpurun_out/pytest_algo5.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_algo5.log
for cfg in "4 0" "5 48" "5 96" "5 24"; do
  set -- $cfg
  for c in c3 c2; do
    CS_PEER_ALGO=$1 CS_PEER_WAVE_MB=$2 timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29$1$2 bench.py --gpus 2 --steps 30 --warmup 5 --config $c --no-e2e > gpurun_out/sw2_a$1_w$2_$c.log 2>&1
  done
done
echo done
