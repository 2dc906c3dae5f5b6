# peer-exchange tuning sweep (run under gpurun --gpus 2)
mkdir -p gpurun_out
CS_PEER_ALGO=2 timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_parity.py -k "peer or two_gpu" -m gpu -q > gpurun_out/pytest_algo2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_algo2.log
for cfg in "0 200" "2 0"; do
  set -- $cfg
  for c in c3 c2; do
    CS_PEER_ALGO=$1 CS_PEER_WAVE_MB=$2 timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2957$1 bench.py --gpus 2 --steps 30 --warmup 5 --config $c --no-e2e > gpurun_out/sw2_a$1_$c.log 2>&1
  done
  CS_PEER_ALGO=$1 CS_PEER_WAVE_MB=$2 timeout 120 python bench.py --config c3 --workers-per-gpu 2 --path peer --steps 30 --warmup 5 --no-cpu --no-e2e > gpurun_out/sw1_a$1.log 2>&1
  CS_PEER_ALGO=$1 CS_PEER_MODE=1 CS_PEER_WAVE_MB=$2 timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2958$1 bench.py --gpus 2 --steps 30 --warmup 5 --config c3 --no-e2e > gpurun_out/sw2_a$1_m1.log 2>&1
done
echo done
