# peer-exchange tuning sweep (run under gpurun --gpus 2)
mkdir -p gpurun_out
CS_PEER_ALGO=4 timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_parity.py -k "peer or two_gpu" -m gpu -q > gpurun_out/pytest_algo4.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_algo4.log
for algo in 2 4; do
  for tp in 0 1; do
    if [ $tp = 1 ]; then export CS_PEER_TIME_PUSH=1; else unset CS_PEER_TIME_PUSH; fi
    CS_PEER_ALGO=$algo timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 295$algo$tp bench.py --gpus 2 --steps 30 --warmup 5 --config c3 --no-e2e > gpurun_out/sw2_a${algo}_t${tp}_c3.log 2>&1
  done
  unset CS_PEER_TIME_PUSH
  CS_PEER_ALGO=$algo timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2966$algo bench.py --gpus 2 --steps 30 --warmup 5 --config c2 --no-e2e > gpurun_out/sw2_a${algo}_c2.log 2>&1
  CS_PEER_ALGO=$algo timeout 120 python bench.py --config c3 --workers-per-gpu 2 --path peer --steps 30 --warmup 5 --no-cpu --no-e2e > gpurun_out/sw1_a${algo}.log 2>&1
done
echo done
