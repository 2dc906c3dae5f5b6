mkdir -p gpurun_out
for cfg in "48 0" "48 4" "96 0" "96 4" "16 4" "200 4"; do
  set -- $cfg
  CS_PEER_WAVE_MB=$1 CS_PEER_MODE=$2 timeout 120 python bench.py --config c3 --workers-per-gpu 2 --path peer --steps 30 --warmup 5 --no-cpu --no-e2e > gpurun_out/sw1_$1_$2.log 2>&1
  CS_PEER_WAVE_MB=$1 CS_PEER_MODE=$2 timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2959$2 bench.py --gpus 2 --steps 30 --warmup 5 --config c3 --no-e2e > gpurun_out/sw2_$1_$2.log 2>&1
done
echo done
