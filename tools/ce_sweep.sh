# Copy-engine exchange for one worker per GPU (CS_PEER_CE=1): parity, then c3 step time
# against the SM push/mix schedule, for several piece counts.
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
CS_PEER_CE=1 timeout 900 python -m pytest tests/test_gpu_multi.py -q -m gpu -k "parity or resnet50 or exponential or diagnostics" \
  > gpurun_out/ce_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ce_pytest.log
for cfg in "0 1" "1 1" "1 2" "1 4" "1 8"; do
  set -- $cfg
  CS_PEER_CE=$1 CS_PEER_CE_PIECES=$2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port 29931 bench.py --gpus $N --steps 100 --warmup 10 --config c3 \
    --no-e2e --no-interval > gpurun_out/ce_c3_n${N}_ce$1_p$2.log 2>&1
done
echo done
