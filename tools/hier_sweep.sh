# Hierarchical step with one group (AllReduce-SGD, c3 vector): copy engines x column pieces.
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
for cfg in "0 1" "1 2" "1 4" "1 8"; do
  set -- $cfg
  CS_HIER_CE=$1 CS_HIER_PIECES=$2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port 29921 bench.py --gpus $N --steps 50 --warmup 5 --config c3 \
    --scheme allreduce --no-e2e --no-interval > gpurun_out/hsweep_ce$1_p$2.log 2>&1
done
CS_HIER_CE=1 CS_HIER_PIECES=4 timeout 900 python -m pytest tests/test_gpu_multi.py -q -m gpu -k "hier" > gpurun_out/hier_pytest_ce.log 2>&1
echo "rc=$?" >> gpurun_out/hier_pytest_ce.log
echo done
