# Round-end multi-GPU evidence: the whole multi-GPU suite, the driver's exact invocation
# (bench.py --gpus N with defaults: c2, e2e on) and the other configs, at every N of the box.
mkdir -p gpurun_out/final_multi
O=gpurun_out/final_multi
NMAX=$(nvidia-smi -L | wc -l)
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -m gpu > $O/pytest_multi_n$NMAX.log 2>&1
echo "rc=$?" >> $O/pytest_multi_n$NMAX.log
for N in 2 4 8; do
  [ "$N" -gt "$NMAX" ] && break
  DEVS=$(seq -s, 0 $((N - 1)))
  CUDA_VISIBLE_DEVICES=$DEVS timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port 2998$N bench.py --gpus $N > $O/bench_default_n$N.log 2>&1
  for c in c3 c4 c5; do
    CUDA_VISIBLE_DEVICES=$DEVS timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
      --master-addr 127.0.0.1 --master-port 2999$N bench.py --gpus $N --config $c --steps 100 --warmup 10 \
      > $O/bench_${c}_n$N.log 2>&1
  done
done
echo done
