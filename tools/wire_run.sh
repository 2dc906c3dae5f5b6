# bf16 wire format: tests + c3/c2 bench at every N of this box, fp32 vs bf16.
mkdir -p gpurun_out
NMAX=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_gpu_wire.py tests/test_gpu_multi.py -q -m gpu -k "wire or bf16" \
  > gpurun_out/wire_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/wire_pytest.log
for N in 2 4 8; do
  [ "$N" -gt "$NMAX" ] && break
  DEVS=$(seq -s, 0 $((N - 1)))
  for c in c3 c2; do
    for wire in fp32 bf16; do
      CUDA_VISIBLE_DEVICES=$DEVS timeout 300 python -m torch.distributed.run --nnodes=1 \
        --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2990$N bench.py --gpus $N \
        --steps 50 --warmup 5 --config $c --wire $wire --no-e2e --no-interval \
        > gpurun_out/wire_n${N}_${c}_${wire}.log 2>&1
    done
  done
done
echo done
