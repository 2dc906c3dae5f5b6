# Fig. 9 analogue: Crossover-SGD vs SGP vs AllReduce-SGD step
# time on the same machinery, for N = 1, 2, 4, ... GPUs of this box: one worker per GPU with
# the ResNet-50 vector (c3, N >= 2) and 16 workers per GPU (c2).  Run under gpurun --gpus N.
mkdir -p gpurun_out
NMAX=$(nvidia-smi -L | wc -l)
for N in 1 2 4 8; do
  [ "$N" -gt "$NMAX" ] && break
  DEVS=$(seq -s, 0 $((N - 1)))
  for scheme in crossover sgp allreduce; do
    for c in c3 c2; do
      [ "$N" = 1 ] && [ "$c" = c3 ] && continue
      # the multi-GPU hierarchical step (AllReduce-SGD = 1 group) takes one worker per GPU
      [ "$N" != 1 ] && [ "$c" = c2 ] && [ "$scheme" = allreduce ] && continue
      log=gpurun_out/scheme_n${N}_${c}_${scheme}.log
      if [ "$N" = 1 ]; then
        CUDA_VISIBLE_DEVICES=$DEVS timeout 300 python bench.py --steps 50 --warmup 5 --config $c \
          --scheme $scheme --no-e2e --no-cpu --no-interval > $log 2>&1
      else
        CUDA_VISIBLE_DEVICES=$DEVS timeout 300 python -m torch.distributed.run --nnodes=1 \
          --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2980$N bench.py --gpus $N \
          --steps 50 --warmup 5 --config $c --scheme $scheme --no-e2e --no-interval > $log 2>&1
      fi
    done
  done
done
echo done
