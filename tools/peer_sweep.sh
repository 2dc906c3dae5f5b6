# peer-exchange tuning sweep (run under gpurun --gpus 2)
mkdir -p gpurun_out
for P in 1 2 3; do
  for c in c3 c2; do
    CS_PEER_PIECES=$P timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 296$P${#c} bench.py --gpus 2 --steps 30 --warmup 5 --config $c --no-e2e > gpurun_out/sw2_p${P}_$c.log 2>&1
  done
done
echo done
