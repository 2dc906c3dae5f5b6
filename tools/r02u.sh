mkdir -p gpurun_out/r02u
timeout 900 python -m pytest tests/test_gpu_emulated.py -q > gpurun_out/r02u/emu.log 2>&1; echo EMU_RC=$? >> gpurun_out/r02u/emu.log
run() { tag=$1; shift; timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 100 --warmup 5 --no-e2e --no-interval --no-cpu "$@" > gpurun_out/r02u/${tag}_n${N}.log 2>&1; echo RC=$? >> gpurun_out/r02u/${tag}_n${N}.log; }
for N in 2 4; do
run c3 --config c3
run c3b --config c3
run c2 --config c2
done
