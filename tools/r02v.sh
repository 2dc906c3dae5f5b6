mkdir -p gpurun_out/r02v
python tools/dbg_walk.py 15 > gpurun_out/r02v/dbg_walk.log 2>&1
timeout 900 python -m pytest tests/test_gpu_emulated.py -q > gpurun_out/r02v/emu.log 2>&1; echo EMU_RC=$? >> gpurun_out/r02v/emu.log
run() { tag=$1; shift; timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 100 --warmup 5 --no-e2e --no-interval --no-cpu "$@" > gpurun_out/r02v/${tag}_n${N}.log 2>&1; echo RC=$? >> gpurun_out/r02v/${tag}_n${N}.log; }
for N in 2 4; do
run c3 --config c3
run c2 --config c2
done
