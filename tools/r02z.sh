mkdir -p gpurun_out/r02z
python tools/dbg_walk.py 8 > gpurun_out/r02z/dbg_walk.log 2>&1
timeout 900 python -m pytest tests/test_gpu_emulated.py -q > gpurun_out/r02z/emu.log 2>&1; echo EMU_RC=$? >> gpurun_out/r02z/emu.log
run() { tag=$1; shift; timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 50 --warmup 5 --no-e2e --no-interval --no-cpu "$@" > gpurun_out/r02z/${tag}_n${N}.log 2>&1; echo RC=$? >> gpurun_out/r02z/${tag}_n${N}.log; }
N=2
timeout 200 python tools/dbg_c2.py 16 11689512 > gpurun_out/r02z/dbg_c2.log 2>&1
CS_MERGE_TRACE=20 run c2tr --config c2
run c3 --config c3
N=4; run c2 --config c2; run c3 --config c3
