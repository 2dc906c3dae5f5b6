mkdir -p gpurun_out/merge_sweep
timeout 400 python -m pytest tests/test_gpu_emulated.py -x -q > gpurun_out/merge_sweep/emu.log 2>&1; echo EMU_RC=$? >> gpurun_out/merge_sweep/emu.log
run() { tag=$1; shift; env "$@" timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --config c3 --steps 100 --warmup 5 --no-e2e --no-interval --no-cpu $EXTRA > gpurun_out/merge_sweep/c3_n${N}_$tag.log 2>&1; echo RC=$? >> gpurun_out/merge_sweep/c3_n${N}_$tag.log; }
for N in 2 4; do
EXTRA= run l0 CS_MERGE_LAG=0
EXTRA= run l2 CS_MERGE_LAG=2
EXTRA= run l4 CS_MERGE_LAG=4
EXTRA= run l2tr CS_MERGE_LAG=2 CS_MERGE_TRACE=30
EXTRA= run l2c2 CS_MERGE_LAG=2 CS_MERGE_CHUNK=2
done
