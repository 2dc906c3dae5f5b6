# 2 GPUs: the mix follows the inbox slots (no position polling), per-warp counters without a
# barrier -> gpurun_out/r02m17/
O=gpurun_out/r02m17; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0 timeout 600 python -m pytest tests/test_gpu_emulated.py -q > $O/pytest_emulated.log 2>&1; echo RC=$? >> $O/pytest_emulated.log
CUDA_VISIBLE_DEVICES=0 timeout 600 python tools/dbg_walk.py 6 > $O/dbg_walk.log 2>&1; echo RC=$? >> $O/dbg_walk.log
grep -q "fails 0" $O/dbg_walk.log || exit 0
B="--gpus 2 --steps 100 --warmup 5 --no-cpu --no-e2e --no-interval"
for rep in 1 2; do
  timeout 300 $TR --master-port 29671 bench.py $B --config c3 > $O/bench_c3_${rep}_n2.log 2>&1
  timeout 300 $TR --master-port 29672 bench.py $B --config c2 > $O/bench_c2_${rep}_n2.log 2>&1
done
