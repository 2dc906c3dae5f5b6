# 2 GPUs: warp-lane-0 position polls with back-off -> gpurun_out/r02m12/
O=gpurun_out/r02m12; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0 timeout 600 python -m pytest tests/test_gpu_emulated.py -q > $O/pytest_emulated.log 2>&1; echo RC=$? >> $O/pytest_emulated.log
CUDA_VISIBLE_DEVICES=0 timeout 600 python tools/dbg_walk.py 6 > $O/dbg_walk.log 2>&1; echo RC=$? >> $O/dbg_walk.log
B="--gpus 2 --steps 100 --warmup 5 --no-cpu --no-e2e --no-interval"
for rep in 1 2; do
  timeout 300 $TR --master-port 29621 bench.py $B --config c3 > $O/bench_c3_${rep}_n2.log 2>&1
  timeout 300 $TR --master-port 29622 bench.py $B --config c2 > $O/bench_c2_${rep}_n2.log 2>&1
done
CS_MERGE_LAG=0 timeout 300 $TR --master-port 29623 bench.py $B --config c3 > $O/bench_c3_lag0_n2.log 2>&1
CS_MERGE_TRACE=20 timeout 300 $TR --master-port 29624 bench.py $B --config c3 > $O/trace_c3_n2.log 2>&1
