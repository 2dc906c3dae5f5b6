# 2 GPUs: tails' own y staged by cp.async; hierarchical pulled group mean -> gpurun_out/r02m6/
O=gpurun_out/r02m6; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0 timeout 600 python -m pytest tests/test_gpu_emulated.py -q > $O/pytest_emulated.log 2>&1; echo RC=$? >> $O/pytest_emulated.log
CUDA_VISIBLE_DEVICES=0 timeout 600 python tools/dbg_walk.py 6 > $O/dbg_walk.log 2>&1; echo RC=$? >> $O/dbg_walk.log
B="--gpus 2 --steps 100 --warmup 5 --no-cpu --no-e2e --no-interval"
for rep in 1 2; do
  timeout 300 $TR --master-port 29551 bench.py $B --config c3 > $O/bench_c3_${rep}_n2.log 2>&1
  timeout 300 $TR --master-port 29552 bench.py $B --config c2 > $O/bench_c2_${rep}_n2.log 2>&1
done
timeout 300 $TR --master-port 29553 bench.py $B --config c5 > $O/bench_c5_n2.log 2>&1
timeout 300 $TR --master-port 29554 bench.py $B --config c4 > $O/bench_c4_pull_n2.log 2>&1
CS_HIER_PULL=0 timeout 300 $TR --master-port 29555 bench.py $B --config c4 > $O/bench_c4_push_n2.log 2>&1
timeout 2400 python -m pytest tests/test_gpu_multi.py -q -m gpu > $O/pytest_multi_n2.log 2>&1; echo RC=$? >> $O/pytest_multi_n2.log
