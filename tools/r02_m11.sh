# 2 GPUs: k_push_merge lag / slot-free sweep (relaxed position polls) -> gpurun_out/r02m11/
O=gpurun_out/r02m11; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
B="--gpus 2 --steps 50 --warmup 5 --no-cpu --no-e2e --no-interval"
for rl in 4 2 1 0; do
  for lag in 0 2; do
    CS_MERGE_READLAG=$rl CS_MERGE_LAG=$lag timeout 300 $TR --master-port 29611 bench.py $B --config c3 > $O/bench_c3_rl${rl}_lag${lag}_n2.log 2>&1
    CS_MERGE_READLAG=$rl CS_MERGE_LAG=$lag timeout 300 $TR --master-port 29612 bench.py $B --config c2 > $O/bench_c2_rl${rl}_lag${lag}_n2.log 2>&1
  done
done
CS_MERGE_TRACE=20 CS_MERGE_READLAG=1 CS_MERGE_LAG=0 timeout 300 $TR --master-port 29613 bench.py $B --config c3 > $O/trace_c3_rl1_lag0_n2.log 2>&1
