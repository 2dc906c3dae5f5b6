# 2 GPUs: k_push_merge trace + lag sweep -> gpurun_out/r02m10/
O=gpurun_out/r02m10; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
B="--gpus 2 --steps 50 --warmup 5 --no-cpu --no-e2e --no-interval"
CS_MERGE_TRACE=20 timeout 300 $TR --master-port 29601 bench.py $B --config c3 > $O/trace_c3_n2.log 2>&1
CS_MERGE_TRACE=20 timeout 300 $TR --master-port 29602 bench.py $B --config c2 > $O/trace_c2_n2.log 2>&1
for lag in 0 1 4 8; do
  CS_MERGE_LAG=$lag timeout 300 $TR --master-port 29603 bench.py $B --config c3 > $O/bench_c3_lag${lag}_n2.log 2>&1
done
(cd .cmp/a34 && CS_MERGE_TRACE=20 timeout 300 $TR --master-port 29604 bench.py $B --config c3 > ../../$O/trace_c3_a34_n2.log 2>&1)
