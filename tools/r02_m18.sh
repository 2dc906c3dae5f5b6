# 2 GPUs: k_push_merge knobs on the final kernel (lag, slot-free lag, copies in flight) -> gpurun_out/r02m18/
O=gpurun_out/r02m18; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
B="--gpus 2 --steps 60 --warmup 5 --no-cpu --no-e2e --no-interval"
for v in "LAG=0" "LAG=4" "READLAG=1" "LAND=7"; do
  env CS_MERGE_$v timeout 300 $TR --master-port 29681 bench.py $B --config c2 > $O/bench_c2_${v}_n2.log 2>&1
  env CS_MERGE_$v timeout 300 $TR --master-port 29682 bench.py $B --config c3 > $O/bench_c3_${v}_n2.log 2>&1
done
