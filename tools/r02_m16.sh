# 2 GPUs: copies in flight per SM (CS_MERGE_LAND) for one worker per GPU -> gpurun_out/r02m16/
O=gpurun_out/r02m16; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
B="--gpus 2 --steps 100 --warmup 5 --no-cpu --no-e2e --no-interval"
for land in 1 2 4 7; do
  CS_MERGE_LAND=$land timeout 300 $TR --master-port 29661 bench.py $B --config c3 > $O/bench_c3_land${land}_n2.log 2>&1
  CS_MERGE_LAND=$land timeout 300 $TR --master-port 29662 bench.py $B --config c3 --wire bf16 > $O/bench_c3bf16_land${land}_n2.log 2>&1
done
for land in 4 7; do
  CS_MERGE_LAND=$land timeout 300 $TR --master-port 29663 bench.py $B --config c2 > $O/bench_c2_land${land}_n2.log 2>&1
done
timeout 300 $TR --master-port 29664 bench.py $B --config c5 > $O/bench_c5_n2.log 2>&1
