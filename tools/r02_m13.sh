# 2 GPUs: lane-0 polls without back-off vs all-lane polls (git stash of r02m11) -> gpurun_out/r02m13/
O=gpurun_out/r02m13; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
B="--gpus 2 --steps 100 --warmup 5 --no-cpu --no-e2e --no-interval"
for rep in 1 2; do
  timeout 300 $TR --master-port 29631 bench.py $B --config c3 > $O/bench_c3_${rep}_n2.log 2>&1
  timeout 300 $TR --master-port 29632 bench.py $B --config c2 > $O/bench_c2_${rep}_n2.log 2>&1
  (cd .cmp/m11 && timeout 300 $TR --master-port 29633 bench.py $B --config c3 > ../../$O/bench_c3_m11_${rep}_n2.log 2>&1)
  (cd .cmp/m11 && timeout 300 $TR --master-port 29634 bench.py $B --config c2 > ../../$O/bench_c2_m11_${rep}_n2.log 2>&1)
  (cd .cmp/a34 && timeout 300 $TR --master-port 29635 bench.py $B --config c3 > ../../$O/bench_c3_a34_${rep}_n2.log 2>&1)
done
