# 2 GPUs: NVLS h1 parity + bench, NVLink counters, c3/c2 vs the two previous commits -> gpurun_out/r02m3/
O=gpurun_out/r02m3; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multi.py -q -m gpu -k "nvls or hierarchical" > $O/pytest_nvls_n2.log 2>&1; echo RC=$? >> $O/pytest_nvls_n2.log
B="--gpus 2 --steps 100 --warmup 5 --no-cpu --no-e2e --no-interval"
for h in p2p nvls nvls-staged; do
  timeout 300 $TR --master-port 29521 bench.py $B --config c4 --h1 $h > $O/bench_c4_${h}_n2.log 2>&1; echo RC=$? >> $O/bench_c4_${h}_n2.log
done
timeout 300 $TR --master-port 29522 bench.py $B --config c4 --scheme allreduce > $O/bench_allreduce_n2.log 2>&1
for rep in 1 2; do
  timeout 300 $TR --master-port 29523 bench.py $B --config c3 > $O/bench_c3_head_${rep}_n2.log 2>&1
  (cd .cmp/e71 && timeout 300 $TR --master-port 29524 bench.py $B --config c3 > ../../$O/bench_c3_e71_${rep}_n2.log 2>&1)
  (cd .cmp/a34 && timeout 300 $TR --master-port 29525 bench.py $B --config c3 > ../../$O/bench_c3_a34_${rep}_n2.log 2>&1)
done
timeout 300 $TR --master-port 29526 bench.py $B --config c2 > $O/bench_c2_head_n2.log 2>&1
(cd .cmp/e71 && timeout 300 $TR --master-port 29527 bench.py $B --config c2 > ../../$O/bench_c2_e71_n2.log 2>&1)
timeout 300 $TR --master-port 29528 bench.py $B --config c2 --schedule deferred > $O/bench_c2_deferred_n2.log 2>&1
timeout 300 $TR --master-port 29529 tools/mc_probe.py > $O/mc_probe.log 2>&1
