# 2 GPUs: the generic-proxy tail merge + dynamic TMA tile claims: races repro, full -m gpu suite,
# c3/c2 bench, 1-GPU c2 static vs dynamic claims -> gpurun_out/r02m4/
O=gpurun_out/r02m4; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for dyn in 1 0 1 0; do
  CS_TMA_DYNAMIC=$dyn CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu --no-e2e --no-interval >> $O/bench_c2_n1_dyn$dyn.log 2>&1
done
CUDA_VISIBLE_DEVICES=0 timeout 600 python tools/dbg_walk.py 15 > $O/dbg_walk.log 2>&1; echo RC=$? >> $O/dbg_walk.log
B="--gpus 2 --steps 100 --warmup 5 --no-cpu --no-e2e --no-interval"
for rep in 1 2; do
  timeout 300 $TR --master-port 29531 bench.py $B --config c3 > $O/bench_c3_${rep}_n2.log 2>&1
  timeout 300 $TR --master-port 29532 bench.py $B --config c2 > $O/bench_c2_${rep}_n2.log 2>&1
done
timeout 300 $TR --master-port 29533 bench.py $B --config c5 > $O/bench_c5_n2.log 2>&1
timeout 2400 python -m pytest tests -q -m gpu > $O/pytest_gpu_n2.log 2>&1; echo RC=$? >> $O/pytest_gpu_n2.log
