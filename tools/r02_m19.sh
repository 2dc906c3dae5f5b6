# 2 GPUs: inbox staging lag 4 (new default) / 6 / 8 + emulated suite -> gpurun_out/r02m19/
O=gpurun_out/r02m19; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0 timeout 600 python -m pytest tests/test_gpu_emulated.py -q > $O/pytest_emulated.log 2>&1; echo RC=$? >> $O/pytest_emulated.log
B="--gpus 2 --steps 60 --warmup 5 --no-cpu --no-e2e --no-interval"
for lag in 4 6 8; do
  CS_MERGE_LAG=$lag timeout 300 $TR --master-port 29691 bench.py $B --config c3 > $O/bench_c3_lag${lag}_n2.log 2>&1
  CS_MERGE_LAG=$lag timeout 300 $TR --master-port 29692 bench.py $B --config c2 > $O/bench_c2_lag${lag}_n2.log 2>&1
done
timeout 300 $TR --master-port 29693 bench.py --gpus 2 --steps 100 --warmup 5 --no-cpu --no-interval --config c3 > $O/bench_c3_default_n2.log 2>&1
