# 2 GPUs: tails merged from their y-out slots; NVLS probes -> gpurun_out/r02m5/
O=gpurun_out/r02m5; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0 timeout 900 python tools/dbg_walk.py 15 > $O/dbg_walk.log 2>&1; echo RC=$? >> $O/dbg_walk.log
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_emulated.py -q -x > $O/pytest_emulated.log 2>&1; echo RC=$? >> $O/pytest_emulated.log
B="--gpus 2 --steps 100 --warmup 5 --no-cpu --no-e2e --no-interval"
for rep in 1 2; do
  timeout 300 $TR --master-port 29541 bench.py $B --config c3 > $O/bench_c3_${rep}_n2.log 2>&1
  timeout 300 $TR --master-port 29542 bench.py $B --config c2 > $O/bench_c2_${rep}_n2.log 2>&1
done
timeout 300 $TR --master-port 29543 bench.py $B --config c5 > $O/bench_c5_n2.log 2>&1
timeout 300 $TR --master-port 29544 bench.py $B --config c3 --wire bf16 > $O/bench_c3_bf16_n2.log 2>&1
for p in 0 1 2; do
  CS_NVLS_PROBE=$p timeout 300 $TR --master-port 29545 bench.py $B --config c4 --h1 nvls > $O/bench_c4_nvls_probe${p}_n2.log 2>&1
done
timeout 2400 python -m pytest tests/test_gpu_multi.py -q -m gpu > $O/pytest_multi_n2.log 2>&1; echo RC=$? >> $O/pytest_multi_n2.log
