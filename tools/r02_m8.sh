# 4 GPUs: multi-GPU suite + bench matrix (in-step merge, hierarchical pull / push / NVLS) -> gpurun_out/r02m8/
O=gpurun_out/r02m8; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
B="--gpus 4 --steps 100 --warmup 5 --no-cpu --no-e2e --no-interval"
timeout 600 $TR --master-port 29571 bench.py --gpus 4 > $O/bench_default_n4.log 2>&1
for rep in 1 2; do
  timeout 300 $TR --master-port 29572 bench.py $B --config c3 > $O/bench_c3_${rep}_n4.log 2>&1
done
timeout 300 $TR --master-port 29573 bench.py $B --config c5 > $O/bench_c5_n4.log 2>&1
timeout 300 $TR --master-port 29574 bench.py $B --config c4 > $O/bench_c4_1x4_pull_n4.log 2>&1
CS_HIER_PULL=0 timeout 300 $TR --master-port 29575 bench.py $B --config c4 > $O/bench_c4_1x4_push_n4.log 2>&1
timeout 300 $TR --master-port 29576 bench.py $B --config c4 --h1 nvls > $O/bench_c4_1x4_nvls_n4.log 2>&1
timeout 300 $TR --master-port 29577 bench.py $B --config c4 --hier-groups 2 > $O/bench_c4_2x2_pull_n4.log 2>&1
CS_HIER_PULL=0 timeout 300 $TR --master-port 29578 bench.py $B --config c4 --hier-groups 2 > $O/bench_c4_2x2_push_n4.log 2>&1
timeout 300 $TR --master-port 29579 bench.py $B --config c3 --scheme sgp > $O/bench_sgp_n4.log 2>&1
timeout 300 $TR --master-port 29580 bench.py $B --config c3 --scheme allreduce > $O/bench_allreduce_n4.log 2>&1
timeout 300 $TR --master-port 29581 bench.py $B --config c3 --wire bf16 > $O/bench_c3_bf16_n4.log 2>&1
timeout 300 $TR --master-port 29582 tools/nccl_allreduce.py > $O/nccl_allreduce_n4.log 2>&1
NCCL_DEBUG=INFO timeout 300 $TR --master-port 29583 tools/mc_probe.py > $O/mc_probe_n4.log 2>&1
timeout 3000 python -m pytest tests/test_gpu_multi.py -q -m gpu > $O/pytest_multi_n4.log 2>&1; echo RC=$? >> $O/pytest_multi_n4.log
