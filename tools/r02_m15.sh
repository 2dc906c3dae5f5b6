# 4 GPUs: NCCL h1 parity + c4 benches (nccl vs point-to-point) -> gpurun_out/r02m15/
O=gpurun_out/r02m15; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
B="--gpus 4 --steps 100 --warmup 5 --no-cpu --no-e2e --no-interval"
timeout 300 $TR --master-port 29651 bench.py $B --config c4 --h1 nccl > $O/bench_c4_1x4_nccl_n4.log 2>&1
timeout 300 $TR --master-port 29652 bench.py $B --config c4 > $O/bench_c4_1x4_p2p_n4.log 2>&1
timeout 300 $TR --master-port 29653 bench.py $B --config c4 --hier-groups 2 --h1 nccl > $O/bench_c4_2x2_nccl_n4.log 2>&1
timeout 300 $TR --master-port 29654 bench.py $B --config c4 --hier-groups 2 > $O/bench_c4_2x2_p2p_n4.log 2>&1
timeout 300 $TR --master-port 29655 bench.py $B --config c3 > $O/bench_c3_n4.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -q -m gpu -k "nccl" > $O/pytest_nccl_n4.log 2>&1; echo RC=$? >> $O/pytest_nccl_n4.log
