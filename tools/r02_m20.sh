# 4 GPUs: c3 and the default line with the final staging lag -> gpurun_out/r02m20/
O=gpurun_out/r02m20; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 120 $TR --master-port 29701 bench.py --gpus 4 --steps 100 --warmup 5 --no-cpu --no-e2e --no-interval --config c3 > $O/bench_c3_n4.log 2>&1
timeout 120 $TR --master-port 29702 bench.py --gpus 4 --steps 50 --warmup 5 --no-cpu --no-e2e --no-interval > $O/bench_c2_n4.log 2>&1
