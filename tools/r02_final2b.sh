# 2 GPUs: NVLS h1 tests + c4 NVLS timing after the unroll change -> gpurun_out/r02final2b/
O=gpurun_out/r02final2b; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 240 python -m pytest tests/test_gpu_multi.py -q -m gpu -k "two_gpu_hierarchical_nvls or two_gpu_hierarchical_nccl" > $O/pytest_nvls_n2.log 2>&1; echo RC=$? >> $O/pytest_nvls_n2.log
timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29721 bench.py --gpus 2 --steps 50 --warmup 5 --no-cpu --no-e2e --no-interval --config c4 --h1 nvls > $O/bench_c4_nvls_n2.log 2>&1
