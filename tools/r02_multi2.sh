# 2-GPU check of HEAD: multicast probe, multi-GPU suite, bench matrix, NVLink ncu (rank 0) -> gpurun_out/r02m2/
O=gpurun_out/r02m2; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 300 $TR --master-port 29501 tools/mc_probe.py > $O/mc_probe.log 2>&1
NCCL_DEBUG=INFO timeout 300 $TR --master-port 29502 tools/mc_probe.py > $O/mc_probe_ncclinfo.log 2>&1
NCCL_ALGO=NVLS timeout 300 $TR --master-port 29503 tools/mc_probe.py > $O/mc_probe_nvls.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_multi.py -q -m gpu > $O/pytest_multi_n2.log 2>&1; echo RC=$? >> $O/pytest_multi_n2.log
for c in c2 c3 c4 c5; do
  timeout 300 $TR --master-port 29511 bench.py --gpus 2 --config $c --steps 100 --warmup 5 --no-cpu > $O/bench_${c}_n2.log 2>&1; echo RC=$? >> $O/bench_${c}_n2.log
done
timeout 300 $TR --master-port 29512 bench.py --gpus 2 > $O/bench_default_n2.log 2>&1; echo RC=$? >> $O/bench_default_n2.log
for c in c3 c2; do
  NCU_OUT=$O/ncu_nvl_${c}_n2 NCU_KERNELS="k_push_merge|k_hyb|k_peer" timeout 600 $TR --master-port 29513 --no-python bash tools/ncu_rank0.sh bench.py --gpus 2 --config $c --steps 5 --warmup 3 --no-cpu --no-e2e --no-interval > $O/ncu_nvl_${c}_n2.log 2>&1; echo RC=$? >> $O/ncu_nvl_${c}_n2.log
done
