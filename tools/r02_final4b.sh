# End-of-round multi-GPU evidence for the final k_push_merge (mix follows the inbox slots):
# benches at N = 2 and 4, then the whole multi-GPU suite on 4 GPUs -> gpurun_out/r02final4b/
O=gpurun_out/r02final4b; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
run() { n=$1; tag=$2; shift 2; DEVS=$(seq -s, 0 $((n - 1)));
  CUDA_VISIBLE_DEVICES=$DEVS timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
    --master-addr 127.0.0.1 --master-port 2971$n bench.py --gpus $n "$@" > $O/bench_${tag}_n$n.log 2>&1; }
for n in 4 2; do
  run $n default --steps 100 --warmup 5
  run $n c3 --config c3 --steps 100 --warmup 5 --no-cpu --no-interval
done
run 4 c5 --config c5 --steps 100 --warmup 5 --no-cpu --no-e2e --no-interval
run 4 c4x2x2 --config c4 --hier-groups 2 --steps 100 --warmup 5 --no-cpu --no-e2e --no-interval
run 4 c3bf16 --config c3 --wire bf16 --steps 100 --warmup 5 --no-cpu --no-e2e --no-interval
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -m gpu > $O/pytest_multi_n4.log 2>&1; echo RC=$? >> $O/pytest_multi_n4.log
