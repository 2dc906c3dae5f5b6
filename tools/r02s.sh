mkdir -p gpurun_out/r02t
run() { tag=$1; shift; timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 50 --warmup 5 --no-e2e --no-interval --no-cpu "$@" > gpurun_out/r02t/${tag}_n${N}.log 2>&1; echo RC=$? >> gpurun_out/r02t/${tag}_n${N}.log; }
for N in 2 4; do
CS_MERGE_TRACE=20 run c3tr --config c3

run c3 --config c3
done
