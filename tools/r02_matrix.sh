# bench matrix at 2 and 4 GPUs (in-step schedule) -> gpurun_out/r02_matrix/
mkdir -p gpurun_out/r02_matrix
run() { tag=$1; shift; timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 50 --warmup 5 --no-e2e --no-interval --no-cpu "$@" > gpurun_out/r02_matrix/${tag}_n${N}.log 2>&1; echo RC=$? >> gpurun_out/r02_matrix/${tag}_n${N}.log; }
for N in 2 4; do
run c3 --config c3
run c4 --config c4
run c4g2 --config c4 --hier-groups 2
run c2 --config c2
run c5 --config c5
run c2def --config c2 --schedule deferred
done
