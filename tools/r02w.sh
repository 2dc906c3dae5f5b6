mkdir -p gpurun_out/r02w
run() { tag=$1; shift; timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 50 --warmup 5 --no-e2e --no-interval --no-cpu "$@" > gpurun_out/r02w/${tag}_n${N}.log 2>&1; echo RC=$? >> gpurun_out/r02w/${tag}_n${N}.log; }
N=2
CS_MERGE_TRACE=20 run c2tr --config c2
run c2 --config c2
run c2def --config c2 --schedule deferred
CS_MERGE_LAG=0 run c2l0 --config c2
CS_MERGE_LAG=8 run c2l8 --config c2
