# Round-end single-GPU refresh: tests, smoke, bench lines, and ncu captures of the multi-GPU
# kernels in single-process peer emulation (every "peer" local; ncu never on multi-rank runs).
mkdir -p gpurun_out/final2
O=gpurun_out/final2
timeout 1500 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench_c2.log 2>&1; echo "rc=$?" >> $O/bench_c2.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_reference.log 2>&1; echo "rc=$?" >> $O/bench_reference.log
CS_PEER_HYBRID=0 timeout 300 python bench.py --config c3 --workers-per-gpu 2 --path peer --steps 30 --warmup 5 --no-cpu --no-e2e --no-interval > $O/bench_emul_push.log 2>&1; echo "rc=$?" >> $O/bench_emul_push.log
CS_PEER_HYBRID=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_peer_push --launch-skip 8 -c 1 -f -o $O/k_peer_push_fused_emul \
  python bench.py --config c3 --workers-per-gpu 2 --path peer --steps 10 --warmup 5 --no-cpu --no-e2e --no-interval > $O/ncu_push.log 2>&1; echo "rc=$?" >> $O/ncu_push.log
timeout 300 python bench.py --config c5 --path peer --steps 30 --warmup 5 --no-cpu --no-e2e --no-interval > $O/bench_emul_hyb.log 2>&1; echo "rc=$?" >> $O/bench_emul_hyb.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hyb_walk --launch-skip 8 -c 1 -f -o $O/k_hyb_walk_emul \
  python bench.py --config c5 --path peer --steps 10 --warmup 5 --no-cpu --no-e2e --no-interval > $O/ncu_hyb.log 2>&1; echo "rc=$?" >> $O/ncu_hyb.log
echo done
