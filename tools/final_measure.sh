# Round-end single-GPU evidence: tests, smoke, bench lines, ncu launch list and full captures.
mkdir -p gpurun_out/final
O=gpurun_out/final
timeout 1500 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench_c2.log 2>&1; echo "rc=$?" >> $O/bench_c2.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_reference.log 2>&1; echo "rc=$?" >> $O/bench_reference.log
timeout 600 python bench.py --config c6 --steps 50 --warmup 5 > $O/bench_c6.log 2>&1; echo "rc=$?" >> $O/bench_c6.log
# ncu: each command below exited 0 above without ncu
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c2.csv \
  python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > $O/ncu_launches.log 2>&1; echo "rc=$?" >> $O/ncu_launches.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gossip_tma -c 1 -f -o $O/k_gossip_tma_c2 \
  python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-interval > $O/ncu_tma.log 2>&1; echo "rc=$?" >> $O/ncu_tma.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_accumulate --launch-skip 2 -c 1 -f \
  -o $O/k_accumulate_c2 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > $O/ncu_acc.log 2>&1; echo "rc=$?" >> $O/ncu_acc.log
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_lars_norms|k_gossip_tma" -c 2 -f \
  -o $O/k_lars_c6 python bench.py --config c6 --steps 3 --warmup 3 --no-cpu --no-e2e --no-interval > $O/ncu_lars.log 2>&1; echo "rc=$?" >> $O/ncu_lars.log
echo done
