# End-of-round 1-GPU evidence: full -m gpu suite, smoke, default bench line, reference arm,
# launch list, ncu --set full of the hot kernel, NVML NVLink probe -> gpurun_out/r02final1/
O=gpurun_out/r02final1; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo RC=$? >> $O/pytest_gpu.log
timeout 120 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo RC=$? >> $O/smoke.log
timeout 600 python bench.py > $O/bench.log 2>&1; echo RC=$? >> $O/bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.log 2>&1; echo RC=$? >> $O/bench_ref.log
timeout 300 python tools/nvml_nvlink_probe.py > $O/nvml_nvlink_probe.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > $O/ncu_launches.log 2>&1; echo RC=$? >> $O/ncu_launches.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gossip_tma -s 3 -c 1 -o $O/k_gossip_tma_c2 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-interval > $O/ncu_full.log 2>&1; echo RC=$? >> $O/ncu_full.log
ncu -i $O/k_gossip_tma_c2.ncu-rep --page raw --csv > $O/k_gossip_tma_c2_raw.csv 2>/dev/null
