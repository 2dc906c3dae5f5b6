# HEAD check on 1 GPU: gpu suite, smoke, default bench, launch list -> gpurun_out/r02c1/
mkdir -p gpurun_out/r02c1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02c1/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02c1/pytest_gpu.log 2>&1; echo RC=$? >> gpurun_out/r02c1/pytest_gpu.log
timeout 120 python __graft_entry__.py smoke > gpurun_out/r02c1/smoke.log 2>&1; echo RC=$? >> gpurun_out/r02c1/smoke.log
timeout 600 python bench.py > gpurun_out/r02c1/bench.log 2>&1; echo RC=$? >> gpurun_out/r02c1/bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02c1/bench_ref.log 2>&1; echo RC=$? >> gpurun_out/r02c1/bench_ref.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02c1/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/r02c1/ncu.log 2>&1; echo RC=$? >> gpurun_out/r02c1/ncu.log
