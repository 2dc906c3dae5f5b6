mkdir -p gpurun_out/r02t1
timeout 600 python -m pytest tests/test_gpu_emulated.py -q -x > gpurun_out/r02t1/emu.log 2>&1; echo RC=$? >> gpurun_out/r02t1/emu.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_lars.py -q -x > gpurun_out/r02t1/parity_lars.log 2>&1; echo RC=$? >> gpurun_out/r02t1/parity_lars.log
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu > gpurun_out/r02t1/bench_n1.log 2>&1; echo RC=$? >> gpurun_out/r02t1/bench_n1.log
