# Final-HEAD 1-GPU re-check: -m gpu suite, smoke, default bench -> gpurun_out/r02final1b/
O=gpurun_out/${OUT:-r02final1b}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo RC=$? >> $O/pytest_gpu.log
timeout 120 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo RC=$? >> $O/smoke.log
timeout 600 python bench.py > $O/bench.log 2>&1; echo RC=$? >> $O/bench.log
