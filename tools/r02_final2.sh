# Final-HEAD 2-GPU spot check of the multi-GPU parity tests -> gpurun_out/r02final2/
O=gpurun_out/r02final2; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 420 python -m pytest tests/test_gpu_multi.py -q -m gpu -k "two_gpu and (parity or in_step or hierarchical_bitwise)" > $O/pytest_multi_n2.log 2>&1; echo RC=$? >> $O/pytest_multi_n2.log
