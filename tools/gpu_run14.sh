timeout 900 python -m pytest tests/test_gpu_partition.py -q -rA --timeout 600 2>&1 | tail -25 > gpurun_out/r14_pytest.log
cat gpurun_out/r14_pytest.log
