R=r27
timeout 300 python -m pytest tests/test_gpu_i8.py -q -x -k gather_gemm_exact 2>&1 | tail -30 > gpurun_out/${R}_i8gemm.log
cat gpurun_out/${R}_i8gemm.log
timeout 900 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -6 > gpurun_out/${R}_pytest.log
cat gpurun_out/${R}_pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err
cat gpurun_out/${R}_bench.json; tail -3 gpurun_out/${R}_bench.err
