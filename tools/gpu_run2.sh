timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -k "assembly or symmetry or linearity" 2>&1 | tail -60 > gpurun_out/r2_pytest.log
