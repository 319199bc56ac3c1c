R=r139
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -1
PKGPU_M2L=dmma timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
python tools/run_cfg2.py --warm 3 --evals 10 --stats > gpurun_out/${R}_s.log 2>&1; python tools/stage_ms.py gpurun_out/${R}_s.log 10 tree lists m2l pinv_up pinv_dn m2m l2l leaf
