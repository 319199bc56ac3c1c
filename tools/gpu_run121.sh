R=r121
source tools/gpu_run45_fn.sh
timeout 300 python -m pytest tests/test_gpu_i8.py tests/test_gpu_parity.py -q -x 2>&1 | tail -1
ll base
PKGPU_I8_BIGMODE=5 ll big5
PKGPU_I8_BIGMODE=5 PKGPU_I8_SMALLMODE=5 ll all5
