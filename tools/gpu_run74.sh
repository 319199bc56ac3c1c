R=r74
source tools/gpu_run45_fn.sh
timeout 300 python -m pytest tests/test_gpu_i8.py -q -x 2>&1 | tail -1
ll base
PKGPU_I8_PAIR=3 ll dual_all
