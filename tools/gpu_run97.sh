R=r97
source tools/gpu_run45_fn.sh
timeout 300 python -m pytest tests/test_gpu_i8.py -q -x 2>&1 | tail -1
ll base
PKGPU_I8_NSA=2 ll nsa2
PKGPU_I8_NSA=4 ll nsa4
PKGPU_I8_DEBUG=2 ll noop
