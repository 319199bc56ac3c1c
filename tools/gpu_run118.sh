R=r118
source tools/gpu_run45_fn.sh
PKGPU_I8_PAIR=5 timeout 300 python -m pytest tests/test_gpu_i8.py -q -x -k "exact or all_levels or agree" 2>&1 | tail -2
PKGPU_I8_PAIR=5 ll pd
PKGPU_I8_PAIR=5 PKGPU_I8_DEBUG=2 ll pd_d2
PKGPU_I8_PAIR=5 PKGPU_I8_DEBUG=1 ll pd_d1
PKGPU_I8_PAIR=5 PKGPU_I8_DEBUG=16 ll pd_d16
