R=r88
source tools/gpu_run45_fn.sh
PKGPU_I8_PAIR=4 timeout 300 python -m pytest tests/test_gpu_i8.py -q -x -k "exact or all_levels" 2>&1 | tail -2
ll base
PKGPU_I8_PAIR=4 ll dualmc
