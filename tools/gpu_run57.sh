R=r57
source tools/gpu_run45_fn.sh
for P in 2 3; do PKGPU_I8_PAIR=$P timeout 300 python -m pytest tests/test_gpu_i8.py -q -x 2>&1 | tail -1; done
PKGPU_I8_PAIR=2 ll mc
PKGPU_I8_PAIR=3 ll dual
PKGPU_I8_PAIR=2 PKGPU_I8_DEBUG=3 ll mc_noloads
PKGPU_I8_PAIR=3 PKGPU_I8_DEBUG=3 ll dual_noloads
