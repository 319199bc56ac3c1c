R=r92
source tools/gpu_run45_fn.sh
ll base
PKGPU_I8_SMALL=5000 ll onerun
PKGPU_I8_SMALL=0 ll sep
