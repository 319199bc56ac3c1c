R=r87
source tools/gpu_run45_fn.sh
ll base
PKGPU_I8_DEBUG=1 ll nogather
PKGPU_I8_DEBUG=2 ll noop
PKGPU_I8_DEBUG=3 ll noloads
