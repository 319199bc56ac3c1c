R=r67
source tools/gpu_run45_fn.sh
ll base
PKGPU_I8_PAIR=3 ll dual_all
PKGPU_I8_DEBUG=16 ll oneop
PKGPU_I8_DEBUG=3 ll noloads
PKGPU_I8_DEBUG=1 ll nogather
PKGPU_I8_DEBUG=2 ll noop
