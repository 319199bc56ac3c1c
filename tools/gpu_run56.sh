R=r56
source tools/gpu_run45_fn.sh
PKGPU_I8_DEBUG=1 ll nogather
PKGPU_I8_DEBUG=2 ll noop
PKGPU_I8_DEBUG=16 ll oneop
PKGPU_I8_DEBUG=17 ll oneop_nogather
