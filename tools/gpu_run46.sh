R=r46
source tools/gpu_run45_fn.sh
PKGPU_I8_DEBUG=3 ll noloads
PKGPU_I8_DEBUG=11 ll noloads_nofence
PKGPU_I8_DEBUG=35 ll noloads_plain
PKGPU_I8_DEBUG=43 ll noloads_plain_nofence
PKGPU_I8_DEBUG=8 ll nofence
PKGPU_I8_DEBUG=32 ll plain
