R=r146
source tools/gpu_run45_fn.sh
ll base
PKGPU_I8_NCHUNK_FORCE=2 ll nc2
PKGPU_I8_NCHUNK_FORCE=4 ll nc4
