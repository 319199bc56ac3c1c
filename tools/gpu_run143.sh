R=r143
source tools/gpu_run45_fn.sh
ll base
for v in 128 112 160; do PKGPU_I8_DUAL_NT=$v ll nt$v; done
