R=r142
source tools/gpu_run45_fn.sh
ll base
for v in 0 128; do PKGPU_I8_L2PROMO=$v ll p$v; done
