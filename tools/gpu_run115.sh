R=r115
source tools/gpu_run45_fn.sh
for d in 1 2 3; do PKGPU_I8_DEBUG=$d ll base_d$d; PKGPU_I8_PAIR=5 PKGPU_I8_DEBUG=$d ll pd_d$d; done
