R=r102
source tools/gpu_run45_fn.sh
for P in 0 2 4 7; do PKGPU_I8_PREFETCH=$P ll pf$P; done
