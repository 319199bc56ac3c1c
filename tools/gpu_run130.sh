R=r130
source tools/gpu_run45_fn.sh
ll base
for pf in 3 6 12 24; do PKGPU_I8_DUALPF=$pf ll pf$pf; done
