R=r117
source tools/gpu_run45_fn.sh
PKGPU_I8_PAIR=5 PKGPU_I8_DEBUG=16 ll pd16
PKGPU_I8_PAIR=5 PKGPU_I8_DEBUG=1 ll pd1
for pf in 4 8 16; do PKGPU_I8_PAIR=5 PKGPU_I8_PREFETCH=$pf ll pf$pf; done
