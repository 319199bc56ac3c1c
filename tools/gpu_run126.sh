R=r126
source tools/gpu_run45_fn.sh
ll base
for c in 6 12; do PKGPU_I8_CHUNKS=$c ll ch$c; done
PKGPU_I8_BYINDEX=1 ll byidx
PKGPU_I8_BYINDEX=1 PKGPU_I8_CHUNKS=8 ll byidx8
PKGPU_I8_SMALLMODE=0 ll single
