R=r66
source tools/gpu_run45_fn.sh
for C in 0 6 9 12 18; do PKGPU_I8_CHUNKS=$C ll c$C; done
