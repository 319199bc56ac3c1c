R=r84
source tools/gpu_run45_fn.sh
for C in 0 4 5 6 8; do PKGPU_I8_CHUNKS=$C ll c$C; done
