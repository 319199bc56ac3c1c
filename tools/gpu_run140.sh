R=r140
source tools/gpu_run45_fn.sh
ll base
PKGPU_I8_SMALL=100 ll s100
PKGPU_I8_SMALL=100 PKGPU_I8_CHUNKS=8 ll s100c8
PKGPU_I8_SMALL=0 ll s0
for v in 1024 100; do PKGPU_I8_SMALL=$v python tools/run_cfg2.py --warm 3 --evals 10 --stats > gpurun_out/${R}_t$v.log 2>&1; python tools/stage_ms.py gpurun_out/${R}_t$v.log 10 m2l; done
