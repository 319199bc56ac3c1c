R=r60
source tools/gpu_run45_fn.sh
ll new
PKGPU_I8_BYINDEX=0 ll byindex0
timeout 300 python tools/run_cfg2.py --evals 6 --warm 2 --stats > gpurun_out/${R}_stats.log 2>&1; grep -E "^m2l|timings" gpurun_out/${R}_stats.log | cut -c1-90
