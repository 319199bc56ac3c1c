R=r59
source tools/gpu_run45_fn.sh
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -4
ll new
PKGPU_I8_PAIR=0 ll single
timeout 300 python tools/run_cfg2.py --evals 6 --warm 2 --stats > gpurun_out/${R}_stats.log 2>&1; grep -E "^m2l|timings" gpurun_out/${R}_stats.log | cut -c1-90
