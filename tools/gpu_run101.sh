R=r101
source tools/gpu_run45_fn.sh
cfgll() { timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -k regex:m2l_i8 --csv --log-file gpurun_out/${R}_$1.csv python tools/run_config.py --cfg 3 --evals 1 > /dev/null 2>&1; echo "$1 $(python tools/launch_times.py gpurun_out/${R}_$1.csv)"; }
PKGPU_I8_HINTS=1 timeout 300 python -m pytest tests/test_gpu_i8.py -q -x -k "exact or all_levels" 2>&1 | tail -1
ll base
PKGPU_I8_HINTS=1 ll hints
cfgll c3base
PKGPU_I8_HINTS=1 cfgll c3hints
