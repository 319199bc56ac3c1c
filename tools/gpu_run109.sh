R=r109
source tools/gpu_run45_fn.sh
timeout 300 python -m pytest tests/test_gpu_i8.py -q -x 2>&1 | tail -1
ll base
cfgll() { timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -k regex:m2l_i8 --csv --log-file gpurun_out/${R}_$1.csv python tools/run_config.py --cfg $1 --evals 1 > /dev/null 2>&1; echo "cfg$1 $(python tools/launch_times.py gpurun_out/${R}_$1.csv)"; }
cfgll 4
cfgll 3
