R=r100
cfgll() { timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -k regex:m2l_i8 --csv --log-file gpurun_out/${R}_$1.csv python tools/run_config.py --cfg 3 --evals 1 > /dev/null 2>&1; echo "$1 $(python tools/launch_times.py gpurun_out/${R}_$1.csv)"; }
cfgll base
PKGPU_I8_DEBUG=2 cfgll noop
PKGPU_I8_DEBUG=1 cfgll nogather
PKGPU_I8_DEBUG=3 cfgll noloads
