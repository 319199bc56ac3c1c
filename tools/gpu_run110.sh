R=r110
cfgll() { timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -k regex:m2l_i8 --csv --log-file gpurun_out/${R}_$1_$2.csv python tools/run_config.py --cfg $1 --evals 1 > /dev/null 2>&1; echo "cfg$1 w=$2 $(python tools/launch_times.py gpurun_out/${R}_$1_$2.csv)"; }
for W in 16384 32768 65536; do PKGPU_I8_WINDOW=$W cfgll 4 $W; done
for W in 16384 65536; do PKGPU_I8_WINDOW=$W cfgll 3 $W; done
