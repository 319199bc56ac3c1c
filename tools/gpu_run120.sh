R=r120
cfgll() { timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -k regex:m2l_i8 --csv --log-file gpurun_out/${R}_$1_$2.csv python tools/run_config.py --cfg $1 --evals 1 > /dev/null 2>&1; echo "cfg$1 $2 $(python tools/launch_times.py gpurun_out/${R}_$1_$2.csv)"; }
cfgll 4 base
PKGPU_I8_BIGMODE=5 cfgll 4 pd
cfgll 3 base
PKGPU_I8_BIGMODE=5 cfgll 3 pd
for c in 3 4; do python tools/run_config.py --cfg $c --evals 2 > gpurun_out/${R}_t$c.json 2>&1; PKGPU_I8_BIGMODE=5 python tools/run_config.py --cfg $c --evals 2 > gpurun_out/${R}_t${c}pd.json 2>&1; done
for f in gpurun_out/${R}_t*.json; do echo $f $(grep -o '"ms_per_eval": [0-9.]*' $f); done
