R=r107
cfgll() { timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -k regex:m2l_i8 --csv --log-file gpurun_out/${R}_$1_$2.csv python tools/run_config.py --cfg $1 --evals 1 > /dev/null 2>&1; echo "cfg$1 $2 $(python tools/launch_times.py gpurun_out/${R}_$1_$2.csv)"; }
for C in 1 2 4; do cfgll $C dual; PKGPU_I8_SMALLMODE=0 cfgll $C single; done
for C in 4; do timeout 900 python tools/run_config.py --cfg $C --evals 2 --stats > gpurun_out/${R}_cfg$C.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/${R}_cfg$C.json').read().strip().splitlines()[-1]); print('cfg$C', d['ms_per_eval'], d['stages']['lists']['ms'])"; done
