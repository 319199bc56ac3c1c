R=r80
source tools/gpu_run45_fn.sh
timeout 300 python -m pytest tests/test_gpu_i8.py -q -x 2>&1 | tail -1
ll base
for C in 3 4; do timeout 900 python tools/run_config.py --cfg $C --evals 1 --stats > gpurun_out/${R}_cfg$C.json 2> gpurun_out/${R}_cfg$C.err; python -c "
import json; d=json.loads(open('gpurun_out/${R}_cfg$C.json').read().strip().splitlines()[-1]); st=d['stages']
print($C, d['ms_per_eval'], 'm2l_i8', st['m2l_i8']['ms'])"; done
