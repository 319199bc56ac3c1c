R=r73
source tools/gpu_run45_fn.sh
timeout 300 python -m pytest tests/test_gpu_i8.py -q -x 2>&1 | tail -1
PKGPU_I8_PAIR=3 timeout 300 python -m pytest tests/test_gpu_i8.py -q -x -k "all_levels or exact" 2>&1 | tail -1
ll base
PKGPU_I8_PAIR=3 ll dual_all
PKGPU_I8_PAIR=3 timeout 900 python tools/run_config.py --cfg 3 --evals 2 --stats > gpurun_out/${R}_cfg3_dual.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/${R}_cfg3_dual.json').read().strip().splitlines()[-1]); print('cfg3 dual_all', d['ms_per_eval'], d['stages']['m2l_i8']['ms'])"
timeout 900 python tools/run_config.py --cfg 3 --evals 2 --stats > gpurun_out/${R}_cfg3.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/${R}_cfg3.json').read().strip().splitlines()[-1]); print('cfg3 default', d['ms_per_eval'], d['stages']['m2l_i8']['ms'])"
