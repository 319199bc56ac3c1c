R=r81
source tools/gpu_run45_fn.sh
PKGPU_I8_L2MB=100000 PKGPU_I8_BYINDEX=0 ll dyn_only
PKGPU_I8_L2MB=100000 ll dyn_byindex
PKGPU_I8_L2MB=20 ll dyn_l2_20
cfg() { timeout 900 python tools/run_config.py --cfg $1 --evals 1 --stats > gpurun_out/${R}_$2.json 2> gpurun_out/${R}_$2.err; python -c "
import json; d=json.loads(open('gpurun_out/${R}_$2.json').read().strip().splitlines()[-1]); st=d['stages']
print('$2', d['ms_per_eval'], 'm2l_i8', st['m2l_i8']['ms'])"; }
PKGPU_I8_L2MB=100000 PKGPU_I8_BYINDEX=0 cfg 3 cfg3_dyn_only
PKGPU_I8_L2MB=100000 cfg 3 cfg3_dyn_byindex
PKGPU_I8_L2MB=20 cfg 3 cfg3_l2_20
PKGPU_I8_L2MB=10 cfg 3 cfg3_l2_10
