R=r114
source tools/gpu_run45_fn.sh
PKGPU_I8_PAIR=5 timeout 300 python -m pytest tests/test_gpu_i8.py -q -x -k "exact or all_levels or agree" 2>&1 | tail -3
ll base
PKGPU_I8_PAIR=5 ll pd
PKGPU_I8_SMALLMODE=5 ll pdsmall
for m in base pd; do :; done
python tools/run_cfg2.py --warm 3 --evals 10 --stats > gpurun_out/${R}_sb.log 2>&1
PKGPU_I8_PAIR=5 python tools/run_cfg2.py --warm 3 --evals 10 --stats > gpurun_out/${R}_sp.log 2>&1
for f in sb sp; do python tools/stage_ms.py gpurun_out/${R}_$f.log 10 m2l pinv_up pinv_dn m2m l2l leaf tree lists; done
