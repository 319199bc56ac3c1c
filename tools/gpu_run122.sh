R=r122
source tools/gpu_run45_fn.sh
timeout 900 python -m pytest tests/ -q -x -m gpu 2>&1 | tail -2
ll base
python tools/run_cfg2.py --warm 3 --evals 10 --stats > gpurun_out/${R}_sb.log 2>&1
python tools/stage_ms.py gpurun_out/${R}_sb.log 10 m2l pinv_up pinv_dn m2m l2l leaf tree lists
