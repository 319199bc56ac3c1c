R=r132
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -1
python tools/run_cfg2.py --warm 3 --evals 10 --stats > gpurun_out/${R}_s.log 2>&1; python tools/stage_ms.py gpurun_out/${R}_s.log 10 tree lists m2l pinv_up pinv_dn m2m l2l leaf
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err; echo "bench rc=$?"; python -c "
import json;d=json.loads(open('gpurun_out/${R}_bench.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['e2e'])"
