R=r77
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -2
timeout 400 python bench.py --no-cpu-baseline > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err; python -c "
import json; d=json.load(open('gpurun_out/${R}_bench.json')); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac']); print({k:round(v['ms_per_step'],3) for k,v in d['stages'].items()})"
