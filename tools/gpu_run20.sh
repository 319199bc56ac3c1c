PKGPU_GEMM_VERBOSE=1 timeout 300 python tools/run_cfg2.py --evals 3 --warm 2 --stats 2>&1 | grep -E "^m2l|timings|pkgpu|Error"
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -2
for c in 3 4; do timeout 600 python tools/run_config.py --cfg $c --evals 2 --stats > gpurun_out/r20_cfg$c.json 2>&1; done
python -c "
import json
for c in (3,4):
    d=json.load(open('gpurun_out/r20_cfg%d.json'%c)); print(c, d['ms_per_eval'], d['stages']['m2l'])"
