R=r136
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -1
source tools/gpu_run45_fn.sh
ll base
for C in 1 4; do timeout 900 python tools/run_config.py --cfg $C --evals 3 --stats > gpurun_out/${R}_cfg$C.json 2> gpurun_out/${R}_cfg$C.err; echo "cfg$C rc=$? $(grep -o '"ms_per_eval": [0-9.]*' gpurun_out/${R}_cfg$C.json)"; done
