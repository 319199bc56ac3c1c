R=r147
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -1
source tools/gpu_run45_fn.sh
ll base
python tools/run_cfg2.py --warm 3 --evals 10 --stats > gpurun_out/${R}_s.log 2>&1; python tools/stage_ms.py gpurun_out/${R}_s.log 10 m2l
for C in 1 3 4; do timeout 900 python tools/run_config.py --cfg $C --evals 2 --stats > gpurun_out/${R}_cfg$C.json 2> gpurun_out/${R}_cfg$C.err; echo "cfg$C rc=$? $(grep -o '"ms_per_eval": [0-9.]*' gpurun_out/${R}_cfg$C.json)"; done
