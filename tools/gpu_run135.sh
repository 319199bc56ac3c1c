R=r135
source tools/gpu_run45_fn.sh
ll base
timeout 900 python tools/run_config.py --cfg 4 --evals 3 --stats > gpurun_out/${R}_cfg4.json 2> gpurun_out/${R}_cfg4.err; echo "cfg4 rc=$? $(grep -o '"ms_per_eval": [0-9.]*' gpurun_out/${R}_cfg4.json)"
