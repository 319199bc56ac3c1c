R=r145
timeout 900 python -m pytest tests/test_gpu_i8.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -1
source tools/gpu_run45_fn.sh
ll base
PKGPU_I8_NOFIT=1 ll nofit
for C in 3 4; do timeout 900 python tools/run_config.py --cfg $C --evals 2 --stats > gpurun_out/${R}_cfg$C.json 2> gpurun_out/${R}_cfg$C.err; echo "cfg$C rc=$? $(grep -o '"ms_per_eval": [0-9.]*' gpurun_out/${R}_cfg$C.json)"; done
