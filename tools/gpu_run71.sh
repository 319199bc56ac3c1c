R=r71
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -3
for C in 2 3; do timeout 900 python tools/run_config.py --cfg $C --evals 3 --stats > gpurun_out/${R}_cfg$C.json 2> gpurun_out/${R}_cfg$C.err; echo "cfg$C rc=$? $(head -c 250 gpurun_out/${R}_cfg$C.json)"; done
timeout 1500 python tools/run_config.py --cfg 5 --evals 1 --stats > gpurun_out/${R}_cfg5.json 2> gpurun_out/${R}_cfg5.err; echo "cfg5 rc=$? $(head -c 300 gpurun_out/${R}_cfg5.json)"; tail -3 gpurun_out/${R}_cfg5.err
