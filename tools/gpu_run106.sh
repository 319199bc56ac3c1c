R=r106
for C in 1 2 3 4; do timeout 900 python tools/run_config.py --cfg $C --evals 3 --stats > gpurun_out/${R}_cfg$C.json 2> gpurun_out/${R}_cfg$C.err; echo "cfg$C rc=$? $(tail -1 gpurun_out/${R}_cfg$C.json | head -c 200)"; done
timeout 1500 python tools/run_config.py --cfg 5 --evals 1 --stats > gpurun_out/${R}_cfg5.json 2> gpurun_out/${R}_cfg5.err; echo "cfg5 rc=$? $(tail -1 gpurun_out/${R}_cfg5.json | head -c 200)"
