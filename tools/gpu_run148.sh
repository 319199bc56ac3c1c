R=r148
python bench.py > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err; echo "bench rc=$?"
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches.csv python tools/run_cfg2.py --warm 1 --evals 1 > /dev/null 2>&1; echo ncu rc=$?
for C in 1 2 3 4; do timeout 900 python tools/run_config.py --cfg $C --evals 5 --stats > gpurun_out/${R}_cfg$C.json 2> gpurun_out/${R}_cfg$C.err; echo "cfg$C rc=$? $(grep -o '"ms_per_eval": [0-9.]*' gpurun_out/${R}_cfg$C.json)"; done
timeout 1500 python tools/run_config.py --cfg 5 --evals 1 --stats > gpurun_out/${R}_cfg5.json 2> gpurun_out/${R}_cfg5.err; echo "cfg5 rc=$? $(grep -o '"ms_per_eval": [0-9.]*' gpurun_out/${R}_cfg5.json)"
