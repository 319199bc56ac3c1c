R=r70
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/${R}_smi.txt
for C in 1 2 3 4; do timeout 900 python tools/run_config.py --cfg $C --evals 3 --stats > gpurun_out/${R}_cfg$C.json 2> gpurun_out/${R}_cfg$C.err; echo "cfg$C rc=$? $(head -c 300 gpurun_out/${R}_cfg$C.json)"; done
timeout 1500 python tools/run_config.py --cfg 5 --evals 1 --stats > gpurun_out/${R}_cfg5.json 2> gpurun_out/${R}_cfg5.err; echo "cfg5 rc=$? $(head -c 300 gpurun_out/${R}_cfg5.json)"
