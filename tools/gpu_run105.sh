R=r105
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/${R}_smi.txt
timeout 900 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -2 > gpurun_out/${R}_pytest.log; cat gpurun_out/${R}_pytest.log
timeout 600 python bench.py > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err; tail -c 300 gpurun_out/${R}_bench.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${R}_bench_ref.json 2> gpurun_out/${R}_bench_ref.err; tail -c 300 gpurun_out/${R}_bench_ref.json
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches.csv python tools/run_cfg2.py --evals 1 --warm 1 > /dev/null 2>&1
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:m2l_i8 --launch-count 2 -o gpurun_out/${R}_m2l python tools/run_cfg2.py --evals 1 --warm 1 > gpurun_out/${R}_ncu.log 2>&1
ls gpurun_out | grep $R
