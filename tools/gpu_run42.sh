R=r42
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${R}_smi.txt
timeout 900 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -8 > gpurun_out/${R}_pytest.log; cat gpurun_out/${R}_pytest.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err; tail -c 600 gpurun_out/${R}_bench.json
timeout 300 python tools/run_cfg2.py --evals 6 --warm 2 --stats > gpurun_out/${R}_stats.log 2>&1
grep -E "^m2l|^pinv|^m2m|^l2l|^tree|^lists|^leaf|timings" gpurun_out/${R}_stats.log
