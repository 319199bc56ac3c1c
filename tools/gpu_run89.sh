R=r89
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -2
timeout 300 python tools/run_cfg2.py --evals 6 --warm 2 --stats > gpurun_out/${R}_stats.log 2>&1; grep -E "^tree|^lists|timings" gpurun_out/${R}_stats.log | cut -c1-100
