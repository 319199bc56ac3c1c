R=r40
timeout 900 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -6 > gpurun_out/${R}_pytest.log; cat gpurun_out/${R}_pytest.log
timeout 300 python tools/run_cfg2.py --evals 3 --warm 2 --stats > gpurun_out/${R}_stats.log 2>&1
grep -E "^m2l|timings" gpurun_out/${R}_stats.log
