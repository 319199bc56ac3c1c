R=r63
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -3
timeout 300 python tools/run_cfg2.py --evals 6 --warm 2 --stats > gpurun_out/${R}_stats.log 2>&1; grep -E "^m2m|^l2l|^pinv|^m2l|timings" gpurun_out/${R}_stats.log | cut -c1-100
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_all.csv python tools/run_cfg2.py --evals 1 --warm 1 > /dev/null 2>&1
