R=r133
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -k regex:slot_scan --csv --log-file gpurun_out/${R}_scan.csv python tools/run_cfg2.py --warm 1 --evals 1 > /dev/null 2>&1
python tools/launch_times.py gpurun_out/${R}_scan.csv
python tools/run_cfg2.py --warm 3 --evals 10 --stats > gpurun_out/${R}_s.log 2>&1; python tools/stage_ms.py gpurun_out/${R}_s.log 10 tree lists m2l pinv_up pinv_dn m2m l2l leaf
