R=r113
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_base.csv python tools/run_cfg2.py --warm 1 --evals 1 > /dev/null 2>&1
echo rc=$?
