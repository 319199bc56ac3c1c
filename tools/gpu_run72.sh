R=r72
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -k regex:m2l_i8 --csv --log-file gpurun_out/${R}_cfg3.csv python tools/run_config.py --cfg 3 --evals 1 > gpurun_out/${R}_cfg3.log 2>&1
python tools/launch_times.py gpurun_out/${R}_cfg3.csv x
