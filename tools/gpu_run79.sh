R=r79
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:m2l_i8_dual --launch-skip 3 --launch-count 1 -o gpurun_out/${R}_cfg3 python tools/run_config.py --cfg 3 --evals 1 > gpurun_out/${R}.log 2>&1
tail -2 gpurun_out/${R}.log
