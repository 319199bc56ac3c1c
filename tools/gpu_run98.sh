R=r98
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:leaf_kernel --launch-count 1 -o gpurun_out/${R}_leaf2 python tools/run_cfg2.py --evals 1 --warm 1 > gpurun_out/${R}.log 2>&1
tail -1 gpurun_out/${R}.log
