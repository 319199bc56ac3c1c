R=r123
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:m2l_i8 -o gpurun_out/${R}_m2l python tools/run_cfg2.py --warm 1 --evals 1 > gpurun_out/${R}_ncu.log 2>&1
echo rc=$?
