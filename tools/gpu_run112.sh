R=r112
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:gather_gemm_tma --launch-count 3 -o gpurun_out/${R}_gg python tools/run_cfg2.py --warm 1 --evals 1 > gpurun_out/${R}_ncu.log 2>&1
echo rc=$?
tail -3 gpurun_out/${R}_ncu.log
