R=r94
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -k regex:"gather_gemm|split_reduce" --csv --log-file gpurun_out/${R}_gemm.csv python tools/run_cfg2.py --evals 1 --warm 1 > /dev/null 2>&1
python tools/launch_times.py gpurun_out/${R}_gemm.csv x
