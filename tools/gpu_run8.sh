python tools/run_cfg2.py --evals 1 > gpurun_out/r8_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gather_gemm_tma -s 28 -c 1 -o gpurun_out/r8_m2l_tma python tools/run_cfg2.py --evals 1 > gpurun_out/r8_ncu.log 2>&1
tail -3 gpurun_out/r8_ncu.log
