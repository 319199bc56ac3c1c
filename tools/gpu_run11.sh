timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -3 > gpurun_out/r11_pytest.log
timeout 300 python tools/run_cfg2.py --evals 3 --warm 2 --stats > gpurun_out/r11_stats.log 2>&1
python tools/run_cfg2.py --evals 1 > gpurun_out/r11_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gather_gemm_tma -s 28 -c 1 -o gpurun_out/r11_m2l_tma python tools/run_cfg2.py --evals 1 > gpurun_out/r11_ncu.log 2>&1
cat gpurun_out/r11_pytest.log; grep -E "m2l|timings" gpurun_out/r11_stats.log
