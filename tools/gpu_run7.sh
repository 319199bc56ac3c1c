timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -3 > gpurun_out/r7_pytest.log
for g in tma cpasync; do
  PKGPU_GEMM=$g timeout 300 python tools/run_cfg2.py --evals 3 --warm 2 --stats > gpurun_out/r7_stats_$g.log 2>&1
done
cat gpurun_out/r7_pytest.log; grep -E "m2l|pinv_up|m2m|l2l|timings" gpurun_out/r7_stats_*.log
