timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -k "evaluate or linearity" 2>&1 | tail -3 > gpurun_out/r6_pytest.log
for g in hybrid cpasync; do
  PKGPU_GEMM=$g timeout 300 python tools/run_cfg2.py --evals 3 --warm 2 --stats > gpurun_out/r6_stats_$g.log 2>&1
done
cat gpurun_out/r6_pytest.log; grep -E "m2l|pinv_up|m2m|l2l|timings" gpurun_out/r6_stats_*.log
