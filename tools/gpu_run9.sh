timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -3 > gpurun_out/r9_pytest.log
for h in 1 0; do
  PKGPU_GEMM_HINT=$h timeout 300 python tools/run_cfg2.py --evals 3 --warm 2 --stats > gpurun_out/r9_stats_h$h.log 2>&1
done
cat gpurun_out/r9_pytest.log; grep -E "m2l|timings" gpurun_out/r9_stats_*.log
