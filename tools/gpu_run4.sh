timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -15 > gpurun_out/r4_pytest.log
for g in tma cpasync; do
  PKGPU_GEMM=$g timeout 300 python tools/run_cfg2.py --evals 3 --warm 2 --stats > gpurun_out/r4_stats_$g.log 2>&1
done
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r4_bench.json 2> gpurun_out/r4_bench.err
cat gpurun_out/r4_pytest.log; grep -E "m2l|pinv|m2m|l2l|timings" gpurun_out/r4_stats_*.log
