R=r29
timeout 120 python -m pytest tests/test_gpu_i8.py -q -x -k gather_gemm_exact 2>&1 | tail -30 > gpurun_out/${R}_i8gemm.log
cat gpurun_out/${R}_i8gemm.log
if grep -q " passed" gpurun_out/${R}_i8gemm.log && ! grep -q "failed" gpurun_out/${R}_i8gemm.log; then
  timeout 600 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -6 > gpurun_out/${R}_pytest.log
  cat gpurun_out/${R}_pytest.log
  for P in 0 1; do
    PKGPU_I8_PAIR=$P timeout 300 python tools/run_cfg2.py --evals 3 --warm 2 --stats > gpurun_out/${R}_stats_pair$P.log 2>&1
    echo "pair=$P"; grep -E "^m2l|timings" gpurun_out/${R}_stats_pair$P.log
  done
fi
